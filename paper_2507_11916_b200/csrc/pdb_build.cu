// pdb_build.cu — PdbTable<D>::build (pdb.hpp:30-64) on the GPU (SURVEY §8(f)
// row 3, optional half): the breadth-first search over the abstract space
// from the abstracted goal, level-synchronous over the whole table.
//
// The reference runs a frontier-vector BFS on one core (the 8-corner Rubik's
// table, 264,539,520 entries, takes ~600 s).  Here level d is one kernel pass
// over the table: every entry equal to d-1 is unranked, its successors are
// generated exactly as Abstraction::successors does, ranked, and every
// successor entry still 0xFF is set to d.  BFS distances are unique, so the
// table is byte-identical to the reference's (tests/test_gpu_pdb_build.py
// compares against tables the reference built, and against the sha256 of the
// reference's 8-corner table).  Concurrent writers of one entry all store the
// same byte d; entries are never read as d-1 and written in the same pass.
//
// Index spaces (restated from the reference):
//   ranking      partial_perm_rank / unrank (ranking.hpp:26-76): lexicographic
//                rank of m distinct positions out of n, weights
//                w_i = (n-i-1)(n-i-2)...(n-m+1)
//   Rubik's      corners only (rubiks.hpp:215-307): rank(pos) * 3^m + the
//                orientations in mixed radix (first pattern corner most
//                significant); a twist moves the corner at position cf[i] to
//                position i and adds co[i] to its orientation (mod 3)
//   tile puzzle  stp.hpp:185-286: with the blank in the pattern the blank
//                swaps with a neighbour cell (carrying a pattern tile found
//                there); without it, each pattern tile steps to a neighbour
//                cell no pattern tile occupies
#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "../../include/bida_gpu.h"

namespace bida_gpu {
std::string &last_error_ref();  // bida_gpu.cu
}

namespace {

constexpr int kMaxPat = 8;
constexpr uint8_t kUnreached = 0xFF;

struct BuildConsts {
    int domain;      // 100: Rubik's corners, N: tile puzzle N x N
    int m;           // pattern length
    int n;           // positions: 8 corners / N*N cells
    int blank_index; // tile puzzle: index of label 0 in the pattern, or -1
    int N;
    unsigned long long w[kMaxPat];  // rank weights
    unsigned long long perm_count;  // n (n-1) ... (n-m+1)
    uint8_t dest[18][8];            // Rubik's: new position of the corner at position p
    uint8_t co_add[18][8];          // Rubik's: twist added on arrival at position i
};

__device__ __forceinline__ unsigned long long perm_rank(const BuildConsts &c, const int (&pos)[kMaxPat]) {
    unsigned long long r = 0;
#pragma unroll
    for (int i = 0; i < kMaxPat; ++i) {
        if (i < c.m) {
            int smaller = 0;
#pragma unroll
            for (int j = 0; j < kMaxPat; ++j)
                if (j < i)
                    smaller += pos[j] < pos[i] ? 1 : 0;
            r += static_cast<unsigned long long>(pos[i] - smaller) * c.w[i];
        }
    }
    return r;
}

// partial_perm_unrank: the idx-th still-available position, in increasing order.
__device__ __forceinline__ void perm_unrank(const BuildConsts &c, unsigned long long r, int (&pos)[kMaxPat]) {
    unsigned used = 0;
#pragma unroll
    for (int i = 0; i < kMaxPat; ++i) {
        if (i < c.m) {
            const int idx = static_cast<int>(r / c.w[i]);
            r %= c.w[i];
            // position of the (idx+1)-th zero bit of `used`
            int k = -1, seen = -1;
            for (int p = 0; p < c.n && seen < idx; ++p)
                if (!((used >> p) & 1u)) {
                    ++seen;
                    k = p;
                }
            pos[i] = k;
            used |= 1u << k;
        }
    }
}

__device__ __forceinline__ void visit(uint8_t *ent, unsigned long long r, uint8_t depth, int *any) {
    if (ent[r] == kUnreached) {
        ent[r] = depth;
        *any = 1;
    }
}

__device__ void expand(const BuildConsts &c, uint8_t *ent, unsigned long long r, uint8_t depth, int *any) {
    int pos[kMaxPat], ori[kMaxPat];
    if (c.domain == 100) {
#pragma unroll
        for (int i = kMaxPat - 1; i >= 0; --i) {
            ori[i] = 0;
            if (i < c.m) {
                ori[i] = static_cast<int>(r % 3);
                r /= 3;
            }
        }
        perm_unrank(c, r, pos);
        for (int a = 0; a < 18; ++a) {
            int np[kMaxPat];
            unsigned long long orr = 0;
#pragma unroll
            for (int i = 0; i < kMaxPat; ++i) {
                np[i] = 0;
                if (i < c.m) {
                    const int d = c.dest[a][pos[i]];
                    np[i] = d;
                    orr = orr * 3 + static_cast<unsigned>((ori[i] + c.co_add[a][d]) % 3);
                }
            }
            unsigned long long p3 = 1;
            for (int i = 0; i < c.m; ++i)
                p3 *= 3;
            visit(ent, perm_rank(c, np) * p3 + orr, depth, any);
        }
        return;
    }
    perm_unrank(c, r, pos);
    const int N = c.N;
    auto neighbours = [&](int cell, int (&nb)[4]) {
        const int row = cell / N, col = cell % N;
        int k = 0;
        if (row > 0) nb[k++] = cell - N;
        if (row < N - 1) nb[k++] = cell + N;
        if (col > 0) nb[k++] = cell - 1;
        if (col < N - 1) nb[k++] = cell + 1;
        return k;
    };
    int nb[4];
    if (c.blank_index >= 0) {
        const int bp = pos[c.blank_index];
        const int deg = neighbours(bp, nb);
        for (int d = 0; d < deg; ++d) {
            int np[kMaxPat];
#pragma unroll
            for (int i = 0; i < kMaxPat; ++i) {
                np[i] = pos[i];
                if (i < c.m && i != c.blank_index && pos[i] == nb[d])
                    np[i] = bp;
            }
            np[c.blank_index] = nb[d];
            visit(ent, perm_rank(c, np), depth, any);
        }
    } else {
        for (int i = 0; i < c.m; ++i) {
            const int deg = neighbours(pos[i], nb);
            for (int d = 0; d < deg; ++d) {
                bool occupied = false;
                for (int j = 0; j < c.m; ++j)
                    occupied |= pos[j] == nb[d];
                if (occupied)
                    continue;
                int np[kMaxPat];
#pragma unroll
                for (int k = 0; k < kMaxPat; ++k)
                    np[k] = pos[k];
                np[i] = nb[d];
                visit(ent, perm_rank(c, np), depth, any);
            }
        }
    }
}

// One BFS level: every entry equal to depth-1 is expanded.  A thread scans 16
// entries with one 16-byte load.
__global__ void pdb_level_kernel(const BuildConsts c, uint8_t *ent, unsigned long long n, uint8_t depth,
                                 int *any) {
    const unsigned long long nvec = (n + 15) / 16;
    const uint8_t want = static_cast<uint8_t>(depth - 1);
    int found = 0;
    for (unsigned long long v = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; v < nvec;
         v += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        unsigned w[4];
        if (v * 16 + 16 <= n) {
            const uint4 q = reinterpret_cast<const uint4 *>(ent)[v];
            w[0] = q.x, w[1] = q.y, w[2] = q.z, w[3] = q.w;
        } else {
            for (int k = 0; k < 4; ++k)
                w[k] = 0xFFFFFFFFu;
            for (int k = 0; v * 16 + k < n; ++k)
                w[k / 4] = (w[k / 4] & ~(0xFFu << (8 * (k % 4)))) | (unsigned(ent[v * 16 + k]) << (8 * (k % 4)));
        }
        unsigned mask = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k)
            mask |= (((w[k / 4] >> (8 * (k % 4))) & 0xFFu) == want ? 1u : 0u) << k;
        while (mask) {
            const int k = __ffs(mask) - 1;
            mask &= mask - 1;
            expand(c, ent, v * 16 + k, depth, &found);
        }
    }
    if (found)
        *any = 1;
}

struct QuarterTurn {
    uint8_t cf[8], co[8];
};

// The six clockwise quarter turns' corner tables (rubiks.hpp move tables: the
// cubie at position cf[i] moves to position i and gains twist co[i]); half and
// counter turns are compositions, as the reference builds them.
constexpr QuarterTurn kQuarter[6] = {
    {{3, 0, 1, 2, 4, 5, 6, 7}, {0, 0, 0, 0, 0, 0, 0, 0}},  // U
    {{0, 1, 2, 3, 5, 6, 7, 4}, {0, 0, 0, 0, 0, 0, 0, 0}},  // D
    {{0, 2, 6, 3, 4, 1, 5, 7}, {0, 1, 2, 0, 0, 2, 1, 0}},  // L
    {{4, 1, 2, 0, 7, 5, 6, 3}, {2, 0, 0, 1, 1, 0, 0, 2}},  // R
    {{1, 5, 2, 3, 0, 4, 6, 7}, {1, 2, 0, 0, 2, 1, 0, 0}},  // F
    {{0, 1, 3, 7, 4, 5, 2, 6}, {0, 0, 1, 2, 0, 0, 2, 1}},  // B
};

QuarterTurn compose(const QuarterTurn &a, const QuarterTurn &b) {  // a then b
    QuarterTurn r{};
    for (int i = 0; i < 8; ++i) {
        r.cf[i] = a.cf[b.cf[i]];
        r.co[i] = static_cast<uint8_t>((a.co[b.cf[i]] + b.co[i]) % 3);
    }
    return r;
}

int set_error(int code, const std::string &msg) {
    bida_gpu::last_error_ref() = msg;
    return code;
}

#define PDB_CUDA(expr)                                                                              \
    do {                                                                                            \
        cudaError_t e_ = (expr);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return set_error(BIDA_ERR_CUDA, std::string(#expr " failed: ") + cudaGetErrorString(e_)); \
    } while (0)

// Validates the pattern and fills the constants; returns the entry count in *size.
int prepare(int domain, const uint8_t *pattern, int m, uint64_t max_entries, BuildConsts *c, uint64_t *size,
            uint64_t *goal_rank) {
    std::memset(c, 0, sizeof(*c));
    const bool rc = domain == BIDA_DOMAIN_RC;
    if (!rc && (domain < BIDA_DOMAIN_STP2 || domain > BIDA_DOMAIN_STP4))
        return set_error(BIDA_ERR_INVALID_ARGUMENT, "unknown domain");
    if (!pattern || m <= 0)
        return set_error(BIDA_ERR_INVALID_ARGUMENT, rc ? "RubiksCube::Abstraction: empty pattern"
                                                       : "TilePuzzle::Abstraction: empty pattern");
    c->domain = rc ? 100 : domain;
    c->N = rc ? 0 : domain;
    c->n = rc ? 8 : domain * domain;
    c->m = m;
    c->blank_index = -1;
    if (m > kMaxPat || m > c->n)
        return set_error(BIDA_ERR_INVALID_ARGUMENT, "PDB pattern must have 1..8 labels");
    for (int i = 0; i < m; ++i) {
        if (pattern[i] >= c->n)
            return set_error(BIDA_ERR_INVALID_ARGUMENT, rc ? "RubiksCube::Abstraction: only corner labels 0..7 supported"
                                                           : "TilePuzzle::Abstraction: label out of range");
        for (int j = 0; j < i; ++j)
            if (pattern[j] == pattern[i])
                return set_error(BIDA_ERR_INVALID_ARGUMENT, "partial_perm_rank: repeated or out-of-range value");
        if (!rc && pattern[i] == 0)
            c->blank_index = i;
    }
    uint64_t count = 1;
    for (int i = 0; i < m; ++i) {
        unsigned long long w = 1;
        for (int a = 0; a < m - i - 1; ++a)
            w *= static_cast<unsigned long long>(c->n - i - 1 - a);
        c->w[i] = w;
        count *= static_cast<uint64_t>(c->n - i);
    }
    c->perm_count = count;
    if (rc)
        for (int i = 0; i < m; ++i)
            count *= 3;
    if (count > max_entries)
        return set_error(BIDA_ERR_RUNTIME, "PDB abstract space needs " + std::to_string(count) +
                                               " entries, cap is " + std::to_string(max_entries));
    *size = count;
    if (rc) {
        QuarterTurn all[18];
        for (int f = 0; f < 6; ++f) {
            all[3 * f] = kQuarter[f];
            all[3 * f + 1] = compose(kQuarter[f], kQuarter[f]);
            all[3 * f + 2] = compose(all[3 * f + 1], kQuarter[f]);
        }
        for (int a = 0; a < 18; ++a)
            for (int i = 0; i < 8; ++i) {
                c->dest[a][all[a].cf[i]] = static_cast<uint8_t>(i);
                c->co_add[a][i] = all[a].co[i];
            }
    }
    // goal = D::solved(): label l sits at position l (cube: orientation 0)
    uint64_t r = 0;
    for (int i = 0; i < m; ++i) {
        int smaller = 0;
        for (int j = 0; j < i; ++j)
            smaller += pattern[j] < pattern[i] ? 1 : 0;
        r += static_cast<uint64_t>(pattern[i] - smaller) * c->w[i];
    }
    if (rc)
        for (int i = 0; i < m; ++i)
            r *= 3;
    *goal_rank = r;
    return BIDA_OK;
}

// Builds into device memory d_ent (size entries); returns the deepest level.
int build_device(const BuildConsts &c, uint8_t *d_ent, uint64_t size, uint64_t goal_rank, int *max_depth) {
    int dev = 0, sms = 148;
    PDB_CUDA(cudaGetDevice(&dev));
    PDB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cudaStream_t st;
    PDB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    int *any = nullptr;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void **>(&any), sizeof(int), cudaHostAllocMapped);
    int *any_dev = nullptr;
    if (e == cudaSuccess)
        e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&any_dev), any, 0);
    if (e == cudaSuccess)
        e = cudaMemsetAsync(d_ent, kUnreached, size, st);
    if (e == cudaSuccess)
        e = cudaMemsetAsync(d_ent + goal_rank, 0, 1, st);
    int depth = 0;
    while (e == cudaSuccess) {
        if (depth == 254) {
            e = cudaErrorInvalidValue;  // cannot happen for the supported spaces (max depth < 100)
            break;
        }
        *any = 0;
        const uint64_t nvec = (size + 15) / 16;
        const int grid = static_cast<int>(std::min<uint64_t>((nvec + 255) / 256, static_cast<uint64_t>(sms) * 8));
        pdb_level_kernel<<<grid, 256, 0, st>>>(c, d_ent, size, static_cast<uint8_t>(depth + 1), any_dev);
        e = cudaGetLastError();
        if (e == cudaSuccess)
            e = cudaStreamSynchronize(st);
        if (e != cudaSuccess || !*(volatile int *)any)
            break;
        ++depth;
    }
    if (any)
        cudaFreeHost(any);
    cudaStreamDestroy(st);
    if (e != cudaSuccess)
        return set_error(BIDA_ERR_CUDA, std::string("PDB build: ") + cudaGetErrorString(e));
    if (max_depth)
        *max_depth = depth;
    return BIDA_OK;
}

} // namespace

namespace bida_gpu {
// Builds the solved-goal table of `pattern` into fresh device memory on the
// current device (bida_gpu_attach_pdb_built).
int pdb_build_device(int domain, const uint8_t *pattern, int m, uint8_t **d_out, uint64_t *n_out) {
    BuildConsts c;
    uint64_t size = 0, goal = 0;
    if (int rc = prepare(domain, pattern, m, 1ull << 28, &c, &size, &goal))
        return rc;
    uint8_t *d = nullptr;
    PDB_CUDA(cudaMalloc(&d, size));
    if (int rc = build_device(c, d, size, goal, nullptr)) {
        cudaFree(d);
        return rc;
    }
    *d_out = d;
    *n_out = size;
    return BIDA_OK;
}
} // namespace bida_gpu

extern "C" {

int bida_gpu_pdb_build(int device, int domain, const uint8_t *pattern, int pattern_len, uint64_t max_entries,
                       uint8_t *entries_out, uint64_t out_cap, uint64_t *n_entries, int *max_depth) {
    BuildConsts c;
    uint64_t size = 0, goal = 0;
    if (int rc = prepare(domain, pattern, pattern_len, max_entries ? max_entries : (1ull << 28), &c, &size, &goal))
        return rc;
    if (n_entries)
        *n_entries = size;
    if (!entries_out || out_cap < size)
        return set_error(BIDA_ERR_CAPACITY, "PDB larger than the output buffer");
    int ndev = 0;
    PDB_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return set_error(BIDA_ERR_INVALID_ARGUMENT, "device index out of range");
    PDB_CUDA(cudaSetDevice(device));
    uint8_t *d = nullptr;
    PDB_CUDA(cudaMalloc(&d, size));
    int rc = build_device(c, d, size, goal, max_depth);
    if (rc == BIDA_OK) {
        const cudaError_t e = cudaMemcpy(entries_out, d, size, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess)
            rc = set_error(BIDA_ERR_CUDA, std::string("PDB download: ") + cudaGetErrorString(e));
    }
    cudaFree(d);
    return rc;
}

int bida_gpu_pdb_build_save(int device, int domain, const uint8_t *pattern, int pattern_len, const char *path) {
    BuildConsts c;
    uint64_t size = 0, goal = 0;
    if (int rc = prepare(domain, pattern, pattern_len, 1ull << 28, &c, &size, &goal))
        return rc;
    std::vector<uint8_t> ent(size);
    if (int rc = bida_gpu_pdb_build(device, domain, pattern, pattern_len, 1ull << 28, ent.data(), size, nullptr,
                                    nullptr))
        return rc;
    // BPDB1 as PdbTable::save writes it (pdb.hpp:78-96)
    std::ofstream f(path ? path : "", std::ios::binary);
    if (!f)
        return set_error(BIDA_ERR_RUNTIME, std::string("cannot write PDB file: ") + (path ? path : ""));
    const bool rc = domain == BIDA_DOMAIN_RC;
    f.write("BPDB1", 5);
    f.put(rc ? 'R' : 'S');
    f.put(static_cast<char>(rc ? 0 : domain * domain));
    f.put(static_cast<char>(pattern_len));
    f.write(reinterpret_cast<const char *>(pattern), pattern_len);
    for (int i = 0; i < 8; ++i)
        f.put(static_cast<char>((size >> (8 * i)) & 0xFF));
    f.write(reinterpret_cast<const char *>(ent.data()), static_cast<std::streamsize>(size));
    if (!f)
        return set_error(BIDA_ERR_RUNTIME, std::string("short write to PDB file: ") + path);
    return BIDA_OK;
}

} // extern "C"
