// walks.cu — synthetic benchmark inputs on the device: n packed random-walk
// scrambles (SURVEY.md §8(d) synthetic workload; the reference's generator is
// random_walk_instance, instance.hpp:36-57).  State i is a non-retracting walk
// of len_min + i % (len_max - len_min + 1) moves from the solved state, packed
// as the reference packs it (stp.hpp:121-126, rubiks.hpp:126-137):
//   Rubik's : each move one of the 18 face twists whose face differs from the
//             previous move's face (the first move: any of 18);
//   puzzle  : each move slides the blank to a neighbour cell, never undoing
//             the previous move.
// The RNG is a counter-based splitmix64 stream per state (not mt19937_64): the
// walks have the reference's distribution, not its exact sequences, which
// parity tests take from oracle/_ref instead.  One thread per state, all state
// in registers (packed bit fields, no local memory).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>

#include "../../include/bida_gpu.h"

namespace bida_gpu {
std::string &last_error_ref();  // bida_gpu.cu
}

namespace {

struct RcMoves {
    uint8_t cf[18][8], co[18][8], ef[18][12], eo[18][12];
};
__constant__ RcMoves c_moves;

__device__ __forceinline__ uint64_t splitmix(uint64_t &s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// uniform integer in [0, m)
__device__ __forceinline__ uint32_t draw(uint64_t &s, uint32_t m) {
    return static_cast<uint32_t>(((splitmix(s) >> 32) * m) >> 32);
}

__global__ void rc_walks_kernel(int64_t n, int len_min, int span, uint64_t seed, ulonglong2 *out) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t s = seed ^ (static_cast<uint64_t>(i) * 0xD1B54A32D192ED03ull);
        splitmix(s);
        uint32_t cp = 0, co = 0, eo = 0;
        uint64_t ep = 0;
        for (int p = 0; p < 8; ++p)
            cp |= static_cast<uint32_t>(p) << (3 * p);
        for (int p = 0; p < 12; ++p)
            ep |= static_cast<uint64_t>(p) << (4 * p);
        const int len = len_min + static_cast<int>(i % span);
        int last_face = -1;
        for (int step = 0; step < len; ++step) {
            int face, turn;
            if (last_face < 0) {
                const uint32_t r = draw(s, 18);
                face = static_cast<int>(r / 3);
                turn = static_cast<int>(r % 3);
            } else {
                const uint32_t r = draw(s, 15);
                face = static_cast<int>(r / 3);
                face += face >= last_face ? 1 : 0;
                turn = static_cast<int>(r % 3);
            }
            const int a = face * 3 + turn;
            uint32_t ncp = 0, nco = 0, neo = 0;
            uint64_t nep = 0;
#pragma unroll
            for (int p = 0; p < 8; ++p) {
                const int src = c_moves.cf[a][p];
                ncp |= ((cp >> (3 * src)) & 7u) << (3 * p);
                nco |= ((((co >> (2 * src)) & 3u) + c_moves.co[a][p]) % 3u) << (2 * p);
            }
#pragma unroll
            for (int p = 0; p < 12; ++p) {
                const int src = c_moves.ef[a][p];
                nep |= ((ep >> (4 * src)) & 15ull) << (4 * p);
                neo |= ((((eo >> src) & 1u) + c_moves.eo[a][p]) & 1u) << p;
            }
            cp = ncp, co = nco, ep = nep, eo = neo;
            last_face = face;
        }
        out[i] = make_ulonglong2(static_cast<uint64_t>(cp) | static_cast<uint64_t>(co) << 24 |
                                     static_cast<uint64_t>(eo) << 40,
                                 ep);
    }
}

__global__ void stp_walks_kernel(int N, int64_t n, int len_min, int span, uint64_t seed, uint64_t *out) {
    const int K = N * N;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t s = seed ^ (static_cast<uint64_t>(i) * 0xD1B54A32D192ED03ull);
        splitmix(s);
        uint64_t tiles = 0;
        for (int c = 0; c < K; ++c)
            tiles |= static_cast<uint64_t>(c) << (4 * c);
        int blank = 0, last = -1;  // actions: up, down, left, right; inverse = a ^ 1
        const int len = len_min + static_cast<int>(i % span);
        for (int step = 0; step < len; ++step) {
            const int r = blank / N, c = blank % N;
            unsigned legal = (r > 0 ? 1u : 0u) | (r < N - 1 ? 2u : 0u) | (c > 0 ? 4u : 0u) | (c < N - 1 ? 8u : 0u);
            if (last >= 0)
                legal &= ~(1u << (last ^ 1));
            uint32_t pick = draw(s, static_cast<uint32_t>(__popc(legal)));
            int a = 0;
            for (; a < 4; ++a)
                if ((legal >> a) & 1u) {
                    if (pick == 0)
                        break;
                    --pick;
                }
            const int target = blank + (a == 0 ? -N : a == 1 ? N : a == 2 ? -1 : 1);
            const uint64_t t = (tiles >> (4 * target)) & 15ull;
            tiles &= ~(15ull << (4 * target));
            tiles &= ~(15ull << (4 * blank));
            tiles |= t << (4 * blank);
            blank = target;
            last = a;
        }
        out[i] = tiles;
    }
}

struct Quarter {
    uint8_t cf[8], co[8], ef[12], eo[12];
};
// rubiks.hpp:340-364 quarter turns (U D L R F B), as in instances.py / pdb_build.cu
constexpr Quarter kQ[6] = {
    {{3, 0, 1, 2, 4, 5, 6, 7}, {0, 0, 0, 0, 0, 0, 0, 0}, {3, 0, 1, 2, 4, 5, 6, 7, 8, 9, 10, 11}, {0}},
    {{0, 1, 2, 3, 5, 6, 7, 4}, {0, 0, 0, 0, 0, 0, 0, 0}, {0, 1, 2, 3, 5, 6, 7, 4, 8, 9, 10, 11}, {0}},
    {{0, 2, 6, 3, 4, 1, 5, 7}, {0, 1, 2, 0, 0, 2, 1, 0}, {0, 1, 10, 3, 4, 5, 9, 7, 8, 2, 6, 11}, {0}},
    {{4, 1, 2, 0, 7, 5, 6, 3}, {2, 0, 0, 1, 1, 0, 0, 2}, {8, 1, 2, 3, 11, 5, 6, 7, 4, 9, 10, 0}, {0}},
    {{1, 5, 2, 3, 0, 4, 6, 7}, {1, 2, 0, 0, 2, 1, 0, 0}, {0, 9, 2, 3, 4, 8, 6, 7, 1, 5, 10, 11},
     {0, 1, 0, 0, 0, 1, 0, 0, 1, 1, 0, 0}},
    {{0, 1, 3, 7, 4, 5, 2, 6}, {0, 0, 1, 2, 0, 0, 2, 1}, {0, 1, 2, 11, 4, 5, 6, 10, 8, 9, 3, 7},
     {0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 1, 1}},
};

Quarter compose(const Quarter &a, const Quarter &b) {  // a then b (rubiks.hpp:324-338)
    Quarter r{};
    for (int i = 0; i < 8; ++i) {
        r.cf[i] = a.cf[b.cf[i]];
        r.co[i] = static_cast<uint8_t>((a.co[b.cf[i]] + b.co[i]) % 3);
    }
    for (int i = 0; i < 12; ++i) {
        r.ef[i] = a.ef[b.ef[i]];
        r.eo[i] = static_cast<uint8_t>((a.eo[b.ef[i]] + b.eo[i]) % 2);
    }
    return r;
}

int set_error(int code, const std::string &msg) {
    bida_gpu::last_error_ref() = msg;
    return code;
}

} // namespace

extern "C" int bida_gpu_random_walks(int device, int domain, int64_t n, int len_min, int len_max, uint64_t seed,
                                     void *d_out, void *stream) {
    if (n < 0 || len_min < 0 || len_max < len_min || (n > 0 && !d_out))
        return set_error(BIDA_ERR_INVALID_ARGUMENT, "random walks: bad arguments");
    if (domain != BIDA_DOMAIN_RC && (domain < BIDA_DOMAIN_STP2 || domain > BIDA_DOMAIN_STP4))
        return set_error(BIDA_ERR_INVALID_ARGUMENT, "unknown domain");
    if (n == 0)
        return BIDA_OK;
    cudaError_t e = cudaSetDevice(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (e == cudaSuccess && domain == BIDA_DOMAIN_RC) {
        static thread_local int uploaded_device = -1;
        if (uploaded_device != device) {
            RcMoves m{};
            for (int f = 0; f < 6; ++f) {
                Quarter t[3] = {kQ[f], compose(kQ[f], kQ[f]), Quarter{}};
                t[2] = compose(t[1], kQ[f]);
                for (int k = 0; k < 3; ++k)
                    for (int i = 0; i < 12; ++i) {
                        if (i < 8) {
                            m.cf[f * 3 + k][i] = t[k].cf[i];
                            m.co[f * 3 + k][i] = t[k].co[i];
                        }
                        m.ef[f * 3 + k][i] = t[k].ef[i];
                        m.eo[f * 3 + k][i] = t[k].eo[i];
                    }
            }
            e = cudaMemcpyToSymbol(c_moves, &m, sizeof(m));
            if (e == cudaSuccess)
                uploaded_device = device;
        }
    }
    if (e == cudaSuccess) {
        const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
        if (domain == BIDA_DOMAIN_RC)
            rc_walks_kernel<<<grid, 256, 0, st>>>(n, len_min, len_max - len_min + 1, seed,
                                                  static_cast<ulonglong2 *>(d_out));
        else
            stp_walks_kernel<<<grid, 256, 0, st>>>(domain, n, len_min, len_max - len_min + 1, seed,
                                                   static_cast<uint64_t *>(d_out));
        e = cudaGetLastError();
    }
    if (e != cudaSuccess)
        return set_error(BIDA_ERR_CUDA, std::string("random walks: ") + cudaGetErrorString(e));
    return BIDA_OK;
}
