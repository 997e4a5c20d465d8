// pdb.cuh — PDB correction in the readout epilogue (north star: "admissible
// class-argmax/PDB-correction readout").
//
// h_PDB = PdbTable::lookup(state) (pdb.hpp:66-69; unreachable 0xFF reads 0)
// with the table index Abstraction::rank_state:
//   Rubik's corners (rubiks.hpp:247-267): pos/ori of each pattern corner,
//     partial_perm_rank(pos, 8) then r = 3 r + ori for each pattern corner;
//   tile puzzle (stp.hpp:208-227): cell of each pattern tile,
//     partial_perm_rank(pos, N*N);
// partial_perm_rank (ranking.hpp:26-51) = sum_i (pos_i - #{j<i: pos_j<pos_i}) * w_i
// with w_i = (n-i-1)(n-i-2)...(n-m+1) precomputed on the host.
// The readout then returns min(h_model, h_PDB) (PDB_MIN, admissible whenever
// the PDB is) or h_PDB with the model still evaluated (PDB_REPLACE: the
// paper's Table-1 mode).
#pragma once
#include <cstdint>

#include "common.cuh"

namespace bida_gpu {

constexpr int kPdbOff = 0, kPdbMin = 1, kPdbReplace = 2;
constexpr int kPdbMaxPattern = 8;

struct PdbArgs {
    const uint8_t *entries;  // device table (nullptr: off)
    unsigned long long n;    // entry count
    unsigned long long w[kPdbMaxPattern];  // rank weights
    int m;                   // pattern length
    int mode;                // kPdbMin / kPdbReplace
    uint8_t pat[kPdbMaxPattern];
};

// Table index of a packed state, or -1 when a pattern label is missing or two
// labels share a position (the reference's partial_perm_rank throws there).
template <int DOMAIN>
__device__ __forceinline__ long long pdb_rank(const PdbArgs &a, uint64_t lo) {
    int pos[kPdbMaxPattern], ori[kPdbMaxPattern];
    constexpr int n = DOMAIN == kRC ? 8 : DOMAIN * DOMAIN;
#pragma unroll
    for (int i = 0; i < kPdbMaxPattern; ++i) {
        pos[i] = -1;
        ori[i] = 0;
        if (i < a.m) {
            const int lbl = a.pat[i];
            if constexpr (DOMAIN == kRC) {
#pragma unroll
                for (int p = 0; p < 8; ++p)
                    if (static_cast<int>((lo >> (3 * p)) & 7u) == lbl) {
                        pos[i] = p;
                        ori[i] = static_cast<int>((lo >> (24 + 2 * p)) & 3u);
                    }
            } else {
#pragma unroll
                for (int c = 0; c < n; ++c)
                    if (static_cast<int>((lo >> (4 * c)) & 15u) == lbl)
                        pos[i] = c;
            }
        }
    }
    long long r = 0;
#pragma unroll
    for (int i = 0; i < kPdbMaxPattern; ++i) {
        if (i < a.m) {
            if (pos[i] < 0)
                return -1;
            int smaller = 0;
#pragma unroll
            for (int j = 0; j < kPdbMaxPattern; ++j)
                if (j < i) {
                    if (pos[j] == pos[i])
                        return -1;
                    smaller += pos[j] < pos[i] ? 1 : 0;
                }
            r += static_cast<long long>(pos[i] - smaller) * static_cast<long long>(a.w[i]);
        }
    }
    if constexpr (DOMAIN == kRC) {
#pragma unroll
        for (int i = 0; i < kPdbMaxPattern; ++i)
            if (i < a.m)
                r = r * 3 + ori[i];
    }
    return r;
}

// Entry for a state: 0..254, or -1 on an invalid state.  Issued early (at
// tile start) so the HBM/L2 latency hides behind the network.
template <int DOMAIN>
__device__ __forceinline__ int pdb_fetch(const PdbArgs &a, uint64_t lo) {
    const long long r = pdb_rank<DOMAIN>(a, lo);
    if (r < 0 || static_cast<unsigned long long>(r) >= a.n)
        return -1;
    const uint8_t e = __ldg(a.entries + r);
    return e == 0xFF ? 0 : static_cast<int>(e);
}

__device__ __forceinline__ int pdb_combine(const PdbArgs &a, int h_model, int h_pdb) {
    return a.mode == kPdbReplace ? h_pdb : (h_pdb < h_model ? h_pdb : h_model);
}

} // namespace bida_gpu
