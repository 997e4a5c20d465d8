// encode.cuh — device side of D::encode for packed states.
//
// The reference materialises a dense float one-hot row per node
// (stp.hpp:141-146, rubiks.hpp:155-166) on the searcher thread.  Here a warp
// turns ONE packed state into its sorted, de-duplicated list of active
// feature indices in shared memory (<= 20 entries): lane t computes the index
// contributed by position t, __match_any_sync removes duplicates (the dense
// row has each x[j] = 1 once, however many positions write it), and a rank
// count sorts them ascending — the order the reference's dense dot product
// visits them (batch_eval.hpp:155-156).  The one-hot tile the tensor-core MLP
// consumes is produced from the same list.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace bida_gpu {

// Feature index written by position t of a packed state, or -1 when t is
// beyond the domain's position count.
template <int DOMAIN>
__device__ __forceinline__ int position_feature(uint64_t lo, uint64_t hi, int t) {
    if constexpr (DOMAIN == kRC) {
        if (t < 8) {
            const int c = static_cast<int>((lo >> (3 * t)) & 7u);
            const int co = static_cast<int>((lo >> (24 + 2 * t)) & 3u);
            return c * 24 + t * 3 + co;
        }
        if (t < 20) {
            const int p = t - 8;
            const int e = static_cast<int>((hi >> (4 * p)) & 15u);
            const int eo = static_cast<int>((lo >> (40 + p)) & 1u);
            return 192 + e * 24 + p * 2 + eo;
        }
        return -1;
    } else {
        constexpr int K = DOMAIN * DOMAIN;
        if (t < K)
            return t * K + static_cast<int>((lo >> (4 * t)) & 15u);
        return -1;
    }
}

template <int DOMAIN>
struct DomainTraits;
template <>
struct DomainTraits<kSTP2> { static constexpr int F = 16, NNZ = 4, PB = 8; };
template <>
struct DomainTraits<kSTP3> { static constexpr int F = 81, NNZ = 9, PB = 8; };
template <>
struct DomainTraits<kSTP4> { static constexpr int F = 256, NNZ = 16, PB = 8; };
template <>
struct DomainTraits<kRC> { static constexpr int F = 480, NNZ = 20, PB = 16; };

// True when some position's feature index falls outside [0, F) -- the same
// predicate as checking position_feature() for every position.  Rubik's cube:
// only an edge label >= 12 can leave the range (192 + e*24 + p*2 + eo >= 480
// iff e >= 12; corner indices stay below 192), i.e. bits 3 and 2 of a hi
// nibble both set.
template <int DOMAIN>
__device__ __forceinline__ bool state_out_of_range(uint64_t lo, uint64_t hi) {
    if constexpr (DOMAIN == kRC) {
        return ((hi & (hi << 1)) & 0x888888888888ull) != 0;
    } else {
        using T = DomainTraits<DOMAIN>;
        bool b = false;
#pragma unroll
        for (int q = 0; q < T::NNZ; ++q) {
            const int j = position_feature<DOMAIN>(lo, hi, q);
            b |= j < 0 || j >= T::F;
        }
        return b;
    }
}

// Warp-cooperative: writes the ascending unique active indices of one state
// into sidx[0..count) and returns count.  *bad is set (warp-uniform) when an
// index falls outside [0, F) — a malformed packed state.
template <int DOMAIN>
__device__ __forceinline__ int warp_active_indices(uint64_t lo, uint64_t hi, int lane, int *sidx,
                                                   bool *bad) {
    using T = DomainTraits<DOMAIN>;
    const int v0 = position_feature<DOMAIN>(lo, hi, lane);
    const bool live = lane < T::NNZ;
    *bad = __any_sync(kFull, live && (v0 < 0 || v0 >= T::F));
    const int v = live ? v0 : 0x7fffffff;
    if constexpr (DOMAIN == kSTP4) {
        // cell*16 + tile with tile < 16: strictly ascending and unique.
        if (live)
            sidx[lane] = v;
        __syncwarp();
        return T::NNZ;
    } else {
        const unsigned same = __match_any_sync(kFull, v);
        const unsigned lower = (1u << lane) - 1u;
        const bool uniq = live && (same & lower) == 0u;
        const unsigned um = __ballot_sync(kFull, uniq);
        int rank = 0;
#pragma unroll
        for (int u = 0; u < T::NNZ; ++u) {
            const int w = __shfl_sync(kFull, v, u);
            rank += (((um >> u) & 1u) && w < v) ? 1 : 0;
        }
        if (uniq)
            sidx[rank] = v;
        __syncwarp();
        return __popc(um);
    }
}

} // namespace bida_gpu
