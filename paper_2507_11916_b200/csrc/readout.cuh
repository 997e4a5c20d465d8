// readout.cuh — the admissible readout, exact in float64.
//
// Restates, per ensemble member, the tail of LinearModelBackend::score
// (batch_eval.hpp:159-166: max_element, exp(l - mx) summed into z in class
// order, p = l / z) and quantile_class with its validate step
// (heuristic.hpp:95-120: smallest c with cum >= q - 1e-12, else C-1; error if
// some p < 0 or |sum p - 1| > 1e-9).  The ensemble minimum
// (heuristic.hpp:122-126) is taken by the caller.
//
// Bit-exactness: every floating-point operation the reference performs is
// performed here in the same order with the same IEEE double rounding —
// sums that the reference accumulates sequentially are accumulated
// sequentially (lanes publish to shared memory, then every lane walks the
// list), division is IEEE '/', and max is order-independent unless a NaN is
// present, in which case the reference's first-wins scan is replayed.  The
// only non-IEEE-specified operation is exp(); see DESIGN.md §3.3.
//
// Layout: one warp per (state, member); lane l owns classes l, l+32, ...
// (CS = class slots per lane).  `scratch` is this warp's C doubles.
#pragma once
#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "sm100.cuh"

namespace bida_gpu {

template <int CS>
__device__ __forceinline__ int warp_quantile_exact(double (&lg)[CS], int C, double thr,
                                                   double *scratch, int lane, int *err_bits) {
    // ---- mx = *max_element(logits) -------------------------------------
    bool nan_here = false;
#pragma unroll
    for (int s = 0; s < CS; ++s) {
        const int c = lane + 32 * s;
        if (c < C && isnan(lg[s]))
            nan_here = true;
    }
    double mx;
    if (!__any_sync(kFull, nan_here)) {
        mx = -INFINITY;
#pragma unroll
        for (int s = 0; s < CS; ++s)
            if (lane + 32 * s < C)
                mx = fmax(mx, lg[s]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
    } else {
        // std::max_element: keep the first element unless (largest < next).
#pragma unroll
        for (int s = 0; s < CS; ++s)
            if (lane + 32 * s < C)
                scratch[lane + 32 * s] = lg[s];
        __syncwarp();
        mx = scratch[0];
        for (int c = 1; c < C; ++c)
            if (mx < scratch[c])
                mx = scratch[c];
        __syncwarp();
    }

    // ---- l = exp(l - mx); z += l in class order -------------------------
#pragma unroll
    for (int s = 0; s < CS; ++s) {
        const int c = lane + 32 * s;
        if (c < C) {
            lg[s] = exp(lg[s] - mx);
            scratch[c] = lg[s];
        }
    }
    __syncwarp();
    double z = 0.0;
    {
        int c = 0;
        for (; c + 4 <= C; c += 4) {
            const double a0 = scratch[c], a1 = scratch[c + 1], a2 = scratch[c + 2], a3 = scratch[c + 3];
            z += a0;
            z += a1;
            z += a2;
            z += a3;
        }
        for (; c < C; ++c)
            z += scratch[c];
    }
    __syncwarp();

    // ---- p = l / z; validate; cumulative walk ---------------------------
    bool neg = false;
#pragma unroll
    for (int s = 0; s < CS; ++s) {
        const int c = lane + 32 * s;
        if (c < C) {
            const double p = lg[s] / z;
            neg |= p < 0.0;
            scratch[c] = p;
        }
    }
    const bool any_neg = __any_sync(kFull, neg);
    __syncwarp();
    double cum = 0.0;
    int hit = -1;
    for (int c = 0; c < C; ++c) {
        cum += scratch[c];
        if (hit < 0 && cum >= thr)
            hit = c;
    }
    __syncwarp();
    // validate() sums p in the same order, so its sum is exactly `cum`.
    if (any_neg || fabs(cum - 1.0) > 1e-9) {
        if (lane == 0)
            raise_error(err_bits, kErrDistribution);
        return 0;
    }
    return hit >= 0 ? hit : C - 1;
}

} // namespace bida_gpu

namespace bida_gpu {

// Warp-parallel certified readout for one (state, member): same decision
// rule and error bound as certified_readout.cuh (thread-per-state), with the
// classes spread over lanes.  Logits lg are exact float64; d_c = lg_c - max
// is formed in float64 and rounded once to float32, exp is ex2.approx, and
// the tail sums T_k = sum_{c>k} e_c and Z come from warp scans.  Terms with
// d_c < -88 underflow (< 1e-38 absolute, far below the comparison slack) and
// are excluded from the relative bound.  Undecided -> exact sequential replay.
template <int CS>
__device__ __forceinline__ int warp_quantile_certified(double (&lg)[CS], int C, double thr, float uLo,
                                                       float uHi, double *scratch, int lane, int *err_bits,
                                                       unsigned long long *replays = nullptr) {
    bool finite = true;
    double mx = -INFINITY;
#pragma unroll
    for (int s = 0; s < CS; ++s)
        if (lane + 32 * s < C) {
            finite &= isfinite(lg[s]);
            mx = fmax(mx, lg[s]);
        }
    if (__all_sync(kFull, finite)) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
        constexpr float kLog2e = 1.4426950408889634f;
        float e[CS];
        float dmax = 0.0f;
        float slot_sum[CS];
#pragma unroll
        for (int s = 0; s < CS; ++s) {
            e[s] = 0.0f;
            if (lane + 32 * s < C) {
                const float d = static_cast<float>(lg[s] - mx);
                if (d >= -88.0f)
                    dmax = fmaxf(dmax, -d);
                e[s] = sm100::ex2_approx(d * kLog2e);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            dmax = fmaxf(dmax, __shfl_xor_sync(kFull, dmax, o));
        // inclusive suffix sums within each slot: S_incl(lane) = sum_{l' >= lane} e
        float incl[CS];
#pragma unroll
        for (int s = 0; s < CS; ++s) {
            float v = e[s];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float t = __shfl_down_sync(kFull, v, o);
                if (lane + o < 32)
                    v += t;
            }
            incl[s] = v;
            slot_sum[s] = __shfl_sync(kFull, v, 0);
        }
        float Z = 0.0f;
#pragma unroll
        for (int s = 0; s < CS; ++s)
            Z += slot_sum[s];
        const float eta = 1.0e-6f * (dmax + 1.0f);
        const float rho = 2.2f * (eta + static_cast<float>(C + 4) * 5.9604645e-8f);
        const float A = uLo * Z * (1.0f - 2.1f * rho);
        const float B = uHi * Z * (1.0f + 2.1f * rho);
        int above = 0;       // classes k with T_k > A
        bool ambiguous = false;
        float later = 0.0f;  // sum of slots after s
#pragma unroll
        for (int s = CS - 1; s >= 0; --s) {
            const int c = lane + 32 * s;
            // exclusive suffix = next lane's inclusive suffix (no cancellation)
            float excl = __shfl_down_sync(kFull, incl[s], 1);
            if (lane == 31)
                excl = 0.0f;
            const float Tk = later + excl;  // sum_{c' > c}
            const bool live = c < C;
            const bool over = live && Tk > A;
            above += __popc(__ballot_sync(kFull, over));
            ambiguous |= __any_sync(kFull, over && !(Tk > B));
            later += slot_sum[s];
        }
        if (!ambiguous)
            return above;  // smallest k with T_k <= A (T_k non-increasing in k)
    }
    if (replays && lane == 0)
        atomicAdd(replays, 1ull);
    return warp_quantile_exact<CS>(lg, C, thr, scratch, lane, err_bits);
}

} // namespace bida_gpu
