// linear_thread.cuh — thread-per-state fused encode + linear ensemble + readout.
//
// Same function as linear.cuh (LinearModelBackend<D>::evaluate / score,
// batch_eval.hpp:98-105,148-168; quantile_class / ensemble_min,
// heuristic.hpp:95-126), mapped one THREAD per state instead of one warp per
// state.  The warp mapping left 11 of 32 lanes idle at C = 21 and spent ~876
// warp-instructions per state on match_any / ballot / shuffle encode and the
// warp-wide readout (profiles/r1_v1_linear.txt).  Here:
//
//   encode   the packed state's active feature indices are produced directly
//            in ascending order in registers: for a Rubik's state whose corner
//            and edge labels are permutations (every state the search
//            generates) corner label c owns feature range [24c, 24c+24) and
//            edge label e owns [192+24e, 216+24e), so visiting labels in order
//            IS the ascending order; the per-label slot is gathered through a
//            5-bit field per label in a 64-bit word (no local memory).  STP
//            indices cell*K + tile ascend with the cell.  Anything else (a
//            repeated label, orientation 3) takes a sort-and-deduplicate path
//            with the reference's dense-row semantics (x[j] = 1 once).
//   logits   per class, the float64 sum of the active weights in ascending
//            feature order -- bit-identical to the reference's dense loop
//            (the +-0.0 products of inactive features never change a sum
//            that starts at +0.0).  Weights are [E][F+1][Cp]
//            floats (Cp = C rounded up to 4; row F is all zero and pads a
//            deduplicated list), read as float4 from shared memory.
//   readout  certified float32 softmax / quantile on d_c = l_c - max (formed
//            in float64, rounded once), with the bound of
//            certified_readout.cuh; undecidable states replay the reference's
//            float64 sequence exactly (and are counted in *replays).
//
// Models with C > 96 classes or non-finite weights use linear.cuh.
#pragma once
#include <cmath>
#include <cstdint>

#include "certified_readout.cuh"
#include "common.cuh"
#include "encode.cuh"
#include "pdb.cuh"
#include "sm100.cuh"

namespace bida_gpu {

constexpr int kLinThreads = 256;
constexpr int kLinMaxClasses = 96;

// Ascending, de-duplicated active feature indices of one packed state, padded
// with F (an all-zero weight row).  Returns false for a state whose encode
// leaves [0, F) (the reference's encode would write out of bounds; here
// BIDA_ERR_STATE).
template <int DOMAIN>
__device__ __forceinline__ bool thread_active_indices(uint64_t lo, uint64_t hi, int (&idx)[DomainTraits<DOMAIN>::NNZ]) {
    using T = DomainTraits<DOMAIN>;
    if constexpr (DOMAIN == kRC) {
        if (state_out_of_range<kRC>(lo, hi))
            return false;
        uint64_t cslot = 0, eslot = 0;
        unsigned cmask = 0, emask = 0, co3 = 0;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            const unsigned c = static_cast<unsigned>(lo >> (3 * p)) & 7u;
            const unsigned co = static_cast<unsigned>(lo >> (24 + 2 * p)) & 3u;
            cmask |= 1u << c;
            co3 |= co == 3u;
            cslot |= static_cast<uint64_t>(p * 3 + co) << (5 * c);
        }
#pragma unroll
        for (int p = 0; p < 12; ++p) {
            const unsigned e = static_cast<unsigned>(hi >> (4 * p)) & 15u;
            const unsigned eo = static_cast<unsigned>(lo >> (40 + p)) & 1u;
            emask |= 1u << e;
            eslot |= static_cast<uint64_t>(p * 2 + eo) << (5 * e);
        }
        if (cmask == 0xFFu && emask == 0xFFFu && !co3) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
                idx[c] = c * 24 + static_cast<int>((cslot >> (5 * c)) & 31u);
#pragma unroll
            for (int e = 0; e < 12; ++e)
                idx[8 + e] = 192 + e * 24 + static_cast<int>((eslot >> (5 * e)) & 31u);
            return true;
        }
        // repeated labels / orientation 3: sort + deduplicate (dense-row semantics)
        int v[T::NNZ];
#pragma unroll
        for (int t = 0; t < T::NNZ; ++t)
            v[t] = position_feature<kRC>(lo, hi, t);
        for (int i = 1; i < T::NNZ; ++i)
            for (int j = i; j > 0 && v[j - 1] > v[j]; --j) {
                const int s = v[j];
                v[j] = v[j - 1];
                v[j - 1] = s;
            }
        int k = 0;
        for (int t = 0; t < T::NNZ; ++t)
            if (t == 0 || v[t] != v[t - 1])
                v[k++] = v[t];
        for (int t = k; t < T::NNZ; ++t)
            v[t] = T::F;
#pragma unroll
        for (int t = 0; t < T::NNZ; ++t)
            idx[t] = v[t];
        return true;
    } else {
        if (state_out_of_range<DOMAIN>(lo, hi))
            return false;
#pragma unroll
        for (int t = 0; t < T::NNZ; ++t)
            idx[t] = position_feature<DOMAIN>(lo, hi, t);  // cell*K + tile: ascending, unique
        return true;
    }
}

// float64 logit of class c of one member: ascending sum of the active weights
// (the reference's dense dot product restricted to x[j] = 1).
template <int NNZ>
__device__ __forceinline__ double linear_logit(const float *Wm, int Cp, const int (&idx)[NNZ], int c) {
    double dot = 0.0;
#pragma unroll
    for (int t = 0; t < NNZ; ++t)
        dot += static_cast<double>(Wm[idx[t] * Cp + c]);
    return dot;
}

// The reference's readout sequence replayed exactly (batch_eval.hpp:159-166,
// heuristic.hpp:95-120) from recomputed float64 logits.  Logits are finite
// here (finite weights), so max_element is the plain maximum.
template <int DOMAIN>
__device__ __noinline__ int linear_exact_replay(const float *Wm, int Cp, uint64_t lo, uint64_t hi, int C, double thr,
                                                bool *bad) {
    constexpr int NNZ = DomainTraits<DOMAIN>::NNZ;
    int idx[NNZ];
    thread_active_indices<DOMAIN>(lo, hi, idx);
    double mx = -INFINITY;
    for (int c = 0; c < C; ++c)
        mx = fmax(mx, linear_logit<NNZ>(Wm, Cp, idx, c));
    double z = 0.0;
    for (int c = 0; c < C; ++c)
        z += exp(linear_logit<NNZ>(Wm, Cp, idx, c) - mx);
    double cum = 0.0;
    int hit = -1;
    bool neg = false;
    for (int c = 0; c < C; ++c) {
        const double p = exp(linear_logit<NNZ>(Wm, Cp, idx, c) - mx) / z;
        neg |= p < 0.0;
        cum += p;
        if (hit < 0 && cum >= thr)
            hit = c;
    }
    if (neg || fabs(cum - 1.0) > 1e-9) {
        *bad = true;
        return 0;
    }
    return hit >= 0 ? hit : C - 1;
}

// Certified class from d_c = fl32(l_c - max) <= 0 (certified_readout.cuh's
// bound with eta = 1e-6 (dmax + 1), dmax = largest |d_c| not underflowing);
// -1 when the float32 bound cannot decide.
template <int CM>
__device__ __forceinline__ int certified_from_shifted(const float (&d)[CM], int C, const ReadoutConsts &k) {
    constexpr float kLog2e = 1.4426950408889634f;
    float e[CM];
    float Z = 0.0f, dmax = 0.0f;
#pragma unroll
    for (int c = 0; c < CM; ++c) {
        e[c] = 0.0f;
        if (c < C) {
            if (d[c] >= -88.0f)
                dmax = fmaxf(dmax, -d[c]);
            e[c] = sm100::ex2_approx(d[c] * kLog2e);
        }
        Z += e[c];
    }
    const float eta = 1.0e-6f * (dmax + 1.0f);
    const float rho = 2.2f * (eta + static_cast<float>(C + 4) * 5.9604645e-8f);
    const float A = k.uLo * Z * (1.0f - 2.1f * rho);
    const float B = k.uHi * Z * (1.0f + 2.1f * rho);
    float T = 0.0f;
    int above = 0;
    bool ambiguous = false;
#pragma unroll
    for (int c = CM - 1; c >= 0; --c) {
        const bool over = c < C && T > A;
        above += over ? 1 : 0;
        ambiguous |= over && !(T > B);
        T += e[c];
    }
    return ambiguous ? -1 : above;
}

struct LinearThreadArgs {
    const void *packed;
    int64_t n;
    int32_t *h_out;
    double *logits_out;      // optional [n][E][C]
    const float *W;          // global [E][F+1][Cp]
    int E, C, Cp;
    ReadoutConsts rk;
    int w_in_smem;
    int *err;
    unsigned long long *replays;  // optional: readouts that took the exact replay
    PdbArgs pdb;
};

// CM: class slots (multiple of 4, >= C).  CM <= 32: the float64 logits stay in
// registers; CM > 32: pass 1 finds the float64 maximum, pass 2 recomputes each
// logit and keeps only fl32(l - max) (the register budget of 96 doubles).
template <int DOMAIN, int CM>
__global__ void __launch_bounds__(kLinThreads, CM <= 32 ? 2 : 1)
linear_thread_kernel(const LinearThreadArgs a) {
    using T = DomainTraits<DOMAIN>;
    constexpr int F = T::F;
    constexpr int NNZ = T::NNZ;
    extern __shared__ __align__(16) unsigned char smem[];
    const int C = a.C, Cp = a.Cp, E = a.E;
    const size_t per_member = static_cast<size_t>(F + 1) * Cp;
    const float *W = a.W;
    if (a.w_in_smem) {
        float4 *dst = reinterpret_cast<float4 *>(smem);
        const float4 *src = reinterpret_cast<const float4 *>(a.W);
        const size_t n4 = per_member * E / 4;
        for (size_t i = threadIdx.x; i < n4; i += blockDim.x)
            dst[i] = __ldg(src + i);
        __syncthreads();
        W = reinterpret_cast<const float *>(smem);
    }
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < a.n; s += stride) {
        uint64_t lo, hi = 0;
        if constexpr (T::PB == 16) {
            const ulonglong2 v = reinterpret_cast<const ulonglong2 *>(a.packed)[s];
            lo = v.x;
            hi = v.y;
        } else {
            lo = reinterpret_cast<const uint64_t *>(a.packed)[s];
        }
        const int hpdb = a.pdb.entries ? pdb_fetch<DOMAIN>(a.pdb, lo) : 0;
        int idx[NNZ];
        int h = 0;
        if (!thread_active_indices<DOMAIN>(lo, hi, idx)) {
            raise_error(a.err, kErrState);
        } else {
            int hmin = 0x7fffffff;
            bool bad = false;
            for (int m = 0; m < E; ++m) {
                const float *Wm = W + m * per_member;
                float d[CM];
                if constexpr (CM <= 32) {
                    // feature-major: one weight row (Cp floats) per active
                    // feature, each class's sum still in ascending feature order
                    double l[CM];
#pragma unroll
                    for (int c = 0; c < CM; ++c)
                        l[c] = 0.0;
#pragma unroll
                    for (int t = 0; t < NNZ; ++t) {
                        const float *row = Wm + idx[t] * Cp;
#pragma unroll
                        for (int c0 = 0; c0 < CM; c0 += 4) {
                            if (c0 < C) {  // c0 <= Cp - 4: the float4 stays inside the row
                                const float4 w = *reinterpret_cast<const float4 *>(row + c0);
                                l[c0] += static_cast<double>(w.x);
                                l[c0 + 1] += static_cast<double>(w.y);
                                l[c0 + 2] += static_cast<double>(w.z);
                                l[c0 + 3] += static_cast<double>(w.w);
                            }
                        }
                    }
                    double mx = -INFINITY;
#pragma unroll
                    for (int c = 0; c < CM; ++c)
                        if (c < C) {
                            mx = fmax(mx, l[c]);
                            if (a.logits_out)
                                a.logits_out[(s * E + m) * C + c] = l[c];
                        }
#pragma unroll
                    for (int c = 0; c < CM; ++c)
                        d[c] = static_cast<float>(l[c] - mx);
                } else {
                    double mx = -INFINITY;
#pragma unroll
                    for (int c0 = 0; c0 < CM; c0 += 4) {
                        if (c0 < C) {
                            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
                            for (int t = 0; t < NNZ; ++t) {
                                const float4 w = *reinterpret_cast<const float4 *>(Wm + idx[t] * Cp + c0);
                                a0 += static_cast<double>(w.x);
                                a1 += static_cast<double>(w.y);
                                a2 += static_cast<double>(w.z);
                                a3 += static_cast<double>(w.w);
                            }
                            const double v4[4] = {a0, a1, a2, a3};
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                if (c0 + i < C) {
                                    mx = fmax(mx, v4[i]);
                                    if (a.logits_out)
                                        a.logits_out[(s * E + m) * C + c0 + i] = v4[i];
                                }
                        }
                    }
#pragma unroll
                    for (int c0 = 0; c0 < CM; c0 += 4) {
                        if (c0 < C) {
                            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
                            for (int t = 0; t < NNZ; ++t) {
                                const float4 w = *reinterpret_cast<const float4 *>(Wm + idx[t] * Cp + c0);
                                a0 += static_cast<double>(w.x);
                                a1 += static_cast<double>(w.y);
                                a2 += static_cast<double>(w.z);
                                a3 += static_cast<double>(w.w);
                            }
                            d[c0] = static_cast<float>(a0 - mx);
                            d[c0 + 1] = static_cast<float>(a1 - mx);
                            d[c0 + 2] = static_cast<float>(a2 - mx);
                            d[c0 + 3] = static_cast<float>(a3 - mx);
                        } else {
                            d[c0] = d[c0 + 1] = d[c0 + 2] = d[c0 + 3] = -INFINITY;
                        }
                    }
                }
                int hm = certified_from_shifted<CM>(d, C, a.rk);
                if (hm < 0) {
                    hm = linear_exact_replay<DOMAIN>(Wm, Cp, lo, hi, C, a.rk.thr, &bad);
                    if (a.replays)
                        atomicAdd(a.replays, 1ull);
                }
                hmin = min(hmin, hm);
            }
            if (bad)
                raise_error(a.err, kErrDistribution);
            h = bad ? 0 : hmin;
        }
        if (a.pdb.entries) {
            if (hpdb < 0) {
                raise_error(a.err, kErrState);
                h = 0;
            } else {
                h = pdb_combine(a.pdb, h, hpdb);
            }
        }
        a.h_out[s] = h;
    }
}

} // namespace bida_gpu
