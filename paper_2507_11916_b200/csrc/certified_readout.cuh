// certified_readout.cuh — thread-per-state readout: fast float32 path with a
// rigorous error bound, exact float64 replay of the reference when the bound
// cannot decide.
//
// Reference semantics (restated in readout.cuh / the oracle): per member,
// logits -> softmax in float64 (batch_eval.hpp:159-166) -> smallest class c
// with cum_c >= thr = q - 1e-12 (heuristic.hpp:109-120).
//
// Fast path.  The class the reference returns is decided by where the true
// tail mass  t_k = sum_{c>k} exp(l_c) / sum_c exp(l_c)  crosses u = 1 - thr:
// the reference's own float64 cum_k differs from 1 - t_k by at most
// eps64 = (4C+16) 2^-53 (C roundings of exp, z, division and the running sum).
// Here every exp(l_c - m) is computed in float32 with relative error <= eta
// (bounded from |logits| and the ex2.approx error), so the float32 tail sums
// T_k and total Z carry relative error <= eta + C 2^-24 each.  With
// rho = 2.2 (eta + (C+4) 2^-24):
//     T_k <= A = uLo Z (1 - 2.1 rho)   proves  cum_k >= thr   (class k reached)
//     T_k >  B = uHi Z (1 + 2.1 rho)   proves  cum_k <  thr   (not yet)
// where uLo/uHi are (u -/+ eps64) rounded outward to float on the host.  The
// answer is certified when the first k with T_k <= A has T_{k-1} > B;
// otherwise (a tail mass within ~rho of u, or non-finite/huge logits) the
// thread replays the reference's float64 sequence exactly.  Softmax is
// shift-invariant, so the float32 path may subtract its own maximum.
#pragma once
#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "sm100.cuh"

namespace bida_gpu {

struct ReadoutConsts {
    double thr;      // q - 1e-12
    float uLo, uHi;  // (1 - thr) -/+ eps64, rounded outward to float
};

// Exact replay of the reference readout in float64 from the exact logits
// lg_c = (double)v_c * sd.  Returns the class; sets *bad on a validate() failure.
template <int CM>
__device__ __noinline__ int readout_exact(const int32_t *v, int C, double sd, double thr, bool *bad) {
    double mx = static_cast<double>(v[0]) * sd;
    for (int c = 1; c < C; ++c) {
        const double l = static_cast<double>(v[c]) * sd;
        if (mx < l)
            mx = l;
    }
    double z = 0.0;
    for (int c = 0; c < C; ++c)
        z += exp(static_cast<double>(v[c]) * sd - mx);
    double cum = 0.0;
    int hit = -1;
    bool neg = false;
    for (int c = 0; c < C; ++c) {
        const double p = exp(static_cast<double>(v[c]) * sd - mx) / z;
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

// v[0..C): exact integer logits (accumulator + bias); sf/sd: out_scale as
// float/double.  *fell_back reports whether the exact path was needed.
template <int CM>
__device__ __forceinline__ int readout_certified(const int32_t (&v)[CM], int C, float sf, double sd,
                                                 const ReadoutConsts &k, bool *bad, bool *fell_back) {
    constexpr float kLog2e = 1.4426950408889634f;
    // pass 1: logits in float32, their max and max magnitude
    float e[CM];
    float m = -INFINITY, lam = 0.0f;
#pragma unroll
    for (int c = 0; c < CM; ++c) {
        e[c] = static_cast<float>(v[c]) * sf;
        if (c < C) {
            m = fmaxf(m, e[c]);
            lam = fmaxf(lam, fabsf(e[c]));
        }
    }
    const float eta = 1.0e-6f * (lam + 1.0f);
    const float rho = 2.2f * (eta + static_cast<float>(C + 4) * 5.9604645e-8f);
    *fell_back = false;
    if (rho < 1.0e-2f) {  // false for NaN / inf / huge logits
        // pass 2: e_c = exp(l_c - m) (independent, pipelined), Z
        float Z = 0.0f;
#pragma unroll
        for (int c = 0; c < CM; ++c) {
            e[c] = c < C ? sm100::ex2_approx((e[c] - m) * kLog2e) : 0.0f;
            Z += e[c];
        }
        const float A = k.uLo * Z * (1.0f - 2.1f * rho);
        const float B = k.uHi * Z * (1.0f + 2.1f * rho);
        // pass 3, branch-free: T_k = sum_{c > k} e_c; the answer is the number
        // of classes with T_k > A (T is non-increasing in k); every such class
        // must also satisfy T_k > B, else the float32 bound cannot decide.
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
        if (!ambiguous)
            return above;
    }
    *fell_back = true;
    int32_t spill[CM];  // only this branch touches local memory
#pragma unroll
    for (int c = 0; c < CM; ++c)
        spill[c] = v[c];
    return readout_exact<CM>(spill, C, sd, k.thr, bad);
}

} // namespace bida_gpu
