// linear.cuh — fused encode + linear-softmax ensemble + readout (K1+K2+K3).
//
// Replaces LinearModelBackend<D>::evaluate (batch_eval.hpp:98-105) and score
// (148-168).  The reference computes logit[c] = sum_j (double)W[c][j]*x[j]
// over the dense one-hot row; with x one-hot the non-zero terms are exactly
// the weights at the active indices, and adding the +/-0.0 products of the
// inactive features never changes a sum that starts at +0.0.  So the kernel
// sums the (<= 20) active weights in ascending feature order in float64 —
// bit-identical to the dense loop — and only rows holding a non-finite weight
// (where inf*0 = NaN matters) replay the dense loop.
//
// Mapping: one warp per state and member, lane l owns classes l, l+32, ...
// Weights are stored transposed [E][F][C] in shared memory (when they fit) so
// a warp's 32 class lanes read 32 consecutive floats for a feature:
// conflict-free broadcast-style gathers.  Packed states are loaded 32 at a
// time (one per lane, coalesced) and h-values are stored 32 at a time.
#pragma once
#include <cstdint>

#include "common.cuh"
#include "encode.cuh"
#include "pdb.cuh"
#include "readout.cuh"

namespace bida_gpu {

struct LinearArgs {
    const void *packed;      // n packed states (device or mapped host)
    int64_t n;
    int32_t *h_out;          // n int32 (device or mapped host)
    double *logits_out;      // optional [n][E][C]
    const float *Wt;         // global [E][F][C]
    const uint8_t *rowflag;  // [E][C]: row holds a non-finite weight
    int E, C;
    double thr;
    float uLo, uHi;          // certified-readout thresholds (certified_readout.cuh)
    int w_in_smem;           // Wt copied to shared memory by every CTA
    int any_rowflag;
    int *err;                // mapped host error words
    unsigned long long *replays;  // readouts that took the exact float64 replay
    PdbArgs pdb;             // optional PDB correction (pdb.cuh)
};

constexpr int kLinearThreads = 256;
constexpr int kLinearWarps = kLinearThreads / 32;

template <int DOMAIN, int CS>
__global__ void __launch_bounds__(kLinearThreads)
linear_eval_kernel(const LinearArgs a) {
    using T = DomainTraits<DOMAIN>;
    constexpr int F = T::F;
    extern __shared__ __align__(16) unsigned char smem[];
    const int C = a.C, E = a.E;
    const int cpad = (C + 1) & ~1;
    const size_t wfloats = static_cast<size_t>(E) * F * C;
    const size_t wbytes = a.w_in_smem ? ((wfloats * 4 + 15) & ~size_t(15)) : 0;
    double *scratch_all = reinterpret_cast<double *>(smem + wbytes);
    int *idx_all = reinterpret_cast<int *>(scratch_all + kLinearWarps * cpad);

    const float *W = a.Wt;
    if (a.w_in_smem) {
        float *sw = reinterpret_cast<float *>(smem);
        const size_t n4 = wfloats / 4;
        const float4 *src = reinterpret_cast<const float4 *>(a.Wt);
        float4 *dst = reinterpret_cast<float4 *>(sw);
        for (size_t i = threadIdx.x; i < n4; i += blockDim.x)
            dst[i] = __ldg(src + i);
        for (size_t i = n4 * 4 + threadIdx.x; i < wfloats; i += blockDim.x)
            sw[i] = __ldg(a.Wt + i);
        __syncthreads();
        W = sw;
    }

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    double *scratch = scratch_all + wib * cpad;
    int *sidx = idx_all + wib * 32;
    const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * kLinearWarps + wib;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kLinearWarps;

    for (int64_t base = gwarp * 32; base < a.n; base += nwarps * 32) {
        const int64_t me = base + lane;
        uint64_t mlo = 0, mhi = 0;
        if (me < a.n) {
            if constexpr (T::PB == 16) {
                const ulonglong2 v = reinterpret_cast<const ulonglong2 *>(a.packed)[me];
                mlo = v.x;
                mhi = v.y;
            } else {
                mlo = reinterpret_cast<const uint64_t *>(a.packed)[me];
            }
        }
        const int cnt = (a.n - base) < 32 ? static_cast<int>(a.n - base) : 32;
        int hres = 0;
        // PDB entry of this lane's own state, fetched before the warp walks the 32 states
        const int hpdb = (a.pdb.entries && me < a.n) ? pdb_fetch<DOMAIN>(a.pdb, mlo) : 0;
        for (int k = 0; k < cnt; ++k) {
            const uint64_t lo = __shfl_sync(kFull, mlo, k);
            const uint64_t hi = (T::PB == 16) ? __shfl_sync(kFull, mhi, k) : 0ull;
            bool bad;
            const int nact = warp_active_indices<DOMAIN>(lo, hi, lane, sidx, &bad);
            int hmin = 0;
            if (bad) {
                if (lane == 0)
                    raise_error(a.err, kErrState);
            } else {
                hmin = 0x7fffffff;
                for (int m = 0; m < E; ++m) {
                    const float *Wm = W + static_cast<size_t>(m) * F * C;
                    double lg[CS];
#pragma unroll
                    for (int s = 0; s < CS; ++s) {
                        const int c = lane + 32 * s;
                        double dot = 0.0;
                        if (c < C) {
                            if (a.any_rowflag && a.rowflag[m * C + c]) {
                                // dense replay of batch_eval.hpp:155-156
                                const float *Wg = a.Wt + static_cast<size_t>(m) * F * C;
                                int t = 0;
                                for (int j = 0; j < F; ++j) {
                                    double x = 0.0;
                                    if (t < nact && sidx[t] == j) {
                                        x = 1.0;
                                        ++t;
                                    }
                                    dot += static_cast<double>(Wg[static_cast<size_t>(j) * C + c]) * x;
                                }
                            } else {
                                for (int t = 0; t < nact; ++t)
                                    dot += static_cast<double>(Wm[sidx[t] * C + c]);
                            }
                        }
                        lg[s] = dot;
                        if (a.logits_out && c < C)
                            a.logits_out[((base + k) * E + m) * C + c] = dot;
                    }
                    const int h = warp_quantile_certified<CS>(lg, C, a.thr, a.uLo, a.uHi, scratch, lane, a.err, a.replays);
                    hmin = min(hmin, h);
                }
            }
            if (lane == k)
                hres = hmin;
            __syncwarp();
        }
        if (me < a.n) {
            if (a.pdb.entries) {
                if (hpdb < 0) {
                    raise_error(a.err, kErrState);
                    hres = 0;
                } else {
                    hres = pdb_combine(a.pdb, hres, hpdb);
                }
            }
            a.h_out[me] = hres;
        }
    }
}

} // namespace bida_gpu
