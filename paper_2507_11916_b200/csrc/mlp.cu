// mlp.cu — BMLP1 integer MLP ensemble: fused encode + tcgen05 int8 MLP +
// certified readout, one persistent CTA per SM.
//
// Per CTA, per tile of 128 states, per ensemble member:
//   encode   : epilogue warps write the one-hot tile x[128][F] (int8, UMMA
//              K-major core-matrix layout) into shared buffer X
//   layer l  : MMA warp issues tcgen05.mma.kind::i8 (M=128, N<=256 per
//              instruction, K=32 per instruction) from the activation buffer
//              and a weight k-chunk streamed by the producer warp with 1-D
//              bulk async copies (TMA engine) into a 4-stage ring; int32
//              accumulators live in TMEM
//   epilogue : tcgen05.ld the accumulator rows, add bias, shift, saturate to
//              u8 0..255 and write the next layer's int8 A operand into the
//              other activation buffer (fused activation / requantisation)
//   readout  : last layer -> exact integer logits -> certified float32
//              softmax/quantile (float64 replay when undecidable) -> min
//              over members -> h
// Warp roles: warp 0 producer (1 thread), warp 1 MMA issuer (1 thread),
// warps 2-9 two encode/epilogue/readout groups (thread = TMEM lane = tile row).
// Schedules: resident / pair / split (mlp_fused_kernel, activations in shared
// memory) and wide (mlp_wide_kernel: hidden layers up to 4096 wide, activations
// in L2-resident global scratch) -- see the comments at each kernel.
//
// Integer arithmetic makes every logit exact, so h is bit-identical to the
// oracle's BMLP1 restatement (oracle/bida_oracle.c) in any MMA order.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "certified_readout.cuh"
#include "common.cuh"
#include "encode.cuh"
#include "mlp.cuh"
#include "pdb.cuh"
#include "sm100.cuh"

namespace bida_gpu {

constexpr int kMaxMembers = 8;
constexpr int kMaxLayers = 5;   // hidden layers <= 4
constexpr int kMaxHidden = 4096;
constexpr int kTileM = 128;
constexpr int kMaxStages = 6;
constexpr int kStageBytes = 16384;
constexpr int kMlpThreads = 320;  // warp 0 producer, warp 1 MMA, warps 2-9 two epilogue groups
constexpr int kKChunk = 32;       // bytes of K per MMA instruction
enum MlpMode { kPair = 0, kSplit = 1, kResident = 2, kWide = 4 };

struct MlpLayer {
    int K, N;          // padded input width (multiple of 32), output width (multiple of 16)
    int nh;            // N-halves streamed/computed separately (split schedule hidden layers: 2)
    int cps;           // K-chunks (of one N-half) per 16 KB stage (streaming modes)
    int shift;         // hidden layers
    int boff;          // bias offset (int32 elements, multiple of 4)
    long long woff;    // weight image offset (bytes)
};

struct MlpParams {
    const uint8_t *wimg;
    const int32_t *bias;
    int E, nl, C, Fpad;
    MlpLayer layer[kMaxMembers][kMaxLayers];
    float scale_f[kMaxMembers];
    double scale_d[kMaxMembers];
    ReadoutConsts rk;
    uint32_t tmem_cols;
    int mode;           // MlpMode
    int cluster;        // 2: CTA pairs share weight stages by TMA multicast (streaming modes)
    int stages;         // weight ring depth (16 KB stages), streaming modes
    int wbytes, wbytes_pad;  // weight image bytes (resident mode)
    int xbytes, ybytes; // activation buffers per slot (even / odd layer inputs)
    // batch
    const void *packed;
    long long n;
    int32_t *h_out;
    double *logits_out;
    int *err;
    unsigned long long *replays;  // optional: readouts that took the exact float64 replay
    long long *trace;   // optional debug timeline (CTA 0): [warp][kTraceSlots] (clock64, tag)
    PdbArgs pdb;        // optional PDB correction (pdb.cuh)
    uint8_t *scratch;   // wide: per-CTA hidden activations, 2 buffers of sbytes (global, L2-resident)
    long long sbytes;
    int stage_bytes;    // wide: bytes per weight/activation stage
    int bias_bytes;     // wide: whole bias vector staged in shared memory (0: read from global)
    int l2hint;         // wide: evict_last L2 policy on scratch stores and stage copies
    int bias_fold;      // resident: biases folded into each layer's accumulator by one
                        // extra MMA K step (bias digits x a constant A block at cA_off)
    int cA_off;         // resident + bias_fold: constant A block offset in the weight image
};

constexpr int kTraceSlots = 256;

// Wide schedule: activation scratch buffers allocated once per model; a launch
// takes one round-robin and orders itself after the buffer's previous user
// with an event (stream-ordered reuse, so concurrent callers on different
// streams never share a buffer in flight).
constexpr int kScratchPool = 4;

struct MlpModel {
    MlpParams p;
    uint8_t *d_wimg = nullptr;
    int32_t *d_bias = nullptr;
    size_t smem = 0;
    int grid_cap = 148;
    int cm = 32;
    long long *trace = nullptr;  // debug timeline buffer (bida_gpu_debug_trace)
    std::once_flag attr_once;    // dynamic-smem attribute set at the first launch only
    cudaError_t attr_err = cudaSuccess;
    uint8_t *scratch[kScratchPool] = {};
    cudaEvent_t scratch_ev[kScratchPool] = {};
    std::mutex scratch_mu[kScratchPool];
    std::atomic<unsigned> scratch_next{0};
};

void mlp_set_trace(MlpModel *m, long long *dev_buf) { m->trace = dev_buf; }
int mlp_trace_slots() { return kTraceSlots; }

namespace {
thread_local std::string g_err;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Debug timeline: lane 0 of each warp of CTA 0 appends (clock64 << 8 | tag).
// Compiled in only for the diagnostic library (build.py trace=True,
// -DBIDA_MLP_TRACE=1): the per-call checks cost ~6% of the fused kernel's
// instructions (profiles/r1_notes.md).
#ifndef BIDA_MLP_TRACE
#define BIDA_MLP_TRACE 0
#endif
struct Tracer {
    static constexpr bool kOn = BIDA_MLP_TRACE != 0;
    long long *buf = nullptr;
    int n = 0;
    __device__ bool on() const { return kOn && buf != nullptr; }
    __device__ void operator()(int tag) {
        if (on() && n < kTraceSlots)
            buf[n++] = (clock64() << 8) | (tag & 0xFF);
    }
    __device__ void value(long long v, int tag) {  // a value instead of a timestamp
        if (on() && n < kTraceSlots)
            buf[n++] = (v << 8) | (tag & 0xFF);
    }
};
} // namespace

// Hidden-layer epilogue of one thread (= TMEM lane = tile row): TMEM columns
// [t0, t0 + n) (n a multiple of 16) hold output columns [o0, o0 + n); each is
// requantised, (acc + bias) >> sh saturated to u8, and stored as the next
// layer's K-major A operand -- into shared memory at `sout` (GLOBAL = false)
// or global scratch at `gout` (GLOBAL = true, 4 KB per 32 columns).  The
// TMEM loads of up to 64 columns are issued back to back and waited for once:
// a tcgen05.ld round trip costs several hundred cycles, so one wait per 16
// columns made the drain latency-bound.
// `bias` (global) or, when bias_s != 0, the same vector staged in shared
// memory at bias_s (the wide schedule: its L1 is too small to keep it).
template <bool GLOBAL>
__device__ __forceinline__ void requant_block(uint32_t t_row, int t0, const int32_t *bias, int o0, int n, int sh,
                                              uint32_t sout, uint8_t *gout, int row, uint32_t bias_s = 0u,
                                              uint64_t l2pol = 0) {
    for (int j = 0; j < n; j += 64) {
        const int m = min(64, n - j);
        int32_t r[4][16];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q * 16 < m)
                sm100::tmem_ld16(t_row + t0 + j + q * 16, r[q]);
        sm100::tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (q * 16 >= m)
                break;
            const int oc = o0 + j + q * 16;
            int4 b4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                b4[u] = bias_s ? sm100::ld_shared_v4(bias_s + (oc + 4 * u) * 4u)
                               : __ldg(reinterpret_cast<const int4 *>(bias + oc) + u);
            uint32_t w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                w[u] = sm100::pack_sat_u8x4((r[q][u * 4 + 0] + b4[u].x) >> sh, (r[q][u * 4 + 1] + b4[u].y) >> sh,
                                            (r[q][u * 4 + 2] + b4[u].z) >> sh, (r[q][u * 4 + 3] + b4[u].w) >> sh);
            if constexpr (GLOBAL) {
                uint8_t *dst = gout + (oc >> 5) * 4096 + ((oc >> 4) & 1) * 2048 + row * 16;
                if (l2pol)
                    sm100::st_global_v4_hint(dst, w[0], w[1], w[2], w[3], l2pol);
                else
                    sm100::st_global_v4(dst, w[0], w[1], w[2], w[3]);
            }
            else
                sm100::st_shared_v4(sout + (oc >> 4) * 2048u + row * 16u, w[0], w[1], w[2], w[3]);
        }
    }
}

// Hidden-layer epilogue into shared memory for the fused schedules (L1-hit
// bias): the TMEM load of the next 16 columns is in flight while the current
// 16 are requantised and stored.  Columns [c_beg, c_end) of this thread's row.
// BIAS = false: the accumulator already holds the bias (MlpParams::bias_fold).
template <bool BIAS>
__device__ __forceinline__ void requant_pipelined(uint32_t t_row, const int32_t *bias, int sh, uint32_t out, int row,
                                                  int c_beg, int c_end) {
    auto requant = [&](const int32_t(&r)[16], const int4(&b4)[4], int c0) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // saturated to u8 0..255
            if constexpr (BIAS)
                w[q] = sm100::pack_sat_u8x4((r[q * 4 + 0] + b4[q].x) >> sh, (r[q * 4 + 1] + b4[q].y) >> sh,
                                            (r[q * 4 + 2] + b4[q].z) >> sh, (r[q * 4 + 3] + b4[q].w) >> sh);
            else
                w[q] = sm100::pack_sat_u8x4(r[q * 4 + 0] >> sh, r[q * 4 + 1] >> sh, r[q * 4 + 2] >> sh,
                                            r[q * 4 + 3] >> sh);
        }
        sm100::st_shared_v4(out + (c0 >> 4) * 2048u + row * 16u, w[0], w[1], w[2], w[3]);
    };
    auto load_bias = [&](int4(&b4)[4], int c0) {
        if constexpr (BIAS) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                b4[q] = __ldg(reinterpret_cast<const int4 *>(bias + c0) + q);
        }
    };
    int32_t ra[16], rb[16];
    int4 ba[4], bb[4];
    sm100::tmem_ld16(t_row + c_beg, ra);
    load_bias(ba, c_beg);
    sm100::tmem_wait_ld();
    for (int c0 = c_beg; c0 < c_end; c0 += 32) {
        const bool has_b = c0 + 16 < c_end;
        if (has_b) {
            sm100::tmem_ld16(t_row + c0 + 16, rb);
            load_bias(bb, c0 + 16);
        }
        requant(ra, ba, c0);
        sm100::tmem_wait_ld();
        if (!has_b)
            break;
        if (c0 + 32 < c_end) {
            sm100::tmem_ld16(t_row + c0 + 32, ra);
            load_bias(ba, c0 + 32);
        }
        requant(rb, bb, c0 + 16);
        sm100::tmem_wait_ld();
    }
}

// One CTA per SM, persistent over the CTA's tiles of 128 states (local tile k
// of this CTA is t = blockIdx.x + k * gridDim.x).  A "job" is one (tile,
// ensemble member) pair.  Three schedules (MlpMode):
//   kPair     : two jobs in flight, epilogue group g owns every other tile
//               (TMEM columns [256g, 256g+256)); the MMA issuer interleaves
//               the two tiles layer by layer; weights streamed per tile.
//   kSplit    : one job in flight, the two groups split every hidden layer's
//               columns; weights streamed (wide models, N > 256).
//   kResident : the whole weight image is loaded into SMEM once per CTA;
//               groups split hidden columns; group 1 encodes job j+1 while
//               group 0 reads out job j, and TMEM is double-buffered by job
//               parity so job j+1's MMAs overlap job j's readout.
// VAR: 0 reads the schedule from p.mode; 1 compiles the resident schedule in
// as a constant (the pair/split branches drop out of the hot loops); 2 is
// resident with folded biases and one ensemble member (the common case); 3
// adds a fixed depth of two hidden layers.
template <int DOMAIN, int CM, int VAR = 0>
__global__ void __launch_bounds__(kMlpThreads, 1) mlp_fused_kernel(const __grid_constant__ MlpParams p) {
    using T = DomainTraits<DOMAIN>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int mode = VAR >= 1 ? static_cast<int>(kResident) : p.mode;
    const int nE = VAR >= 2 ? 1 : p.E;
    const bool bfold = VAR >= 2 ? true : p.bias_fold != 0;
    const int nL = VAR == 3 ? 3 : p.nl;  // 3: two hidden layers + the output layer
    const int nsets = mode == kPair ? 2 : 1;  // activation buffer sets
    const int set_bytes = p.xbytes + p.ybytes;
    uint8_t *wbuf = smem + nsets * set_bytes;  // ring stages or resident image
    const int wbuf_bytes = mode == kResident ? p.wbytes_pad : p.stages * kStageBytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(wbuf + wbuf_bytes);
    uint64_t *full = bars;                       // [kMaxStages]
    uint64_t *empty = bars + kMaxStages;         // [kMaxStages]
    uint64_t *act_ready = bars + 2 * kMaxStages; // [2]
    uint64_t *d_full = act_ready + 2;            // [2]
    uint64_t *x_ready = d_full + 2;              // resident: one-hot of the next job written
    uint64_t *w_ready = x_ready + 1;             // resident: weight image landed
    uint64_t *o_full = w_ready + 1;              // split: output-layer accumulator ready
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(o_full + 1);

    const int warp = threadIdx.x >> 5;
    const long long ntiles = (p.n + kTileM - 1) / kTileM;
    // CTA pairs (p.cluster == 2) stream the weights together, so both CTAs of a
    // pair run the same number of tile iterations (the pair's even CTA has the
    // larger share); surplus iterations of the odd CTA are empty tiles.
    const bool mc = p.cluster == 2;
    const uint32_t crank = mc ? sm100::cluster_rank() : 0u;
    const long long b0 = static_cast<long long>(blockIdx.x) - crank;
    const long long nloc = b0 < ntiles ? (ntiles - b0 + gridDim.x - 1) / gridDim.x : 0;
    const bool tdbl = p.tmem_cols == 512u;  // TMEM halves available for double-buffering

    if (threadIdx.x == 0) {
        for (int s = 0; s < kMaxStages; ++s) {
            sm100::mbar_init(&full[s], 1);
            sm100::mbar_init(&empty[s], mc ? 2 : 1);  // both CTAs' MMAs release a shared stage
        }
        for (int s = 0; s < 2; ++s) {
            sm100::mbar_init(&act_ready[s], mode == kResident ? 256 : 128);
            sm100::mbar_init(&d_full[s], 1);
        }
        sm100::mbar_init(x_ready, 128);
        sm100::mbar_init(w_ready, 1);
        sm100::mbar_init(o_full, 1);
        sm100::fence_barrier_init();
    }
    if (warp == 1)
        sm100::tmem_alloc(tmem_slot, p.tmem_cols);
    sm100::tc_fence_before();
    __syncthreads();
    if (mc)
        sm100::cluster_sync();  // peer barriers initialised before any multicast lands
    sm100::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    Tracer tr;
    if (Tracer::kOn && p.trace && blockIdx.x == 0 && lane_id() == 0)
        tr.buf = p.trace + static_cast<long long>(warp) * kTraceSlots;

    if (warp == 0) {
        // ------------------------------------------------ weight producer
        if (lane_id() == 0 && nloc > 0) {
            if (mode == kResident) {
                sm100::mbar_arrive_expect_tx(w_ready, static_cast<uint32_t>(p.wbytes));
                for (int off = 0; off < p.wbytes; off += kStageBytes) {
                    const int b = min(kStageBytes, p.wbytes - off);
                    sm100::bulk_g2s(wbuf + off, p.wimg + off, static_cast<uint32_t>(b), w_ready);
                }
            } else {
                const int per = mode == kPair ? 2 : 1;
                int s = 0;
                uint32_t ph = 0, g = 0;  // g: global stage counter (multicast: CTA g%2 issues)
                for (long long k0 = 0; k0 < nloc; k0 += per)
                    for (int e = 0; e < nE; ++e)
                        for (int l = 0; l < nL; ++l)
                            for (int sl = 0; sl < per && k0 + sl < nloc; ++sl) {
                                const MlpLayer &ly = p.layer[e][l];
                                const int nch = ly.K / kKChunk, cps = ly.cps;
                                const uint32_t cbytes = static_cast<uint32_t>(ly.N / ly.nh) * kKChunk;
                                for (int h = 0; h < ly.nh; ++h)
                                    for (int kc = 0; kc < nch; kc += cps) {
                                        const int cnt = min(cps, nch - kc);
                                        sm100::mbar_wait(&empty[s], ph ^ 1u);
                                        sm100::mbar_arrive_expect_tx(&full[s], cnt * cbytes);
                                        const uint8_t *src = p.wimg + ly.woff + static_cast<size_t>(h * nch + kc) * cbytes;
                                        if (!mc)
                                            sm100::bulk_g2s(wbuf + s * kStageBytes, src, cnt * cbytes, &full[s]);
                                        else if ((g & 1u) == crank)
                                            sm100::bulk_g2s_mc(wbuf + s * kStageBytes, src, cnt * cbytes, &full[s], 0x3);
                                        ++g;
                                        if (++s == p.stages) {
                                            s = 0;
                                            ph ^= 1u;
                                        }
                                    }
                            }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        // The whole warp walks the schedule (uniform control flow, descriptors
        // in uniform registers); one elected lane issues the tcgen05 ops.
        if (nloc > 0 && mode == kSplit) {
            // N-half pipelined schedule: half h of a hidden layer is committed to
            // d_full[h] and drained by group h while the MMAs of the other half
            // (or of the next layer's first K half) run; K-chunks below nch/2 of
            // the next layer need only group 0's output (act_ready[0]).
            int s = 0;
            uint32_t ph = 0, aph[2] = {0u, 0u};
            const uint32_t sbase = sm100::smem_u32(smem), sW = sm100::smem_u32(wbuf);
            for (long long k0 = 0; k0 < nloc; ++k0)
                for (int e = 0; e < nE; ++e) {
                    int prev_half = 0;  // columns group 0 drained in the previous layer (0 = none)
                    for (int l = 0; l < nL; ++l) {
                        const MlpLayer ly = p.layer[e][l];
                        const int nch = ly.K / kKChunk, cps = ly.cps, Nh = ly.N / ly.nh;
                        const uint32_t cbytes = static_cast<uint32_t>(Nh) * kKChunk;
                        const uint32_t idesc = sm100::make_idesc_i8(Nh);
                        const uint32_t abase = sbase + ((l & 1) ? p.xbytes : 0);
                        const int split = nch / 2;  // K-chunks [0, split) come from group 0
                        if (lane_id() == 0)
                            tr(10 + l);
                        sm100::mbar_wait(&act_ready[0], aph[0]);
                        aph[0] ^= 1u;
                        bool have1 = false;
                        // TMEM hazard: this layer's first half writes beyond what group 0 drained
                        if (l == 0 || split == 0 || (prev_half > 0 && Nh > prev_half)) {
                            sm100::mbar_wait(&act_ready[1], aph[1]);
                            aph[1] ^= 1u;
                            have1 = true;
                        }
                        if (lane_id() == 0)
                            tr(20 + l);
                        sm100::tc_fence_after();
                        for (int h = 0; h < ly.nh; ++h) {
                            const uint32_t dcol = tmem + h * Nh;
                            uint64_t adesc = sm100::make_smem_desc(abase, 2048u, 128u);
                            for (int kc = 0; kc < nch; kc += cps) {
                                const int cnt = min(cps, nch - kc);
                                if (!have1 && kc + cnt > split) {
                                    sm100::mbar_wait(&act_ready[1], aph[1]);
                                    aph[1] ^= 1u;
                                    have1 = true;
                                    sm100::tc_fence_after();
                                }
                                sm100::mbar_wait(&full[s], ph);
                                sm100::tc_fence_after();
                                uint64_t bdesc = sm100::make_smem_desc(sW + s * kStageBytes, cbytes >> 1, 128u);
                                if (sm100::elect_one()) {
                                    for (int j = 0; j < cnt; ++j) {
                                        sm100::mma_i8(dcol, adesc, bdesc, idesc, (kc + j) > 0 ? 1u : 0u);
                                        adesc += 4096u >> 4;
                                        bdesc += cbytes >> 4;
                                    }
                                } else {
                                    adesc += static_cast<uint64_t>(cnt) * (4096u >> 4);
                                }
                                __syncwarp();
                                if (sm100::elect_one())
                                    (mc ? sm100::mma_commit_mc(&empty[s], 0x3) : sm100::mma_commit(&empty[s]));
                                __syncwarp();
                                if (++s == p.stages) {
                                    s = 0;
                                    ph ^= 1u;
                                }
                            }
                            if (sm100::elect_one())
                                sm100::mma_commit(l + 1 < nL ? &d_full[h] : o_full);
                            __syncwarp();
                        }
                        if (lane_id() == 0)
                            tr(30 + l);
                        prev_half = ly.N / 2;
                    }
                }
        } else if (nloc > 0) {
            int s = 0;
            uint32_t ph = 0, aph[2] = {0u, 0u}, xph = 0;
            const uint32_t sbase = sm100::smem_u32(smem), sW = sm100::smem_u32(wbuf);
            if (mode == kResident)
                sm100::mbar_wait(w_ready, 0);
            const int per = mode == kPair ? 2 : 1;
            long long job = 0;
            for (long long k0 = 0; k0 < nloc; k0 += per)
                for (int e = 0; e < nE; ++e, ++job)
                    for (int l = 0; l < nL; ++l) {
                        const MlpLayer ly = p.layer[e][l];  // one copy per layer, not per MMA
                        const int nch = ly.K / kKChunk;
                        const int cps = mode == kResident ? nch : ly.cps;
                        const uint32_t cbytes = static_cast<uint32_t>(ly.N) * kKChunk;
                        // pair / resident schedules: every layer is <= 256 wide (one MMA per K step)
                        const uint32_t idesc_a = sm100::make_idesc_i8(ly.N);
                        for (int sl = 0; sl < per && k0 + sl < nloc; ++sl) {
                            if (lane_id() == 0)
                                tr(10 + l + 4 * sl);
                            if (mode == kResident && l == 0) {
                                sm100::mbar_wait(x_ready, xph);
                                xph ^= 1u;
                            } else {
                                sm100::mbar_wait(&act_ready[sl], aph[sl]);
                                aph[sl] ^= 1u;
                            }
                            if (lane_id() == 0)
                                tr(20 + l + 4 * sl);
                            sm100::tc_fence_after();
                            const uint32_t abase = sbase + sl * set_bytes + ((l & 1) ? p.xbytes : 0);
                            const uint32_t dcol =
                                tmem + (mode == kPair ? sl * 256u : (mode == kResident && tdbl ? (job & 1) * 256u : 0u));
                            // descriptor of k-step 0; k-step i adds i*4096 B (A) / i*cbytes (B)
                            uint64_t adesc = sm100::make_smem_desc(abase, 2048u, 128u);
                            const bool fold = mode == kResident && bfold;
                            if (fold && sm100::elect_one())  // D = bias (digits x constant A), then += X.W
                                sm100::mma_i8(dcol, sm100::make_smem_desc(sW + static_cast<uint32_t>(p.cA_off), 2048u, 128u),
                                              sm100::make_smem_desc(sW + static_cast<uint32_t>(ly.woff) + nch * cbytes,
                                                                    cbytes >> 1, 128u),
                                              idesc_a, 0u);
                            for (int kc = 0; kc < nch; kc += cps) {
                                const int cnt = min(cps, nch - kc);
                                uint32_t stg;
                                if (mode == kResident) {
                                    stg = sW + static_cast<uint32_t>(ly.woff) + kc * cbytes;
                                } else {
                                    sm100::mbar_wait(&full[s], ph);
                                    sm100::tc_fence_after();
                                    stg = sW + s * kStageBytes;
                                }
                                uint64_t bdesc = sm100::make_smem_desc(stg, cbytes >> 1, 128u);
                                if (sm100::elect_one()) {
                                    for (int j = 0; j < cnt; ++j) {
                                        const uint32_t acc = (fold || kc + j > 0) ? 1u : 0u;
                                        sm100::mma_i8(dcol, adesc, bdesc, idesc_a, acc);
                                        adesc += 4096u >> 4;
                                        bdesc += cbytes >> 4;
                                    }
                                } else {
                                    adesc += static_cast<uint64_t>(cnt) * (4096u >> 4);
                                }
                                __syncwarp();
                                if (mode != kResident) {
                                    if (sm100::elect_one())
                                        (mc ? sm100::mma_commit_mc(&empty[s], 0x3) : sm100::mma_commit(&empty[s]));
                                    __syncwarp();
                                    if (++s == p.stages) {
                                        s = 0;
                                        ph ^= 1u;
                                    }
                                }
                            }
                            if (sm100::elect_one())
                                sm100::mma_commit(&d_full[sl]);
                            __syncwarp();
                            if (lane_id() == 0)
                                tr(30 + l + 4 * sl);
                        }
                    }
        }
    } else {
        // ------------------------------------------------ encode / epilogue / readout
        const int grp = (warp - 2) >> 2;           // epilogue group 0 / 1
        const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
        const int row = quad * 32 + lane_id();     // tile row == TMEM lane
        const int sl = mode == kPair ? grp : 0;
        const uint32_t sX = sm100::smem_u32(smem) + sl * set_bytes;
        const uint32_t sY = sX + p.xbytes;
        // split: group g owns act_ready[g] / d_full[g] (its K half / N half)
        uint64_t *my_ready = &act_ready[mode == kSplit ? grp : sl];
        uint64_t *my_full = &d_full[mode == kSplit ? grp : sl];
        uint32_t dph = 0, oph = 0;
        // pair: this group's own tiles; split/resident: every tile of the CTA
        const long long kfirst = mode == kPair ? grp : 0, kstep = mode == kPair ? 2 : 1;
        // who encodes / reads out: pair -> both groups (own tiles); split -> group 0;
        // resident -> group 1 encodes (one job ahead), group 0 reads out
        // split: group 1 encodes job j+1 while group 0 reads out job j; group 0
        // releases TMEM (act_ready[0]) as soon as it has loaded job j's logits
        const bool encoder = mode == kPair || grp == 1;
        const bool reader = mode == kPair || grp == 0;

        auto load_state = [&](long long kk, uint64_t &lo_, uint64_t &hi_) {
            lo_ = hi_ = 0;
            const long long s_ = (blockIdx.x + kk * gridDim.x) * kTileM + row;
            if (kk < nloc && s_ < p.n) {
                if constexpr (T::PB == 16) {
                    const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2 *>(p.packed) + s_);
                    lo_ = v.x;
                    hi_ = v.y;
                } else {
                    lo_ = __ldcs(reinterpret_cast<const unsigned long long *>(p.packed) + s_);
                }
            }
        };
        auto state_bad = [&](uint64_t lo_, uint64_t hi_) { return state_out_of_range<DOMAIN>(lo_, hi_); };
        // one-hot row of a packed state into X (layer 0's A operand), then publish
        // (the split schedule's one-hot is written whole by group 1; see below)
        constexpr int kX16 = (T::F + 31) / 32 * 2;  // 16-column chunks of the one-hot tile (Fpad / 16)
        auto encode = [&](uint64_t lo_, uint64_t hi_, bool live_, uint64_t *bar) {
            tr(40);
#pragma unroll
            for (int c16 = 0; c16 < kX16; ++c16)
                sm100::st_shared_v4(sX + c16 * 2048u + row * 16u, 0u, 0u, 0u, 0u);
            if (live_) {
#pragma unroll
                for (int q = 0; q < T::NNZ; ++q) {
                    const int j = position_feature<DOMAIN>(lo_, hi_, q);
                    sm100::st_shared_u8(sX + (j >> 4) * 2048u + row * 16u + (j & 15), 1u);
                }
            }
            sm100::fence_proxy_async_smem();
            tr(41);
            sm100::mbar_arrive(bar);
        };
        auto tile_valid = [&](long long kk) { return kk < nloc && (blockIdx.x + kk * gridDim.x) * kTileM + row < p.n; };

        uint64_t nlo = 0, nhi = 0;
        load_state(kfirst, nlo, nhi);
        if (mode == kResident && encoder && nloc > 0)  // first job's one-hot
            encode(nlo, nhi, tile_valid(kfirst) && !state_bad(nlo, nhi), x_ready);
        long long job = kfirst * nE;
        for (long long k = kfirst; k < nloc; k += kstep) {
            const long long st = (blockIdx.x + k * gridDim.x) * kTileM + row;
            const bool valid = st < p.n;
            const uint64_t lo = nlo, hi = nhi;
            tr(84);
            load_state(k + kstep, nlo, nhi);
            tr(85);
            const bool bad = valid && state_bad(lo, hi);
            // PDB entry prefetched at tile start; consumed when h is written
            const int hpdb = (p.pdb.entries && reader && valid) ? pdb_fetch<DOMAIN>(p.pdb, lo) : 0;
            if (bad && reader)
                raise_error(p.err, kErrState);
            const bool live = valid && !bad;
            int hmin = 0x7fffffff;
            bool dist_bad = false;
            tr(86);
            for (int e = 0; e < nE; ++e, ++job) {
                const uint32_t tcol = mode == kPair ? sl * 256u : (mode == kResident && tdbl ? (job & 1) * 256u : 0u);
                const uint32_t t_row = tmem + tcol + (static_cast<uint32_t>(quad * 32) << 16);
                if (mode != kResident) {
                    if (encoder)
                        encode(lo, hi, live, my_ready);
                    else if (mode != kSplit || job == kfirst * nE)
                        sm100::mbar_arrive(my_ready);  // split: later jobs arrive at the previous readout
                }
                for (int l = 0; l < nL; ++l) {
                    const MlpLayer &ly = p.layer[e][l];
                    tr(50 + l);
                    if (mode == kSplit && l + 1 == nL) {
                        sm100::mbar_wait(o_full, oph);
                        oph ^= 1u;
                    } else {
                        sm100::mbar_wait(my_full, dph);
                        dph ^= 1u;
                    }
                    tr(60 + l);
                    sm100::tc_fence_after();
                    const int32_t *bias = p.bias + ly.boff;
                    if (l + 1 < nL) {
                        // hidden layer epilogue: (acc + bias) >> shift -> u8 A operand of layer l+1
                        const uint32_t out = ((l + 1) & 1) ? sY : sX;
                        const int half = mode == kPair ? ly.N : ly.N / 2;
                        const int c_beg = mode == kPair ? 0 : grp * half, c_end = c_beg + half;
                        if (bfold)
                            requant_pipelined<false>(t_row, bias, ly.shift, out, row, c_beg, c_end);
                        else
                            requant_pipelined<true>(t_row, bias, ly.shift, out, row, c_beg, c_end);
                        sm100::tc_fence_before();
                        sm100::fence_proxy_async_smem();
                        tr(70 + l);
                        sm100::mbar_arrive(my_ready);
                    } else {
                        if (reader) {
                            // output layer: exact integer logits -> certified readout
                            constexpr int CV = (CM + 15) / 16 * 16;  // whole 16-column TMEM loads
                            int32_t v[CV];
#pragma unroll
                            for (int c0 = 0; c0 < CV; c0 += 16) {
                                if (c0 < p.C) {
                                    int32_t r[16];
                                    sm100::tmem_ld16(t_row + c0, r);
                                    int4 b4[4] = {};
                                    if (!bfold) {
#pragma unroll
                                        for (int q = 0; q < 4; ++q)
                                            b4[q] = __ldg(reinterpret_cast<const int4 *>(bias + c0) + q);
                                    }
                                    sm100::tmem_wait_ld();
#pragma unroll
                                    for (int q = 0; q < 4; ++q) {
                                        v[c0 + 4 * q + 0] = r[4 * q + 0] + b4[q].x;
                                        v[c0 + 4 * q + 1] = r[4 * q + 1] + b4[q].y;
                                        v[c0 + 4 * q + 2] = r[4 * q + 2] + b4[q].z;
                                        v[c0 + 4 * q + 3] = r[4 * q + 3] + b4[q].w;
                                    }
                                }
                            }
                            sm100::tc_fence_before();
                            if (mode == kSplit && (e + 1 < nE || k + 1 < nloc))
                                sm100::mbar_arrive(my_ready);  // TMEM free: next job's layer 0 may start
                            tr(81);
                            if (p.logits_out && valid) {
                                double *dst = p.logits_out + (static_cast<size_t>(st) * nE + e) * p.C;
                                for (int c = 0; c < p.C; ++c)
                                    dst[c] = static_cast<double>(v[c]) * p.scale_d[e];
                            }
                            bool fb = false;
                            const int h =
                                readout_certified<CM>(reinterpret_cast<const int32_t(&)[CM]>(v), p.C, p.scale_f[e],
                                                      p.scale_d[e], p.rk, &dist_bad, &fb);
                            if (fb && p.replays)
                                atomicAdd(p.replays, 1ull);
                            hmin = min(hmin, h);
                            tr(fb ? 83 : 82);
                            tr(80);
                        }
                        if (mode == kResident && encoder) {
                            // next job's one-hot: X is free once this job's last layer completed
                            const bool last_member = e + 1 == nE;
                            const long long kn = last_member ? k + 1 : k;
                            if (kn < nloc) {
                                const uint64_t elo = last_member ? nlo : lo, ehi = last_member ? nhi : hi;
                                encode(elo, ehi, tile_valid(kn) && !state_bad(elo, ehi), x_ready);
                            }
                        }
                    }
                }
            }
            if (reader && valid) {
                if (dist_bad)
                    raise_error(p.err, kErrDistribution);
                int h = (live && !dist_bad) ? hmin : 0;
                if (p.pdb.entries && live) {
                    if (hpdb < 0) {
                        raise_error(p.err, kErrState);
                        h = 0;
                    } else {
                        h = pdb_combine(p.pdb, h, hpdb);
                    }
                }
                p.h_out[st] = h;
            }
        }
    }

    __syncwarp();  // reconverge the single-thread roles before the aligned barrier
    sm100::tc_fence_before();
    __syncthreads();
    if (mc)
        sm100::cluster_sync();  // no multicast or remote commit may target an exited CTA
    sm100::tc_fence_after();
    if (warp == 1)
        sm100::tmem_dealloc(tmem, p.tmem_cols);
}

// ------------------------------------------------------------------ wide schedule
// kWide: hidden layers of any width up to kMaxHidden.  A tile's activations
// no longer fit in shared memory (128 x 1632 B = 204 KB for the paper's
// 13.6 MB model), so every layer l >= 1 streams its A operand from a per-CTA
// global scratch buffer (L2-resident, written by the previous layer's
// epilogue in the UMMA core-matrix layout) together with the weights.
// Output columns are produced in chunks of 256 (one N <= 256 MMA per 32-byte
// K step) into two TMEM buffers, so the epilogue drains chunk c (both groups,
// half the columns each) while the MMAs of chunk c+1 run.  A stage carries ks
// consecutive K steps, [A ks x 4 KB][B ks x chunk x 32 B], so the issuer's
// per-stage cost (barrier wait, commit) is amortised over ks MMAs.  Layer 0
// reads the one-hot tile X from shared memory, as in the other schedules.
//
// PAIR (default): CTA pairs run M = 256 MMAs (tcgen05 cta_group::2): each CTA
// holds its own tile's A rows and HALF of every weight chunk, so the weight
// bytes each SM pulls from L2 per state halve.  The even CTA issues the MMAs;
// the odd CTA's idle MMA warp relays its local "stage full" (st.async), "TMEM
// drained" and "one-hot written" events to the even CTA.
constexpr int kWideChunk = 256;
constexpr int kWideStageA = 128 * kKChunk;  // 4 KB of A per K step
constexpr int kWideMaxStages = 16;

// K steps per stage of a chunk (producer, issuer and relay agree on it).
__device__ __forceinline__ int wide_ks(int l, int cw, int ns, int nk, int stage_bytes) {
    const int kb = (l > 0 ? kWideStageA : 0) + cw / ns * kKChunk;
    return max(1, min(nk, stage_bytes / kb));
}

template <int DOMAIN, int CM, bool PAIR>
__global__ void __launch_bounds__(kMlpThreads, 1) mlp_wide_kernel(const __grid_constant__ MlpParams p) {
    using T = DomainTraits<DOMAIN>;
    constexpr int NS = PAIR ? 2 : 1;  // CTAs sharing one weight chunk
    extern __shared__ __align__(1024) uint8_t smem[];
    const int stage_bytes = p.stage_bytes;
    uint8_t *stages = smem + p.xbytes;
    uint8_t *bias_sm = stages + p.stages * stage_bytes;  // [bias_bytes] optional
    uint64_t *bars = reinterpret_cast<uint64_t *>(bias_sm + p.bias_bytes);
    uint64_t *full = bars;                          // [kWideMaxStages] local TMA landed
    uint64_t *empty = bars + kWideMaxStages;        // [kWideMaxStages] pair's MMAs done with the stage
    uint64_t *full2 = bars + 2 * kWideMaxStages;    // [kWideMaxStages] PAIR, even CTA: peer's stage landed
    uint64_t *x_ready = bars + 3 * kWideMaxStages;  // one-hot of the tile written (group 1)
    uint64_t *d_full = x_ready + 1;                 // [2] TMEM buffer's chunk complete (commit)
    uint64_t *tmem_free = d_full + 2;               // [2] TMEM buffer drained (256 epilogue threads)
    uint64_t *act_done = tmem_free + 2;             // hidden layer written to scratch (256)
    uint64_t *x_ready2 = act_done + 1;              // PAIR, even CTA: peer's one-hot written
    uint64_t *tmem_free2 = x_ready2 + 1;            // [2] PAIR, even CTA: peer's buffer drained
    uint64_t *b_ready = tmem_free2 + 2;             // bias staged
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(b_ready + 1);
    uint32_t *sink = tmem_slot + 1;                 // PAIR, even CTA: target of the peer's st.async signals

    const int warp = threadIdx.x >> 5;
    const uint32_t rank = PAIR ? sm100::cluster_rank() : 0u;
    const long long ntiles = (p.n + kTileM - 1) / kTileM;
    // tile of local iteration kk: CTA pairs take consecutive tile pairs, so both
    // CTAs of a pair run the same iterations (the odd CTA's may be empty)
    const long long unit = PAIR ? (blockIdx.x >> 1) : blockIdx.x, nunits = PAIR ? (gridDim.x >> 1) : gridDim.x;
    const long long nu = PAIR ? (ntiles + 1) / 2 : ntiles;
    const long long nloc = unit < nu ? (nu - unit + nunits - 1) / nunits : 0;
    auto tile_of = [&](long long kk) { return PAIR ? 2 * (unit + kk * nunits) + rank : unit + kk * nunits; };
    uint8_t *scr = p.scratch + static_cast<long long>(blockIdx.x) * 2 * p.sbytes;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kWideMaxStages; ++s) {
            sm100::mbar_init(&full[s], 1);
            sm100::mbar_init(&empty[s], 1);
            sm100::mbar_init(&full2[s], 1);
        }
        sm100::mbar_init(x_ready, 128);
        for (int b = 0; b < 2; ++b) {
            sm100::mbar_init(&d_full[b], 1);
            sm100::mbar_init(&tmem_free[b], 256);
            sm100::mbar_init(&tmem_free2[b], 1);
        }
        sm100::mbar_init(act_done, 256);
        sm100::mbar_init(x_ready2, 1);
        sm100::mbar_init(b_ready, 1);
        sm100::fence_barrier_init();
    }
    if (warp == 1) {
        if constexpr (PAIR)
            sm100::tmem_alloc_pair(tmem_slot, 512);
        else
            sm100::tmem_alloc(tmem_slot, 512);
    }
    sm100::tc_fence_before();
    __syncthreads();
    if constexpr (PAIR)
        sm100::cluster_sync();  // peer barriers initialised before any remote arrive / multicast commit
    sm100::tc_fence_after();
    const uint64_t l2pol = p.l2hint ? sm100::l2_policy_evict_last() : 0ull;
    const uint32_t tmem = *tmem_slot;
    Tracer tr;
    if (Tracer::kOn && p.trace && blockIdx.x == 0 && lane_id() == 0)
        tr.buf = p.trace + static_cast<long long>(warp) * kTraceSlots;

    if (warp == 0) {
        // ------------------------------------------------ producer: [A ks x 4 KB][B ks x chunk part] stages
        if (lane_id() == 0 && nloc > 0) {
            if (p.bias_bytes) {
                sm100::mbar_arrive_expect_tx(b_ready, static_cast<uint32_t>(p.bias_bytes));
                sm100::bulk_g2s(bias_sm, p.bias, static_cast<uint32_t>(p.bias_bytes), b_ready);
            }
            int s = 0;
            uint32_t ph = 0, adph = 0;
            for (long long k = 0; k < nloc; ++k)
                for (int e = 0; e < p.E; ++e)
                    for (int l = 0; l < p.nl; ++l) {
                        const MlpLayer &ly = p.layer[e][l];
                        const int nk = ly.K / kKChunk;
                        const uint8_t *a_src = scr + ((l - 1) & 1) * p.sbytes;
                        if (l > 0) {  // the previous layer's activations are in scratch
                            sm100::mbar_wait(act_done, adph);
                            adph ^= 1u;
                        }
                        for (int c0 = 0; c0 < ly.N; c0 += kWideChunk) {
                            const int cw = min(kWideChunk, ly.N - c0);
                            const int bb = cw / NS * kKChunk;  // this CTA's B bytes per K step
                            const int ks = wide_ks(l, cw, NS, nk, stage_bytes);
                            const uint8_t *b_src =
                                p.wimg + ly.woff + static_cast<long long>(c0) * ly.K + static_cast<long long>(rank) * bb / kKChunk * ly.K;
                            for (int kc = 0; kc < nk; kc += ks) {
                                const int kn = min(ks, nk - kc);
                                sm100::mbar_wait(&empty[s], ph ^ 1u);
                                uint8_t *st = stages + s * stage_bytes;
                                const int abytes = l > 0 ? kn * kWideStageA : 0;
                                sm100::mbar_arrive_expect_tx(&full[s], abytes + kn * bb);
                                if (PAIR && rank == 0)  // the peer relay's st.async signal for this stage
                                    sm100::mbar_arrive_expect_tx(&full2[s], 4u);
                                if (p.l2hint) {  // scratch + weights: keep in L2 (evict_last)
                                    if (l > 0)
                                        sm100::bulk_g2s_hint(st, a_src + kc * kWideStageA, abytes, &full[s], l2pol);
                                    sm100::bulk_g2s_hint(st + (l > 0 ? ks * kWideStageA : 0),
                                                         b_src + static_cast<long long>(kc) * bb, kn * bb, &full[s], l2pol);
                                } else {
                                    if (l > 0)
                                        sm100::bulk_g2s(st, a_src + kc * kWideStageA, abytes, &full[s]);
                                    sm100::bulk_g2s(st + (l > 0 ? ks * kWideStageA : 0),
                                                    b_src + static_cast<long long>(kc) * bb, kn * bb, &full[s]);
                                }
                                if (++s == p.stages) {
                                    s = 0;
                                    ph ^= 1u;
                                }
                            }
                        }
                    }
        }
    } else if (warp == 1 && rank == 1) {
        // ------------------------------------------------ PAIR odd CTA: relay local events to the even CTA,
        // in the order its MMA issuer consumes them
        if (lane_id() == 0 && nloc > 0) {
            const uint32_t r_full2 = sm100::mapa_shared(full2, 0), r_x2 = sm100::mapa_shared(x_ready2, 0),
                           r_tf2 = sm100::mapa_shared(tmem_free2, 0), r_sink = sm100::mapa_shared(sink, 0);
            int s = 0;
            uint32_t ph = 0, xph = 0, cidx = 0;
            for (long long k = 0; k < nloc; ++k)
                for (int e = 0; e < p.E; ++e)
                    for (int l = 0; l < p.nl; ++l) {
                        const MlpLayer &ly = p.layer[e][l];
                        const int nk = ly.K / kKChunk;
                        if (l == 0 && e == 0) {
                            sm100::mbar_wait(x_ready, xph);
                            xph ^= 1u;
                            sm100::mbar_arrive_cluster_relaxed(r_x2);
                        }
                        for (int c0 = 0; c0 < ly.N; c0 += kWideChunk, ++cidx) {
                            const int cw = min(kWideChunk, ly.N - c0);
                            const int ks = wide_ks(l, cw, NS, nk, stage_bytes);
                            for (int kc = 0; kc < nk; kc += ks) {
                                sm100::mbar_wait(&full[s], ph);
                                sm100::st_async_signal(r_sink, 1u, r_full2 + s * 8u);  // no round-trip wait
                                if (++s == p.stages) {
                                    s = 0;
                                    ph ^= 1u;
                                }
                            }
                            const uint32_t b = cidx & 1u;
                            sm100::mbar_wait(&tmem_free[b], (cidx >> 1) & 1u);  // this chunk drained here
                            sm100::mbar_arrive_cluster_relaxed(r_tf2 + b * 8u);
                        }
                    }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (even CTA of a pair)
        if (nloc > 0) {
            int s = 0;
            uint32_t ph = 0, xph = 0, cidx = 0;
            const uint32_t sX = sm100::smem_u32(smem), sS = sm100::smem_u32(stages);
            const uint64_t sdelta = static_cast<uint64_t>(stage_bytes) >> 4;
            uint64_t soff = 0;  // descriptor offset of stage s
            for (long long k = 0; k < nloc; ++k)
                for (int e = 0; e < p.E; ++e)
                    for (int l = 0; l < p.nl; ++l) {
                        const MlpLayer ly = p.layer[e][l];
                        const int nk = ly.K / kKChunk;
                        if (l == 0 && e == 0) {
                            if (lane_id() == 0)
                                tr(10);
                            sm100::mbar_wait(x_ready, xph);
                            if constexpr (PAIR)
                                sm100::mbar_wait(x_ready2, xph);
                            xph ^= 1u;
                        }
                        for (int c0 = 0; c0 < ly.N; c0 += kWideChunk, ++cidx) {
                            const int cw = min(kWideChunk, ly.N - c0);
                            const int ks = wide_ks(l, cw, NS, nk, stage_bytes);
                            const uint32_t b = cidx & 1u, idesc = sm100::make_idesc_i8(cw, 128u * NS);
                            const uint32_t dcol = tmem + b * 256u;
                            sm100::mbar_wait(&tmem_free[b], ((cidx >> 1) & 1u) ^ 1u);  // chunk cidx-2 drained
                            if constexpr (PAIR)
                                sm100::mbar_wait(&tmem_free2[b], ((cidx >> 1) & 1u) ^ 1u);
                            if (lane_id() == 0)
                                tr(20 + l);
                            sm100::tc_fence_after();
                            // descriptors advanced by adds (no per-step address math on the issue path)
                            const uint32_t bb = cw / NS * kKChunk;
                            const uint64_t a0 = sm100::make_smem_desc(sS, 2048u, 128u);
                            const uint64_t b0 = sm100::make_smem_desc(sS + (l > 0 ? ks * kWideStageA : 0), bb >> 1, 128u);
                            uint64_t xd = sm100::make_smem_desc(sX, 2048u, 128u);
                            long long wsum = 0;  // debug timeline: cycles spent waiting for stages
                            for (int kc = 0; kc < nk; kc += ks) {
                                const int kn = min(ks, nk - kc);
                                const long long tw0 = tr.on() ? clock64() : 0;
                                sm100::mbar_wait(&full[s], ph);
                                if constexpr (PAIR)
                                    sm100::mbar_wait(&full2[s], ph);
                                if (tr.on())
                                    wsum += clock64() - tw0;
                                sm100::tc_fence_after();
                                uint64_t ad = l == 0 ? xd : a0 + soff, bd = b0 + soff;
                                if (sm100::elect_one()) {
                                    for (int j = 0; j < kn; ++j) {
                                        const uint32_t acc = (kc + j) > 0 ? 1u : 0u;
                                        if constexpr (PAIR)
                                            sm100::mma_i8_pair(dcol, ad, bd, idesc, acc);
                                        else
                                            sm100::mma_i8(dcol, ad, bd, idesc, acc);
                                        ad += kWideStageA >> 4;
                                        bd += bb >> 4;
                                    }
                                    if constexpr (PAIR)
                                        sm100::mma_commit_pair(&empty[s]);
                                    else
                                        sm100::mma_commit(&empty[s]);
                                }
                                __syncwarp();
                                xd += static_cast<uint64_t>(kn) * (kWideStageA >> 4);
                                soff += sdelta;
                                if (++s == p.stages) {
                                    s = 0;
                                    soff = 0;
                                    ph ^= 1u;
                                }
                            }
                            if (sm100::elect_one()) {
                                if constexpr (PAIR)
                                    sm100::mma_commit_pair(&d_full[b]);
                                else
                                    sm100::mma_commit(&d_full[b]);
                            }
                            __syncwarp();
                            if (lane_id() == 0) {
                                tr(30 + l);
                                tr.value(wsum, 90);
                            }
                        }
                    }
        }
    } else {
        // ------------------------------------------------ encode / epilogue / readout
        const int grp = (warp - 2) >> 2;  // drains half grp of every chunk's columns
        const int quad = warp & 3;
        const int row = quad * 32 + lane_id();
        const uint32_t sX = sm100::smem_u32(smem);
        const uint32_t t_row0 = tmem + (static_cast<uint32_t>(quad * 32) << 16);
        uint32_t cidx = 0;
        const bool reader = grp == 0, encoder = grp == 1;

        auto state_of = [&](long long kk) { return tile_of(kk) * kTileM + row; };
        auto load_state = [&](long long kk, uint64_t &lo_, uint64_t &hi_) {
            lo_ = hi_ = 0;
            const long long s_ = state_of(kk);
            if (kk < nloc && s_ < p.n) {
                if constexpr (T::PB == 16) {
                    const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2 *>(p.packed) + s_);
                    lo_ = v.x;
                    hi_ = v.y;
                } else {
                    lo_ = __ldcs(reinterpret_cast<const unsigned long long *>(p.packed) + s_);
                }
            }
        };
        auto state_bad = [&](uint64_t lo_, uint64_t hi_) { return state_out_of_range<DOMAIN>(lo_, hi_); };
        auto tile_valid = [&](long long kk) { return kk < nloc && state_of(kk) < p.n; };
        constexpr int kX16 = (T::F + 31) / 32 * 2;  // 16-column chunks of the one-hot tile (Fpad / 16)
        auto encode = [&](uint64_t lo_, uint64_t hi_, bool live_) {
            tr(40);
#pragma unroll
            for (int c16 = 0; c16 < kX16; ++c16)
                sm100::st_shared_v4(sX + c16 * 2048u + row * 16u, 0u, 0u, 0u, 0u);
            if (live_) {
#pragma unroll
                for (int q = 0; q < T::NNZ; ++q) {
                    const int j = position_feature<DOMAIN>(lo_, hi_, q);
                    sm100::st_shared_u8(sX + (j >> 4) * 2048u + row * 16u + (j & 15), 1u);
                }
            }
            sm100::fence_proxy_async_smem();
            tr(41);
            sm100::mbar_arrive(x_ready);
        };

        uint64_t nlo = 0, nhi = 0;
        load_state(0, nlo, nhi);
        if (encoder && nloc > 0)
            encode(nlo, nhi, tile_valid(0) && !state_bad(nlo, nhi));
        const uint32_t bias_s = p.bias_bytes ? sm100::smem_u32(bias_sm) : 0u;
        if (p.bias_bytes && nloc > 0)
            sm100::mbar_wait(b_ready, 0);
        for (long long k = 0; k < nloc; ++k) {
            const long long st = state_of(k);
            const bool valid = st < p.n;
            const uint64_t lo = nlo, hi = nhi;
            load_state(k + 1, nlo, nhi);
            const bool bad = valid && state_bad(lo, hi);
            const int hpdb = (p.pdb.entries && reader && valid) ? pdb_fetch<DOMAIN>(p.pdb, lo) : 0;
            if (bad && reader)
                raise_error(p.err, kErrState);
            const bool live = valid && !bad;
            int hmin = 0x7fffffff;
            bool dist_bad = false;
            for (int e = 0; e < p.E; ++e) {
                for (int l = 0; l < p.nl; ++l) {
                    const MlpLayer &ly = p.layer[e][l];
                    const int32_t *bias = p.bias + ly.boff;
                    const bool hidden = l + 1 < p.nl;
                    uint8_t *out = scr + (l & 1) * p.sbytes;
                    for (int c0 = 0; c0 < ly.N; c0 += kWideChunk, ++cidx) {
                        const int cw = min(kWideChunk, ly.N - c0);
                        const uint32_t b = cidx & 1u;
                        const uint32_t t_row = t_row0 + b * 256u;
                        tr(50 + l);
                        sm100::mbar_wait(&d_full[b], (cidx >> 1) & 1u);
                        tr(60 + l);
                        sm100::tc_fence_after();
                        if (hidden) {
                            const int half = cw >> 1;  // multiple of 16: widths are padded to 32
                            requant_block<true>(t_row, grp * half, bias, c0 + grp * half, half, ly.shift, 0u, out, row,
                                                bias_s ? bias_s + ly.boff * 4u : 0u, l2pol);
                            sm100::tc_fence_before();
                            sm100::mbar_arrive(&tmem_free[b]);
                            tr(70 + l);
                            continue;
                        }
                        // output layer (one chunk: C <= 256)
                        if (!reader) {
                            sm100::tc_fence_before();
                            sm100::mbar_arrive(&tmem_free[b]);
                            continue;
                        }
                        int32_t v[CM];
#pragma unroll
                        for (int q0 = 0; q0 < CM; q0 += 16) {
                            if (q0 < p.C) {
                                int32_t r[16];
                                sm100::tmem_ld16(t_row + q0, r);
                                int4 b4[4];
#pragma unroll
                                for (int q = 0; q < 4; ++q)
                                    b4[q] = __ldg(reinterpret_cast<const int4 *>(bias + q0) + q);
                                sm100::tmem_wait_ld();
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    v[q0 + 4 * q + 0] = r[4 * q + 0] + b4[q].x;
                                    v[q0 + 4 * q + 1] = r[4 * q + 1] + b4[q].y;
                                    v[q0 + 4 * q + 2] = r[4 * q + 2] + b4[q].z;
                                    v[q0 + 4 * q + 3] = r[4 * q + 3] + b4[q].w;
                                }
                            }
                        }
                        sm100::tc_fence_before();
                        sm100::mbar_arrive(&tmem_free[b]);
                        if (p.logits_out && valid) {
                            double *dst = p.logits_out + (static_cast<size_t>(st) * p.E + e) * p.C;
                            for (int c = 0; c < p.C; ++c)
                                dst[c] = static_cast<double>(v[c]) * p.scale_d[e];
                        }
                        bool fb = false;
                        const int h = readout_certified<CM>(v, p.C, p.scale_f[e], p.scale_d[e], p.rk, &dist_bad, &fb);
                        if (fb && p.replays)
                            atomicAdd(p.replays, 1ull);
                        hmin = min(hmin, h);
                        tr(80);
                    }
                    if (hidden) {
                        sm100::fence_proxy_async_global();  // scratch writes -> the producer's bulk reads
                        sm100::mbar_arrive(act_done);
                    }
                    if (l == 0 && e + 1 == p.E && encoder && k + 1 < nloc)
                        encode(nlo, nhi, tile_valid(k + 1) && !state_bad(nlo, nhi));  // X free: layer 0 done
                }
            }
            if (reader && valid) {
                if (dist_bad)
                    raise_error(p.err, kErrDistribution);
                int h = (live && !dist_bad) ? hmin : 0;
                if (p.pdb.entries && live) {
                    if (hpdb < 0) {
                        raise_error(p.err, kErrState);
                        h = 0;
                    } else {
                        h = pdb_combine(p.pdb, h, hpdb);
                    }
                }
                p.h_out[st] = h;
            }
        }
    }

    __syncwarp();
    sm100::tc_fence_before();
    __syncthreads();
    if constexpr (PAIR)
        sm100::cluster_sync();  // no remote arrive or multicast commit may target an exited CTA
    sm100::tc_fence_after();
    if (warp == 1) {
        if constexpr (PAIR)
            sm100::tmem_dealloc_pair(tmem, 512);
        else
            sm100::tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ host

namespace {

int fail(std::string *err, int code, const std::string &msg) {
    *err = msg;
    return code;
}

uint32_t rd32(const unsigned char *b) {
    return uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 | uint32_t(b[3]) << 24;
}

template <int DOMAIN, int CM>
int launch_t(MlpModel *m, const MlpParams &p, cudaStream_t st) {
    auto kern = [&] {
        if constexpr (CM == 24)  // fused schedules only (mlp_create)
            return p.mode == kResident ? (p.bias_fold && p.E == 1 ? (p.nl == 3 ? mlp_fused_kernel<DOMAIN, 24, 3> : mlp_fused_kernel<DOMAIN, 24, 2>)
                                                                   : mlp_fused_kernel<DOMAIN, 24, 1>)
                                       : mlp_fused_kernel<DOMAIN, 24>;
        else if constexpr (CM <= 64)
            return p.mode == kResident ? (p.bias_fold && p.E == 1 ? (p.nl == 3 ? mlp_fused_kernel<DOMAIN, CM, 3> : mlp_fused_kernel<DOMAIN, CM, 2>)
                                                                   : mlp_fused_kernel<DOMAIN, CM, 1>)
                   : p.mode != kWide   ? mlp_fused_kernel<DOMAIN, CM>
                   : (p.cluster == 2 ? mlp_wide_kernel<DOMAIN, CM, true> : mlp_wide_kernel<DOMAIN, CM, false>);
        else
            return p.mode != kWide ? mlp_fused_kernel<DOMAIN, CM>
                                   : (p.cluster == 2 ? mlp_wide_kernel<DOMAIN, CM, true> : mlp_wide_kernel<DOMAIN, CM, false>);
    }();
    const int threads = kMlpThreads;
    std::call_once(m->attr_once, [&] {
        m->attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(m->smem));
    });
    cudaError_t e = m->attr_err;
    if (e != cudaSuccess) {
        g_err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e);
        return 1;
    }
    const long long ntiles = (p.n + kTileM - 1) / kTileM;
    int grid = static_cast<int>(std::max<long long>(1, std::min<long long>(ntiles, m->grid_cap)));
    if (p.cluster == 2)
        grid = (grid + 1) & ~1;
    MlpParams q = p;
    std::unique_lock<std::mutex> slk;
    int sslot = -1;
    if (p.mode == kWide) {
        sslot = static_cast<int>(m->scratch_next.fetch_add(1, std::memory_order_relaxed) % kScratchPool);
        slk = std::unique_lock<std::mutex>(m->scratch_mu[sslot]);
        q.scratch = m->scratch[sslot];
        e = cudaStreamWaitEvent(st, m->scratch_ev[sslot], 0);
        if (e != cudaSuccess) {
            g_err = std::string("mlp scratch: ") + cudaGetErrorString(e);
            return 1;
        }
    }
    if (p.cluster == 2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kMlpThreads);
        cfg.dynamicSmemBytes = m->smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kern, q);
    } else {
        kern<<<grid, threads, m->smem, st>>>(q);
    }
    if (e == cudaSuccess)
        e = cudaGetLastError();
    if (sslot >= 0) {
        const cudaError_t fe = cudaEventRecord(m->scratch_ev[sslot], st);
        if (e == cudaSuccess)
            e = fe;
    }
    if (e != cudaSuccess) {
        g_err = std::string("mlp launch: ") + cudaGetErrorString(e);
        return 1;
    }
    return 0;
}

template <int DOMAIN>
int launch_d(MlpModel *m, const MlpParams &p, cudaStream_t st) {
    switch (m->cm) {
    case 24: return launch_t<DOMAIN, 24>(m, p, st);
    case 32: return launch_t<DOMAIN, 32>(m, p, st);
    case 64: return launch_t<DOMAIN, 64>(m, p, st);
    default: return launch_t<DOMAIN, 256>(m, p, st);
    }
}

} // namespace

int mlp_create(const unsigned char *b, size_t len, int F, double thr, int num_sms, MlpModel **out,
               MlpShape *shape, std::string *err) {
    *out = nullptr;
    if (!b || len < 21 || std::memcmp(b, "BMLP1", 5) != 0)
        return fail(err, 2, "not a BMLP1 file");
    const uint32_t fF = rd32(b + 5), C = rd32(b + 9), E = rd32(b + 13), L = rd32(b + 17);
    if (fF != static_cast<uint32_t>(F))
        return fail(err, 2, "BMLP1 header does not match domain");
    if (E == 0 || E > kMaxMembers)
        return fail(err, 1, "BMLP1: ensemble size must be 1..8");
    if (C == 0 || C > 256)
        return fail(err, 1, "BMLP1: classes must be 1..256");
    if (L == 0 || L > kMaxLayers - 1)
        return fail(err, 1, "BMLP1: hidden layers must be 1..4");
    size_t off = 21;
    if (len < off + 4 * L)
        return fail(err, 2, "truncated BMLP1 file");
    std::vector<int> H(L);
    for (uint32_t l = 0; l < L; ++l) {
        H[l] = static_cast<int>(rd32(b + off));
        off += 4;
        if (H[l] < 1 || H[l] > kMaxHidden)
            return fail(err, 1, "BMLP1: hidden widths must be in [1, 4096]");
    }
    const int Fpad = (F + 31) / 32 * 32;
    std::vector<int> Hp(L);  // widths padded to the 32-byte MMA K step (zero weights and bias)
    for (uint32_t l = 0; l < L; ++l)
        Hp[l] = (H[l] + 31) / 32 * 32;
    const int Cpad = (static_cast<int>(C) + 31) / 32 * 32;  // N of the output MMA: a multiple of 32 (CTA pairs)
    const int nl = static_cast<int>(L) + 1;
    auto *m = new MlpModel();
    MlpParams &p = m->p;
    std::memset(&p, 0, sizeof(p));
    p.E = static_cast<int>(E);
    p.nl = nl;
    p.C = static_cast<int>(C);
    p.Fpad = Fpad;
    int KX = Fpad, KY = 0, Nmax = Cpad;  // KX: even-layer inputs, KY: odd-layer inputs
    for (uint32_t l = 0; l < L; ++l) {
        Nmax = std::max(Nmax, Hp[l]);
        if ((l + 1) % 2 == 0)
            KX = std::max(KX, Hp[l]);
        else
            KY = std::max(KY, Hp[l]);
    }
    std::vector<uint8_t> img;
    std::vector<int32_t> bias;
    struct WSrc {
        const int8_t *W;
        int in, outn;
    };
    std::vector<WSrc> wsrc;  // [e][l]
    size_t wtotal = 0;
    for (uint32_t e = 0; e < E; ++e) {
        for (int l = 0; l < nl; ++l) {
            const int in = l ? H[l - 1] : F;
            const int outn = l < static_cast<int>(L) ? H[l] : static_cast<int>(C);
            const int K = l ? Hp[l - 1] : Fpad;
            const int N = l < static_cast<int>(L) ? Hp[l] : Cpad;
            const size_t nw = static_cast<size_t>(in) * outn;
            if (len < off + nw + 4ull * outn) {
                delete m;
                return fail(err, 2, "truncated BMLP1 file");
            }
            const int8_t *W = reinterpret_cast<const int8_t *>(b + off);
            off += nw;
            MlpLayer &ly = p.layer[e][l];
            ly.K = K;
            ly.N = N;
            wtotal += static_cast<size_t>(N) * K;
            ly.boff = static_cast<int>(bias.size());
            wsrc.push_back({W, in, outn});  // image written once the schedule is known
            for (int n = 0; n < N; ++n) {
                int32_t v = 0;
                if (n < outn)
                    std::memcpy(&v, b + off + 4 * n, 4);
                bias.push_back(v);
            }
            off += 4ull * outn;
            if (l < static_cast<int>(L)) {
                if (len < off + 4) {
                    delete m;
                    return fail(err, 2, "truncated BMLP1 file");
                }
                const uint32_t s = rd32(b + off);
                off += 4;
                if (s > 31) {
                    delete m;
                    return fail(err, 1, "BMLP1: shift must be <= 31");
                }
                ly.shift = static_cast<int>(s);
            }
        }
        if (len < off + 4) {
            delete m;
            return fail(err, 2, "truncated BMLP1 file");
        }
        float sc;
        std::memcpy(&sc, b + off, 4);
        off += 4;
        if (!std::isfinite(sc)) {
            delete m;
            return fail(err, 1, "BMLP1: out_scale must be finite");
        }
        p.scale_f[e] = sc;
        p.scale_d[e] = static_cast<double>(sc);
    }
    // readout constants (certified_readout.cuh)
    p.rk.thr = thr;
    const double u = 1.0 - thr;
    const double eps64 = (4.0 * C + 16.0) * std::ldexp(1.0, -53);
    p.rk.uLo = std::nextafter(static_cast<float>(u - eps64), 0.0f);
    p.rk.uHi = std::nextafter(static_cast<float>(u + eps64), INFINITY);
    p.xbytes = kTileM * KX;
    p.ybytes = kTileM * KY;
    p.wbytes = static_cast<int>(wtotal);
    p.wbytes_pad = (p.wbytes + 1023) & ~1023;
    const size_t bar_bytes = 8 * (2 * kMaxStages + 6) + 16;
    const size_t budget = 227 * 1024;
    const size_t set1 = static_cast<size_t>(p.xbytes) + p.ybytes;
    auto stages_for = [&](size_t act) -> int {
        if (act + bar_bytes + 2 * kStageBytes > budget)
            return 0;
        return static_cast<int>(std::min<size_t>(kMaxStages, (budget - act - bar_bytes) / kStageBytes));
    };
    auto pow2cols = [](int n) {
        uint32_t c = 32;
        while (c < static_cast<uint32_t>(n))
            c <<= 1;
        return c;
    };
    // 0) a layer wider than 256 (or nothing else fits): wide (activations in
    //    L2-resident global scratch, A and B streamed; h512 1.27 vs 1.17 G/s split)
    // 1) every layer <= 256 wide and the whole weight image fits next to one
    //    activation set: resident
    // 2) every layer <= 256 wide and two activation sets fit: pair (streamed)
    // 3) every layer <= 512 wide: split (streamed; BIDA_MLP_FORCE_MODE=split)
    // BIDA_MLP_FORCE_MODE=wide|resident|pair|split (tests): use that schedule
    // when it fits.
    const char *force = std::getenv("BIDA_MLP_FORCE_MODE");
    const std::string fm = force ? force : "";
    int Kmax = Fpad;
    for (uint32_t l = 0; l < L; ++l)
        Kmax = std::max(Kmax, Hp[l]);
    const bool fit_res = Nmax <= 256 && set1 + p.wbytes_pad + bar_bytes <= budget;
    // Resident models whose biases fit |b| <= kFoldMax fold them into the
    // accumulators: one extra K step per layer multiplies a constant A block
    // (column 0 = 1, columns 1..31 = 255) by the bias written as s8 digits, so
    // the epilogues skip the per-column bias loads and adds
    // (BIDA_MLP_BIAS_FOLD=0 disables).  Integer sums: the result is identical.
    constexpr long long kFoldMax = 127 + 255LL * 31 * 127;
    size_t fold_bytes = kTileM * kKChunk;  // the constant A block
    bool fold_ok = true;
    for (int32_t v : bias)
        fold_ok = fold_ok && std::llabs(static_cast<long long>(v)) <= kFoldMax;
    for (uint32_t e = 0; e < E; ++e)
        for (int l = 0; l < nl; ++l)
            fold_bytes += static_cast<size_t>(p.layer[e][l].N) * kKChunk;
    const int fold_pad = static_cast<int>((wtotal + fold_bytes + 1023) & ~static_cast<size_t>(1023));
    const char *fv = std::getenv("BIDA_MLP_BIAS_FOLD");
    fold_ok = fold_ok && !(fv && fv[0] == '0') && Nmax <= 256 && set1 + fold_pad + bar_bytes <= budget;
    const bool fit_pair = Nmax <= 256 && stages_for(2 * set1) >= 2;
    const bool want_split = fm == "split" && stages_for(set1) >= 2;
    const bool fit_split = Nmax <= 512 && stages_for(set1) >= 2;
    // wide: CTA pairs (M = 256 MMAs, half of every weight chunk per CTA) only with
    // BIDA_MLP_WIDE_PAIR=1: measured slower than one CTA per tile (profiles/r1_notes.md)
    const char *wpv = std::getenv("BIDA_MLP_WIDE_PAIR");
    const bool wide_pair = wpv && wpv[0] == '1';
    // a stage holds 3 K steps of a full chunk: [A 3 x 4 KB][B 3 x 256 x 32 B (/2 per CTA of a pair)]
    const int wide_stage = 3 * (kWideStageA + kWideChunk * kKChunk / (wide_pair ? 2 : 1));
    const size_t wide_bars = 8 * (3 * kWideMaxStages + 10) + 16;
    const size_t xwide = static_cast<size_t>(kTileM) * Fpad;
    const size_t wide_bias = bias.size() * 4;  // staged in shared memory when 4 stages still fit
    const size_t wide_bias_sm = xwide + wide_bars + wide_bias + 4 * static_cast<size_t>(wide_stage) <= budget ? wide_bias : 0;
    const int wide_stages =
        xwide + wide_bars + wide_bias_sm + 2 * wide_stage > budget
            ? 0
            : static_cast<int>(std::min<size_t>(kWideMaxStages, (budget - xwide - wide_bars - wide_bias_sm) / wide_stage));
    if (wide_stages >= 2 && (fm == "wide" || (Nmax > 256 && fm != "split") || (!fit_res && !fit_pair && !fit_split))) {
        p.mode = kWide;
        p.stages = wide_stages;
        p.xbytes = static_cast<int>(xwide);
        p.ybytes = 0;
        p.tmem_cols = 512u;
        p.sbytes = static_cast<long long>(kTileM) * Kmax;
        p.stage_bytes = wide_stage;
        p.bias_bytes = static_cast<int>(wide_bias_sm);
        p.cluster = wide_pair ? 2 : 1;
        // evict_last L2 policy on the activation scratch and stage copies
        // (BIDA_MLP_L2HINT=0 disables; profiles/r2_notes.md)
        const char *hv = std::getenv("BIDA_MLP_L2HINT");
        p.l2hint = !(hv && hv[0] == '0');
        m->smem = xwide + static_cast<size_t>(wide_stages) * wide_stage + wide_bias_sm + wide_bars;
    } else if (!want_split && fit_res && (fm.empty() || fm == "resident" || (fm == "pair" && !fit_pair))) {  // (TMEM double-buffered by job)
        p.mode = kResident;
        p.stages = 0;
        p.tmem_cols = 512u;
        if (fold_ok) {
            p.bias_fold = 1;
            p.wbytes = static_cast<int>(wtotal + fold_bytes);
            p.wbytes_pad = fold_pad;
            p.cA_off = static_cast<int>(wtotal + fold_bytes - kTileM * kKChunk);
        }
        m->smem = set1 + p.wbytes_pad + bar_bytes;
    } else if (!want_split && fit_pair) {
        p.mode = kPair;
        p.stages = stages_for(2 * set1);
        p.tmem_cols = 512;
        m->smem = 2 * set1 + static_cast<size_t>(p.stages) * kStageBytes + bar_bytes;
    } else if (fit_split) {
        p.mode = kSplit;
        p.stages = stages_for(set1);
        p.tmem_cols = pow2cols(Nmax);
        m->smem = set1 + static_cast<size_t>(p.stages) * kStageBytes + bar_bytes;
    } else {
        delete m;
        return fail(err, 1, "BMLP1: model too wide for shared memory");
    }
    // Weight image, per layer in MMA consumption order: nh N-halves (2 for the
    // split schedule's hidden layers, else 1), each K/32 chunks of
    // [2 K-halves][N/nh/8 row groups][8 rows][16 bytes] (UMMA K-major, no swizzle).
    img.assign(p.bias_fold ? static_cast<size_t>(p.wbytes) : wtotal, 0);
    {
        size_t pos0 = 0;
        for (int e = 0; e < static_cast<int>(E); ++e)
            for (int l = 0; l < nl; ++l) {
                MlpLayer &ly = p.layer[e][l];
                const WSrc &w = wsrc[static_cast<size_t>(e) * nl + l];
                if (p.mode == kWide) {
                    // chunks of <= 512 output columns, each K/32 steps of
                    // [half 0: w0 rows x 32 B][half 1: w1 rows x 32 B] (core-matrix layout)
                    ly.nh = 1;
                    ly.cps = 1;
                    ly.woff = static_cast<long long>(pos0);
                    // chunks of <= 256 output columns; a chunk is NS parts (CTA r of a pair
                    // holds rows [r*cw/2, (r+1)*cw/2)), each K/32 consecutive steps of
                    // rows x 32 B in the core-matrix layout (a stage loads ks steps at once)
                    const int ns = p.cluster == 2 ? 2 : 1;
                    for (int c0 = 0; c0 < ly.N; c0 += kWideChunk) {
                        const int cw = std::min(kWideChunk, ly.N - c0), rows = cw / ns;
                        for (int nn = 0; nn < cw; ++nn) {
                            const int n = c0 + nn;
                            if (n >= w.outn)
                                continue;
                            const int part = nn / rows, r = nn % rows;
                            for (int kk = 0; kk < w.in; ++kk) {
                                const int kc = kk / 32, k = kk % 32;
                                const size_t pos = pos0 + static_cast<size_t>(c0) * ly.K + static_cast<size_t>(part) * rows * ly.K +
                                                   static_cast<size_t>(kc) * rows * 32 + (k / 16) * (rows * 16) + (r / 8) * 128 +
                                                   (r % 8) * 16 + (k % 16);
                                img[pos] = static_cast<uint8_t>(w.W[static_cast<size_t>(n) * w.in + kk]);
                            }
                        }
                    }
                    pos0 += static_cast<size_t>(ly.N) * ly.K;
                    continue;
                }
                ly.nh = (p.mode == kSplit && l + 1 < nl) ? 2 : 1;
                const int Nh = ly.N / ly.nh;
                ly.cps = std::max(1, kStageBytes / (Nh * kKChunk));
                ly.woff = static_cast<long long>(pos0);
                for (int h = 0; h < ly.nh; ++h)
                    for (int kc = 0; kc < ly.K / 32; ++kc)
                        for (int nn = 0; nn < Nh; ++nn) {
                            const int n = h * Nh + nn;
                            if (n >= w.outn)
                                continue;
                            for (int k = 0; k < 32; ++k) {
                                const int kk = kc * 32 + k;
                                if (kk >= w.in)
                                    continue;
                                const size_t pos = pos0 + (static_cast<size_t>(h) * (ly.K / 32) + kc) * Nh * 32 +
                                                   (k / 16) * (Nh * 16) + (nn / 8) * 128 + (nn % 8) * 16 + (k % 16);
                                img[pos] = static_cast<uint8_t>(w.W[static_cast<size_t>(n) * w.in + kk]);
                            }
                        }
                pos0 += static_cast<size_t>(ly.N) * ly.K;
                if (p.bias_fold) {
                    // bias chunk after the layer's K/32 chunks: b = d0 + 255 * (d1 + ... + d31)
                    for (int n = 0; n < ly.N; ++n) {
                        const long long b = bias[static_cast<size_t>(ly.boff) + n];
                        long long q = (b >= 0 ? b + 127 : b - 127) / 255;
                        int8_t d[32];
                        d[0] = static_cast<int8_t>(b - 255 * q);
                        for (int k = 1; k < 32; ++k) {
                            const long long t = std::max(-127LL, std::min(127LL, q));
                            d[k] = static_cast<int8_t>(t);
                            q -= t;
                        }
                        for (int k = 0; k < 32; ++k)
                            img[pos0 + (k / 16) * (static_cast<size_t>(ly.N) * 16) + (n / 8) * 128 + (n % 8) * 16 + (k % 16)] =
                                static_cast<uint8_t>(d[k]);
                    }
                    pos0 += static_cast<size_t>(ly.N) * kKChunk;
                }
            }
        if (p.bias_fold)  // constant A block, K-major core-matrix layout
            for (int r = 0; r < kTileM; ++r)
                for (int k = 0; k < kKChunk; ++k)
                    img[static_cast<size_t>(p.cA_off) + (k / 16) * 2048 + r * 16 + (k % 16)] = k == 0 ? 1 : 255;
    }
    // BIDA_MLP_MULTICAST=1: streaming schedules run as CTA pairs sharing weight
    // stages by TMA multicast.  Off by default: measured slower on B200 (h512
    // 1.16 vs 1.26 G evals/s) -- the pair's lockstep costs more than the halved
    // per-SM copy issue saves (profiles/r1_notes.md).
    const char *mcv = std::getenv("BIDA_MLP_MULTICAST");
    if (p.mode != kWide)
        p.cluster = ((p.mode == kPair || p.mode == kSplit) && mcv && mcv[0] == '1') ? 2 : 1;
    m->cm = C <= 32 ? 32 : (C <= 64 ? 64 : 256);
    // C <= 24 on a fused schedule: a 24-wide readout (BIDA_MLP_CM24=0: 32)
    const char *c24 = std::getenv("BIDA_MLP_CM24");
    if (C <= 24 && p.mode != kWide && !(c24 && c24[0] == '0'))
        m->cm = 24;
    m->grid_cap = num_sms;
    if (const char *mc = std::getenv("BIDA_MLP_MAX_CTAS"))  // tests: many tiles per CTA on small batches
        m->grid_cap = std::max(1, std::min(num_sms, std::atoi(mc)));
    cudaError_t ce = cudaMalloc(&m->d_wimg, img.size());
    if (ce == cudaSuccess)
        ce = cudaMemcpy(m->d_wimg, img.data(), img.size(), cudaMemcpyHostToDevice);
    if (ce == cudaSuccess)
        ce = cudaMalloc(&m->d_bias, bias.size() * 4);
    if (ce == cudaSuccess)
        ce = cudaMemcpy(m->d_bias, bias.data(), bias.size() * 4, cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {
        mlp_destroy(m);
        return fail(err, 3, std::string("BMLP1 upload: ") + cudaGetErrorString(ce));
    }
    if (p.mode == kWide) {
        const size_t sb = static_cast<size_t>(((m->grid_cap + 1) & ~1)) * 2 * static_cast<size_t>(p.sbytes);
        for (int i = 0; i < kScratchPool && ce == cudaSuccess; ++i) {
            ce = cudaMalloc(reinterpret_cast<void **>(&m->scratch[i]), sb);
            if (ce == cudaSuccess)
                ce = cudaEventCreateWithFlags(&m->scratch_ev[i], cudaEventDisableTiming);
        }
        if (ce != cudaSuccess) {
            mlp_destroy(m);
            return fail(err, 3, std::string("BMLP1 scratch: ") + cudaGetErrorString(ce));
        }
    }
    p.wimg = m->d_wimg;
    p.bias = m->d_bias;
    shape->F = F;
    shape->C = static_cast<int>(C);
    shape->E = static_cast<int>(E);
    shape->L = static_cast<int>(L);
    for (uint32_t l = 0; l < L && l < 8; ++l)
        shape->H[l] = H[l];
    *out = m;
    return 0;
}

int mlp_launch(MlpModel *m, int domain, const void *d_packed, int64_t n, int32_t *d_h, double *d_logits,
               int *err_dev, unsigned long long *replays, cudaStream_t st, std::atomic<int64_t> *launches,
               const PdbArgs *pdb) {
    MlpParams p = m->p;  // per-call copy: concurrent launches on one handle are safe
    if (pdb)
        p.pdb = *pdb;
    else
        p.pdb.entries = nullptr;
    p.trace = m->trace;
    p.packed = d_packed;
    p.n = n;
    p.h_out = d_h;
    p.logits_out = d_logits;
    p.err = err_dev;
    p.replays = replays;
    int rc;
    switch (domain) {
    case kSTP2: rc = launch_d<kSTP2>(m, p, st); break;
    case kSTP3: rc = launch_d<kSTP3>(m, p, st); break;
    case kSTP4: rc = launch_d<kSTP4>(m, p, st); break;
    default: rc = launch_d<kRC>(m, p, st); break;
    }
    if (!rc && launches)
        launches->fetch_add(1, std::memory_order_relaxed);
    return rc;
}

namespace {
template <int DOMAIN, int CM>
int prepare_t(MlpModel *m, const MlpParams &p, KernelLaunch *out) {
    auto kern = [&] {
        if constexpr (CM <= 64)
            return p.mode == kResident ? (p.bias_fold && p.E == 1 ? (p.nl == 3 ? mlp_fused_kernel<DOMAIN, CM, 3> : mlp_fused_kernel<DOMAIN, CM, 2>)
                                                                   : mlp_fused_kernel<DOMAIN, CM, 1>)
                                       : mlp_fused_kernel<DOMAIN, CM>;
        else
            return mlp_fused_kernel<DOMAIN, CM>;
    }();
    std::call_once(m->attr_once, [&] {
        m->attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(m->smem));
    });
    if (m->attr_err != cudaSuccess)
        return 1;
    const long long ntiles = (p.n + kTileM - 1) / kTileM;
    out->func = reinterpret_cast<const void *>(kern);
    out->grid = dim3(static_cast<unsigned>(std::max<long long>(1, std::min<long long>(ntiles, m->grid_cap))));
    out->block = dim3(kMlpThreads);
    out->smem = m->smem;
    out->set_args(p);
    return 0;
}
template <int DOMAIN>
int prepare_d(MlpModel *m, const MlpParams &p, KernelLaunch *out) {
    switch (m->cm) {
    case 24: return prepare_t<DOMAIN, 24>(m, p, out);
    case 32: return prepare_t<DOMAIN, 32>(m, p, out);
    case 64: return prepare_t<DOMAIN, 64>(m, p, out);
    default: return prepare_t<DOMAIN, 256>(m, p, out);
    }
}
} // namespace

int mlp_prepare(MlpModel *m, int domain, const void *d_packed, int64_t n, int32_t *d_h, int *err_dev,
                unsigned long long *replays, const PdbArgs *pdb, KernelLaunch *out) {
    if (m->p.mode == kWide || m->p.cluster != 1 || m->trace)
        return 1;
    MlpParams p = m->p;
    if (pdb)
        p.pdb = *pdb;
    else
        p.pdb.entries = nullptr;
    p.trace = nullptr;
    p.packed = d_packed;
    p.n = n;
    p.h_out = d_h;
    p.logits_out = nullptr;
    p.err = err_dev;
    p.replays = replays;
    switch (domain) {
    case kSTP2: return prepare_d<kSTP2>(m, p, out);
    case kSTP3: return prepare_d<kSTP3>(m, p, out);
    case kSTP4: return prepare_d<kSTP4>(m, p, out);
    default: return prepare_d<kRC>(m, p, out);
    }
}

void mlp_destroy(MlpModel *m) {
    if (!m)
        return;
    if (m->d_wimg)
        cudaFree(m->d_wimg);
    if (m->d_bias)
        cudaFree(m->d_bias);
    for (int i = 0; i < kScratchPool; ++i) {
        if (m->scratch[i])
            cudaFree(m->scratch[i]);
        if (m->scratch_ev[i])
            cudaEventDestroy(m->scratch_ev[i]);
    }
    delete m;
}

const char *mlp_last_error() { return g_err.c_str(); }

} // namespace bida_gpu
