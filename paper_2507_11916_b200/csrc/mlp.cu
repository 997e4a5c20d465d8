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
// warps 2-5 encode/epilogue/readout (thread = TMEM lane = tile row).
//
// Integer arithmetic makes every logit exact, so h is bit-identical to the
// oracle's BMLP1 restatement (oracle/bida_oracle.c) in any MMA order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "certified_readout.cuh"
#include "common.cuh"
#include "encode.cuh"
#include "mlp.cuh"
#include "sm100.cuh"

namespace bida_gpu {

constexpr int kMaxMembers = 8;
constexpr int kMaxLayers = 5;   // hidden layers <= 4
constexpr int kTileM = 128;
constexpr int kMaxStages = 6;
constexpr int kStageBytes = 16384;
constexpr int kMlpThreads = 320;  // warp 0 producer, warp 1 MMA, warps 2-9 two epilogue groups
constexpr int kKChunk = 32;       // bytes of K per MMA instruction

struct MlpLayer {
    int K, N;          // padded input width (multiple of 32), output width (multiple of 16)
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
    int slots;          // 2: two tiles in flight (ping-pong); 1: both groups split one tile's columns
    int stages;         // weight ring depth (16 KB stages)
    int xbytes, ybytes; // activation buffers per slot (even / odd layer inputs)
    // batch
    const void *packed;
    long long n;
    int32_t *h_out;
    double *logits_out;
    int *err;
};

struct MlpModel {
    MlpParams p;
    uint8_t *d_wimg = nullptr;
    int32_t *d_bias = nullptr;
    size_t smem = 0;
    int grid_cap = 148;
    int cm = 32;
};

namespace {
thread_local std::string g_err;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// K-chunks (32 B of K each) carried by one 16 KB stage for a layer with N outputs.
__device__ __forceinline__ int chunks_per_stage(int N) {
    const int c = kStageBytes / (N * kKChunk);
    return c < 1 ? 1 : c;
}
} // namespace

// One CTA per SM, persistent over the CTA's tiles of 128 states.  Local tile
// k of this CTA is t = blockIdx.x + k * gridDim.x; with two slots, tiles
// alternate between slot 0 and 1 (epilogue group g owns slot g), and the MMA
// issuer interleaves the slots layer by layer so one slot's tensor-core work
// overlaps the other slot's epilogue.
template <int DOMAIN, int CM>
__global__ void __launch_bounds__(kMlpThreads, 1) mlp_fused_kernel(const __grid_constant__ MlpParams p) {
    using T = DomainTraits<DOMAIN>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int slot_bytes = p.xbytes + p.ybytes;
    uint8_t *stages = smem + p.slots * slot_bytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(stages + p.stages * kStageBytes);
    uint64_t *full = bars;                       // [kMaxStages]
    uint64_t *empty = bars + kMaxStages;         // [kMaxStages]
    uint64_t *act_ready = bars + 2 * kMaxStages; // [2]
    uint64_t *d_full = act_ready + 2;            // [2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(d_full + 2);

    const int warp = threadIdx.x >> 5;
    const long long ntiles = (p.n + kTileM - 1) / kTileM;
    const long long nloc = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const int slots = p.slots;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kMaxStages; ++s) {
            sm100::mbar_init(&full[s], 1);
            sm100::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            sm100::mbar_init(&act_ready[s], slots == 2 ? 128 : 256);
            sm100::mbar_init(&d_full[s], 1);
        }
        sm100::fence_barrier_init();
    }
    if (warp == 1)
        sm100::tmem_alloc(tmem_slot, p.tmem_cols);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ weight producer
        if (lane_id() == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (long long k0 = 0; k0 < nloc; k0 += slots)
                for (int e = 0; e < p.E; ++e)
                    for (int l = 0; l < p.nl; ++l)
                        for (int sl = 0; sl < slots && k0 + sl < nloc; ++sl) {
                            const MlpLayer &ly = p.layer[e][l];
                            const int nch = ly.K / kKChunk, cps = chunks_per_stage(ly.N);
                            const uint32_t cbytes = static_cast<uint32_t>(ly.N) * kKChunk;
                            for (int kc = 0; kc < nch; kc += cps) {
                                const int cnt = min(cps, nch - kc);
                                sm100::mbar_wait(&empty[s], ph ^ 1u);
                                sm100::mbar_arrive_expect_tx(&full[s], cnt * cbytes);
                                sm100::bulk_g2s(stages + s * kStageBytes, p.wimg + ly.woff + static_cast<size_t>(kc) * cbytes,
                                                cnt * cbytes, &full[s]);
                                if (++s == p.stages) {
                                    s = 0;
                                    ph ^= 1u;
                                }
                            }
                        }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane_id() == 0) {
            int s = 0;
            uint32_t ph = 0, aph[2] = {0u, 0u};
            const uint32_t sbase = sm100::smem_u32(smem), sS = sm100::smem_u32(stages);
            for (long long k0 = 0; k0 < nloc; k0 += slots)
                for (int e = 0; e < p.E; ++e)
                    for (int l = 0; l < p.nl; ++l)
                        for (int sl = 0; sl < slots && k0 + sl < nloc; ++sl) {
                            const MlpLayer &ly = p.layer[e][l];
                            sm100::mbar_wait(&act_ready[sl], aph[sl]);
                            aph[sl] ^= 1u;
                            sm100::tc_fence_after();
                            const uint32_t abase = sbase + sl * slot_bytes + ((l & 1) ? p.xbytes : 0);
                            const uint32_t dcol = tmem + sl * 256u;
                            const uint32_t lbo_b = static_cast<uint32_t>(ly.N) * 16u;
                            const int nch = ly.K / kKChunk, cps = chunks_per_stage(ly.N);
                            const uint32_t idesc_full = sm100::make_idesc_i8(ly.N < 256 ? ly.N : 256);
                            for (int kc = 0; kc < nch; kc += cps) {
                                const int cnt = min(cps, nch - kc);
                                sm100::mbar_wait(&full[s], ph);
                                sm100::tc_fence_after();
                                const uint32_t stg = sS + s * kStageBytes;
                                for (int j = 0; j < cnt; ++j) {
                                    const uint64_t adesc = sm100::make_smem_desc(abase + (kc + j) * 4096u, 2048u, 128u);
                                    const uint32_t cb = stg + j * static_cast<uint32_t>(ly.N) * kKChunk;
                                    for (int n0 = 0; n0 < ly.N; n0 += 256) {
                                        const int nn = ly.N - n0 < 256 ? ly.N - n0 : 256;
                                        const uint64_t bdesc = sm100::make_smem_desc(cb + (n0 / 8) * 128u, lbo_b, 128u);
                                        sm100::mma_i8(dcol + n0, adesc, bdesc,
                                                      nn == 256 ? idesc_full : sm100::make_idesc_i8(nn),
                                                      (kc + j) > 0 ? 1u : 0u);
                                    }
                                }
                                sm100::mma_commit(&empty[s]);
                                if (++s == p.stages) {
                                    s = 0;
                                    ph ^= 1u;
                                }
                            }
                            sm100::mma_commit(&d_full[sl]);
                        }
        }
    } else {
        // ------------------------------------------------ encode / epilogue / readout
        const int grp = (warp - 2) >> 2;           // epilogue group 0 / 1
        const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
        const int row = quad * 32 + lane_id();     // tile row == TMEM lane
        const int sl = slots == 2 ? grp : 0;
        const bool leader = slots == 2 || grp == 0;  // encodes, reads out, writes h
        const uint32_t t_row = tmem + sl * 256u + (static_cast<uint32_t>(quad * 32) << 16);
        const uint32_t sX = sm100::smem_u32(smem) + sl * slot_bytes;
        const uint32_t sY = sX + p.xbytes;
        uint64_t *my_ready = &act_ready[sl];
        uint64_t *my_full = &d_full[sl];
        uint32_t dph = 0;
        const long long kstep = slots == 2 ? 2 : 1;
        // packed states are prefetched one tile ahead (HBM latency off the critical path)
        auto load_state = [&](long long kk, uint64_t &lo_, uint64_t &hi_) {
            lo_ = hi_ = 0;
            const long long s_ = (blockIdx.x + kk * gridDim.x) * kTileM + row;
            if (kk < nloc && s_ < p.n && leader) {
                if constexpr (T::PB == 16) {
                    const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2 *>(p.packed) + s_);
                    lo_ = v.x;
                    hi_ = v.y;
                } else {
                    lo_ = __ldcs(reinterpret_cast<const unsigned long long *>(p.packed) + s_);
                }
            }
        };
        uint64_t nlo, nhi;
        load_state(slots == 2 ? grp : 0, nlo, nhi);
        for (long long k = (slots == 2 ? grp : 0); k < nloc; k += kstep) {
            const long long t = blockIdx.x + k * gridDim.x;
            const long long st = t * kTileM + row;
            const bool valid = st < p.n;
            const uint64_t lo = nlo, hi = nhi;
            load_state(k + kstep, nlo, nhi);
            int idx[T::NNZ];
            bool bad = false;
#pragma unroll
            for (int q = 0; q < T::NNZ; ++q) {
                idx[q] = position_feature<DOMAIN>(lo, hi, q);
                bad |= idx[q] < 0 || idx[q] >= T::F;
            }
            bad = bad && valid && leader;
            if (bad)
                raise_error(p.err, kErrState);
            const bool live = valid && !bad;
            int hmin = 0x7fffffff;
            bool dist_bad = false;
            for (int e = 0; e < p.E; ++e) {
                if (leader) {
                    // ---- encode: one-hot row into X (layer 0's A operand)
                    for (int c16 = 0; c16 < p.Fpad / 16; ++c16)
                        sm100::st_shared_v4(sX + c16 * 2048u + row * 16u, 0u, 0u, 0u, 0u);
                    if (live) {
#pragma unroll
                        for (int q = 0; q < T::NNZ; ++q) {
                            const int j = idx[q];
                            sm100::st_shared_u8(sX + (j >> 4) * 2048u + row * 16u + (j & 15), 1u);
                        }
                    }
                    sm100::fence_proxy_async_smem();
                }
                sm100::mbar_arrive(my_ready);
                for (int l = 0; l < p.nl; ++l) {
                    const MlpLayer &ly = p.layer[e][l];
                    sm100::mbar_wait(my_full, dph);
                    dph ^= 1u;
                    sm100::tc_fence_after();
                    const int32_t *bias = p.bias + ly.boff;
                    if (l + 1 < p.nl) {
                        // hidden layer epilogue: bias, shift, clamp -> int8 A operand of layer l+1
                        const uint32_t out = ((l + 1) & 1) ? sY : sX;
                        const int half = slots == 2 ? ly.N : ly.N / 2;
                        const int c_beg = slots == 2 ? 0 : grp * half, c_end = c_beg + half;
                        // software-pipelined: the TMEM load of the next 16 columns is in
                        // flight while the current 16 are requantised and stored
                        const int sh = ly.shift;
                        auto requant = [&](const int32_t(&r)[16], const int4(&b4)[4], int c0) {
                            uint32_t w[4];
#pragma unroll
                            for (int q = 0; q < 4; ++q)  // (acc + bias) >> shift, saturated to u8 0..255
                                w[q] = sm100::pack_sat_u8x4((r[q * 4 + 0] + b4[q].x) >> sh, (r[q * 4 + 1] + b4[q].y) >> sh,
                                                            (r[q * 4 + 2] + b4[q].z) >> sh, (r[q * 4 + 3] + b4[q].w) >> sh);
                            sm100::st_shared_v4(out + (c0 >> 4) * 2048u + row * 16u, w[0], w[1], w[2], w[3]);
                        };
                        auto load_bias = [&](int4(&b4)[4], int c0) {
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                b4[q] = __ldg(reinterpret_cast<const int4 *>(bias + c0) + q);
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
                        sm100::tc_fence_before();
                        sm100::fence_proxy_async_smem();
                        sm100::mbar_arrive(my_ready);
                    } else if (leader) {
                        // output layer: exact integer logits -> certified readout
                        int32_t v[CM];
#pragma unroll
                        for (int c0 = 0; c0 < CM; c0 += 16) {
                            if (c0 < p.C) {
                                int32_t r[16];
                                sm100::tmem_ld16(t_row + c0, r);
                                sm100::tmem_wait_ld();
#pragma unroll
                                for (int j = 0; j < 16; ++j)
                                    v[c0 + j] = r[j] + ((c0 + j < p.C) ? __ldg(bias + c0 + j) : 0);
                            }
                        }
                        sm100::tc_fence_before();
                        if (p.logits_out && valid) {
                            double *dst = p.logits_out + (static_cast<size_t>(st) * p.E + e) * p.C;
                            for (int c = 0; c < p.C; ++c)
                                dst[c] = static_cast<double>(v[c]) * p.scale_d[e];
                        }
                        bool fb = false;
                        const int h = readout_certified<CM>(v, p.C, p.scale_f[e], p.scale_d[e], p.rk, &dist_bad, &fb);
                        hmin = min(hmin, h);
                    }
                }
            }
            if (leader && valid) {
                if (dist_bad)
                    raise_error(p.err, kErrDistribution);
                p.h_out[st] = (live && !dist_bad) ? hmin : 0;
            }
        }
    }

    __syncwarp();  // reconverge the single-thread roles before the aligned barrier
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    if (warp == 1)
        sm100::tmem_dealloc(tmem, p.tmem_cols);
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
    auto kern = mlp_fused_kernel<DOMAIN, CM>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(m->smem));
    if (e != cudaSuccess) {
        g_err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e);
        return 1;
    }
    const long long ntiles = (p.n + kTileM - 1) / kTileM;
    const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>(ntiles, m->grid_cap)));
    kern<<<grid, kMlpThreads, m->smem, st>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) {
        g_err = std::string("mlp launch: ") + cudaGetErrorString(e);
        return 1;
    }
    return 0;
}

template <int DOMAIN>
int launch_d(MlpModel *m, const MlpParams &p, cudaStream_t st) {
    switch (m->cm) {
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
        if (H[l] < 32 || H[l] > 512 || H[l] % 32)
            return fail(err, 1, "BMLP1: hidden widths must be multiples of 32 in [32, 512]");
    }
    const int Fpad = (F + 31) / 32 * 32;
    const int Cpad = std::max(16, (static_cast<int>(C) + 15) / 16 * 16);
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
        Nmax = std::max(Nmax, H[l]);
        if ((l + 1) % 2 == 0)
            KX = std::max(KX, H[l]);
        else
            KY = std::max(KY, H[l]);
    }
    std::vector<uint8_t> img;
    std::vector<int32_t> bias;
    for (uint32_t e = 0; e < E; ++e) {
        for (int l = 0; l < nl; ++l) {
            const int in = l ? H[l - 1] : F;
            const int outn = l < static_cast<int>(L) ? H[l] : static_cast<int>(C);
            const int K = l ? H[l - 1] : Fpad;
            const int N = l < static_cast<int>(L) ? H[l] : Cpad;
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
            ly.woff = static_cast<long long>(img.size());
            ly.boff = static_cast<int>(bias.size());
            // weight image: K/32 chunks of [2 halves][N/8 groups][8 rows][16 bytes]
            const size_t base = img.size();
            img.resize(base + static_cast<size_t>(N) * K, 0);
            for (int kc = 0; kc < K / 32; ++kc)
                for (int n = 0; n < outn; ++n)
                    for (int k = 0; k < 32; ++k) {
                        const int kk = kc * 32 + k;
                        if (kk >= in)
                            continue;
                        const size_t pos = base + static_cast<size_t>(kc) * N * 32 + (k / 16) * (N * 16) +
                                           (n / 8) * 128 + (n % 8) * 16 + (k % 16);
                        img[pos] = static_cast<uint8_t>(W[static_cast<size_t>(n) * in + kk]);
                    }
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
    const size_t bar_bytes = 8 * (2 * kMaxStages + 4) + 16;
    const size_t budget = 227 * 1024;
    auto stages_for = [&](int slots) -> int {
        const size_t act = static_cast<size_t>(slots) * (p.xbytes + p.ybytes);
        if (act + bar_bytes + 2 * kStageBytes > budget)
            return 0;
        return static_cast<int>(std::min<size_t>(4, (budget - act - bar_bytes) / kStageBytes));
    };
    // Two tiles in flight when both accumulators fit TMEM (2 x 256 columns)
    // and both slots' activation buffers fit shared memory; else one tile
    // whose columns the two epilogue groups split.
    if (Nmax <= 256 && stages_for(2) >= 2) {
        p.slots = 2;
        p.stages = stages_for(2);
        p.tmem_cols = 512;
    } else if (stages_for(1) >= 2) {
        p.slots = 1;
        p.stages = stages_for(1);
        uint32_t cols = 32;
        while (cols < static_cast<uint32_t>(Nmax))
            cols <<= 1;
        p.tmem_cols = cols;
    } else {
        delete m;
        return fail(err, 1, "BMLP1: model too wide for shared memory");
    }
    m->cm = C <= 32 ? 32 : (C <= 64 ? 64 : 256);
    m->smem = static_cast<size_t>(p.slots) * (p.xbytes + p.ybytes) + static_cast<size_t>(p.stages) * kStageBytes + bar_bytes;
    m->grid_cap = num_sms;
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
               int *err_dev, cudaStream_t st, std::atomic<int64_t> *launches) {
    MlpParams p = m->p;  // per-call copy: concurrent launches on one handle are safe
    p.packed = d_packed;
    p.n = n;
    p.h_out = d_h;
    p.logits_out = d_logits;
    p.err = err_dev;
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

void mlp_destroy(MlpModel *m) {
    if (!m)
        return;
    if (m->d_wimg)
        cudaFree(m->d_wimg);
    if (m->d_bias)
        cudaFree(m->d_bias);
    delete m;
}

const char *mlp_last_error() { return g_err.c_str(); }

} // namespace bida_gpu
