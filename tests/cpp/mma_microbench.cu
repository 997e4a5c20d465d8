// mma_microbench.cu — measures the issue-to-completion cost of back-to-back
// tcgen05.mma.kind::i8 (M=128, K=32) from shared-memory operands for several
// N and smem layouts (SWIZZLE_NONE interleave vs 128B swizzle).  Diagnostic
// only; results go to profiles/.  Build: see tests/cpp/Makefile (mma_microbench).
#include <cstdio>
#include <cstdint>
#include <string>
#include <cuda_runtime.h>

#include "../../paper_2507_11916_b200/csrc/sm100.cuh"

using namespace bida_gpu;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1) << 16;              // LBO (unused for swizzled K-major) = 16 B
    d |= static_cast<uint64_t>(1024 >> 4) << 32;      // SBO = 1024 B between 8-row groups
    d |= static_cast<uint64_t>(1) << 46;              // version
    d |= static_cast<uint64_t>(2) << 61;              // SWIZZLE_128B
    return d;
}

__global__ void __launch_bounds__(128, 1) bench(int n_mma, int N, int layout, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        sm100::mbar_init(&bar, 1);
        sm100::fence_barrier_init();
    }
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    sm100::fence_proxy_async_smem();
    if (warp == 0)
        sm100::tmem_alloc(&tslot, 512);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint32_t sA = sm100::smem_u32(smem), sB = sA + 32 * 1024;
        const uint32_t idesc = sm100::make_idesc_i8(N);
        const long long t0 = clock64();
        for (int i = 0; i < n_mma; ++i) {
            uint64_t a, b;
            const int ks = i & 3;
            if (layout == 0) {  // interleave: K halves 2048 B apart (A), N*16 apart (B)
                a = sm100::make_smem_desc(sA + ks * 4096u, 2048u, 128u);
                b = sm100::make_smem_desc(sB + ks * (N * 32u), N * 16u, 128u);
            } else {            // 128B swizzle: advance 32 B within the 128 B row
                a = desc_sw128(sA + ks * 32u);
                b = desc_sw128(sB + ks * 32u);
            }
            sm100::mma_i8(tmem, a, b, idesc, i > 0 ? 1u : 0u);
        }
        sm100::mma_commit(&bar);
        const long long t1 = clock64();
        sm100::mbar_wait(&bar, 0);
        const long long t2 = clock64();
        out[blockIdx.x * 2 + 0] = t1 - t0;
        out[blockIdx.x * 2 + 1] = t2 - t0;
    }
    __syncwarp();
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    if (warp == 0)
        sm100::tmem_dealloc(tmem, 512);
}

// SS MMAs (A and B from SMEM) issued by warp 0 while `sts_warps` other warps
// stream st.shared.v4 into a separate SMEM region: does epilogue-style SMEM
// traffic slow the tensor core's operand reads?  ts=1: A from TMEM instead.
__global__ void __launch_bounds__(512, 1) contention(int n_mma, int N, int sts_warps, int ts, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar, bar2;
    __shared__ uint32_t tslot;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        sm100::mbar_init(&bar, 1);
        sm100::mbar_init(&bar2, 1);
        sm100::fence_barrier_init();
        stop = 0;
    }
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    sm100::fence_proxy_async_smem();
    if (warp == 0)
        sm100::tmem_alloc(&tslot, 512);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        if (threadIdx.x == 0) {
            const uint32_t sA = sm100::smem_u32(smem), sB = sA + 32 * 1024;
            const uint32_t idesc = sm100::make_idesc_i8(N);
            const long long t0 = clock64();
            for (int i = 0; i < n_mma; ++i) {
                const int ks = i & 3;
                const uint64_t b = sm100::make_smem_desc(sB + ks * (N * 32u), N * 16u, 128u);
                if (ts == 1) {
                    // A operand in TMEM columns [256 + 8ks, +8): 128 lanes x 32 int8
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                        "r"(tmem + 256 + ks * 8), "l"(b), "r"(idesc), "r"(i > 0 ? 1u : 0u)
                        : "memory");
                } else {
                    const uint64_t a = sm100::make_smem_desc(sA + ks * 4096u, 2048u, 128u);
                    sm100::mma_i8(tmem, a, b, idesc, i > 0 ? 1u : 0u);
                }
            }
            sm100::mma_commit(&bar);
            sm100::mbar_wait(&bar, 0);
            out[blockIdx.x] = clock64() - t0;
            stop = 1;
            sm100::mbar_arrive(&bar2);
        }
    } else if (warp <= sts_warps) {
        if (ts >= 2) {
            // ts 2: waiting epilogue warps polling an mbarrier (mbarrier.try_wait
            // loop, as mbar_wait does); ts 3: same with a 64 ns sleep per poll
            while (!stop) {
                if (sm100::mbar_try_wait(&bar2, 0))
                    break;
                if (ts == 3)
                    __nanosleep(64);
            }
        } else {
            const uint32_t base = sm100::smem_u32(smem) + 64 * 1024 + (warp - 1) * 512 + (threadIdx.x & 31) * 16;
            while (!stop)
                for (int r = 0; r < 16; ++r)
                    sm100::st_shared_v4(base, r, r, r, r);
        }
    }
    __syncwarp();
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    if (warp == 0)
        sm100::tmem_dealloc(tmem, 512);
}

// SS MMAs (N = 128, the h128 schedule's shape) issued by warp 0 while
// `ld_warps` other warps loop tcgen05.ld.32x32b.x16 + wait::ld over TMEM
// columns [256, 384): does an epilogue draining the other TMEM half slow the
// MMAs of the next job?  (profiles/r2_mma_tmem_contention.txt)
__global__ void __launch_bounds__(512, 1) tmem_contention(int n_mma, int N, int ld_warps, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        sm100::mbar_init(&bar, 1);
        sm100::fence_barrier_init();
        stop = 0;
    }
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    sm100::fence_proxy_async_smem();
    if (warp == 0)
        sm100::tmem_alloc(&tslot, 512);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = tslot;
    int sink = 0;
    if (warp == 0) {
        if (threadIdx.x == 0) {
            const uint32_t sA = sm100::smem_u32(smem), sB = sA + 32 * 1024;
            const uint32_t idesc = sm100::make_idesc_i8(N);
            const long long t0 = clock64();
            for (int i = 0; i < n_mma; ++i) {
                const int ks = i & 3;
                const uint64_t a = sm100::make_smem_desc(sA + ks * 4096u, 2048u, 128u);
                const uint64_t b = sm100::make_smem_desc(sB + ks * (N * 32u), N * 16u, 128u);
                sm100::mma_i8(tmem, a, b, idesc, i > 0 ? 1u : 0u);
            }
            sm100::mma_commit(&bar);
            sm100::mbar_wait(&bar, 0);
            out[blockIdx.x] = clock64() - t0;
            stop = 1;
        }
    } else if (warp <= ld_warps) {
        const uint32_t taddr = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 256u;
        int32_t r[16];
        int k = 0;
        while (!stop) {
            sm100::tmem_ld16(taddr + (k & 7) * 16u, r);
            sm100::tmem_wait_ld();
            sink += r[0] + r[15];
            ++k;
        }
    }
    if (sink == 0x7fffffff)
        out[0] = sink;
    __syncwarp();
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    if (warp == 0)
        sm100::tmem_dealloc(tmem, 512);
}

// Streaming operands: every MMA reads a DIFFERENT A (4 KB) and B (N*32 B) from
// a ring of `nbuf` operand sets, optionally while warp 1 keeps the TMA engine
// writing `tma_kb` KB stages from global memory into a separate region (the
// wide schedule's situation).  Reports cycles per MMA.
__global__ void __launch_bounds__(128, 1) stream(int n_mma, int N, int nbuf, int tma_kb, const uint8_t *gsrc,
                                                 long long *out, int commit_every) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar, tbar, cbar;
    __shared__ uint32_t tslot;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5;
    const uint32_t setb = 4096u + N * 32u;
    if (threadIdx.x == 0)
        sm100::mbar_init(&cbar, 1);
    if (threadIdx.x == 0) {
        sm100::mbar_init(&bar, 1);
        sm100::mbar_init(&tbar, 1);
        sm100::fence_barrier_init();
        stop = 0;
    }
    for (int i = threadIdx.x; i < (int)(nbuf * setb / 16); i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    sm100::fence_proxy_async_smem();
    if (warp == 0)
        sm100::tmem_alloc(&tslot, 512);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        // whole warp walks the loop, descriptors advanced by adds, elected lane issues
        const uint32_t base = sm100::smem_u32(smem);
        const uint32_t idesc = sm100::make_idesc_i8(N);
        const uint64_t a0 = sm100::make_smem_desc(base, 2048u, 128u);
        const uint64_t b0 = sm100::make_smem_desc(base + 4096u, N * 16u, 128u);
        const long long t0 = clock64();
        uint64_t off = 0;
        int j = 0;
        for (int i = 0; i < n_mma; ++i) {
            if (sm100::elect_one()) {
                sm100::mma_i8(tmem, a0 + off, b0 + off, idesc, i > 0 ? 1u : 0u);
                if (commit_every && (i % commit_every) == commit_every - 1)
                    sm100::mma_commit(&cbar);  // per-stage release, as the streaming schedules do
            }
            __syncwarp();
            off += setb >> 4;
            if (++j == nbuf) {
                j = 0;
                off = 0;
            }
        }
        if (sm100::elect_one())
            sm100::mma_commit(&bar);
        __syncwarp();
        sm100::mbar_wait(&bar, 0);
        if (threadIdx.x == 0) {
            out[blockIdx.x] = clock64() - t0;
            stop = 1;
        }
    } else if (warp == 1 && tma_kb > 0) {
        if (threadIdx.x == 32) {
            uint8_t *dst = smem + nbuf * setb;
            uint32_t ph = 0;
            const uint32_t bytes = tma_kb * 1024u;
            long long off = (blockIdx.x * 7919LL * 1024) % (64LL << 20);
            while (!stop) {
                sm100::mbar_arrive_expect_tx(&tbar, bytes);
                sm100::bulk_g2s(dst, gsrc + off, bytes, &tbar);
                sm100::mbar_wait(&tbar, ph);
                ph ^= 1u;
                off = (off + bytes) % (64LL << 20);
            }
        }
    }
    __syncwarp();
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    if (warp == 0)
        sm100::tmem_dealloc(tmem, 512);
}

// Sustained dense int8 rate on every SM: back-to-back M=128 N=256 K=32
// kind::i8 MMAs from SMEM (the per-SM tcgen05 floor) for ~0.25 s per launch,
// timed with CUDA events -- the roofline denominator for the BMLP1 kernels
// (profiles/r2_int8_peak.txt).
static int sustained() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long *d_out;
    cudaMalloc(&d_out, sizeof(long long) * 2 * sms);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int n = 4000000, N = 256;
    bench<<<sms, 128, 64 * 1024>>>(1000, N, 0, d_out);  // warm
    cudaDeviceSynchronize();
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a);
        bench<<<sms, 128, 64 * 1024>>>(n, N, 0, d_out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = 2.0 * sms * static_cast<double>(n) * 128 * N * 32;
        printf("{\"what\": \"int8_dense_sustained\", \"sms\": %d, \"mma\": \"M128 N256 K32 kind::i8, SMEM operands\", "
               "\"ms\": %.3f, \"tops\": %.1f}\n", sms, ms, ops / (ms * 1e-3) / 1e12);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

static int tmem_contention_run() {
    long long *d_out, h_out[148];
    cudaMalloc(&d_out, sizeof(h_out));
    cudaFuncSetAttribute(tmem_contention, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int N : {128, 256})
        for (int w : {0, 4, 8, 15}) {
            const int n = 2048;
            tmem_contention<<<148, 512, 64 * 1024>>>(n, N, w, d_out);
            if (cudaDeviceSynchronize() != cudaSuccess)
                return 1;
            cudaMemcpy(h_out, d_out, sizeof(h_out), cudaMemcpyDeviceToHost);
            double tot = 0;
            for (int g = 0; g < 148; ++g)
                tot += h_out[g];
            printf("tmem_ld contention N=%3d ld_warps=%2d  %.1f cyc/mma (floor %.0f)\n", N, w, tot / 148 / n,
                   128.0 * N / 256.0);
        }
    return 0;
}

int main(int argc, char **argv) {
    if (argc > 1 && std::string(argv[1]) == "sustained")
        return sustained();
    if (argc > 1 && std::string(argv[1]) == "tmem")
        return tmem_contention_run();
    long long *d_out, h_out[2 * 148];
    cudaMalloc(&d_out, sizeof(h_out));
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int layout = 0; layout < 2; ++layout)
        for (int N : {32, 64, 128, 256}) {
            const int n = 512;
            for (int grid : {1, 148}) {
                bench<<<grid, 128, 64 * 1024>>>(n, N, layout, d_out);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("error %s\n", cudaGetErrorString(e));
                    return 1;
                }
                cudaMemcpy(h_out, d_out, sizeof(long long) * 2 * grid, cudaMemcpyDeviceToHost);
                double issue = 0, total = 0;
                for (int g = 0; g < grid; ++g) {
                    issue += h_out[2 * g];
                    total += h_out[2 * g + 1];
                }
                issue /= grid;
                total /= grid;
                const double floor_cyc = 128.0 * N / 256.0;
                printf("layout=%s N=%3d grid=%3d  issue %.1f cyc/mma  complete %.1f cyc/mma  floor %.1f  -> %.0f%% of peak\n",
                       layout ? "sw128" : "interleave", N, grid, issue / n, total / n, floor_cyc,
                       100.0 * floor_cyc / (total / n));
            }
        }
    cudaFuncSetAttribute(contention, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    for (int ts = 0; ts < 4; ++ts)
        for (int N : {32, 128, 256})
            for (int w : {0, 4, 8, 15}) {
                const int n = 512;
                contention<<<148, 512, 96 * 1024>>>(n, N, w, ts, d_out);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("error %s\n", cudaGetErrorString(e));
                    return 1;
                }
                cudaMemcpy(h_out, d_out, sizeof(long long) * 148, cudaMemcpyDeviceToHost);
                double tot = 0;
                for (int g = 0; g < 148; ++g)
                    tot += h_out[g];
                tot /= 148;
                printf("contention %s N=%3d warps=%2d  %.1f cyc/mma (floor %.0f)\n",
                       ts == 0 ? "A=smem sts" : ts == 1 ? "A=tmem sts" : ts == 2 ? "A=smem mbar-spin" : "A=smem mbar-sleep", N, w,
                       tot / n, 128.0 * N / 256.0);
            }
    {
        uint8_t *g;
        cudaMalloc(&g, (64 << 20) + (64 << 10));
        cudaMemset(g, 1, (64 << 20) + (64 << 10));
        cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        for (int ce : {0, 1, 2, 4})
        for (int N : {32, 128, 256})
            for (int nbuf : {8})
                for (int tkb : {0}) {
                    const int n = 2048;
                    const int setb = 4096 + N * 32;
                    if (nbuf * setb + tkb * 1024 > 200 * 1024)
                        continue;
                    stream<<<148, 128, 200 * 1024>>>(n, N, nbuf, tkb, g, d_out, ce);
                    cudaError_t e = cudaDeviceSynchronize();
                    if (e != cudaSuccess) {
                        printf("error %s\n", cudaGetErrorString(e));
                        return 1;
                    }
                    cudaMemcpy(h_out, d_out, sizeof(long long) * 148, cudaMemcpyDeviceToHost);
                    double tot = 0;
                    for (int g2 = 0; g2 < 148; ++g2)
                        tot += h_out[g2];
                    tot /= 148;
                    printf("stream N=%3d operand sets=%d tma_stage=%2d KB commit_every=%d  %.1f cyc/mma (floor %.0f)  smem read %.0f B/clk\n", N,
                           nbuf, tkb, ce, tot / n, 128.0 * N / 256.0, (4096.0 + N * 32.0) / (tot / n));
                }
    }
    return 0;
}
