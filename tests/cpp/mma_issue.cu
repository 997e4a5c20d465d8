// mma_issue.cu — cost of issuing a layer's worth of tcgen05.mma.kind::i8
// (M=128, K=32, N=128, 16 distinct K steps, then commit + wait) under several
// issue-loop shapes, to find why the fused MLP kernel's MMA phases run at
// ~140 cycles per MMA when back-to-back MMAs reach the 64-cycle floor
// (profiles/r2_mma_issue.txt).  Diagnostic only.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <string>

#include "../../paper_2507_11916_b200/csrc/sm100.cuh"

using namespace bida_gpu;

template <int SHAPE, int NK>
__global__ void __launch_bounds__(128, 1) issue(int rounds, int nk_rt, int N, long long *out, int sts) {
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
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    sm100::fence_proxy_async_smem();
    if (warp == 0)
        sm100::tmem_alloc(&tslot, 512);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        const uint32_t sA = sm100::smem_u32(smem), sB = sA + 64 * 1024;
        const uint32_t cbytes = static_cast<uint32_t>(N) * 32u;
        const uint32_t idesc = sm100::make_idesc_i8(N);
        const int nk = NK > 0 ? NK : nk_rt;
        uint32_t ph = 0;
        const long long t0 = clock64();
        for (int r = 0; r < rounds; ++r) {
            const uint32_t dcol = tmem + (r & 1) * 256u;
            uint64_t adesc = sm100::make_smem_desc(sA, 2048u, 128u);
            uint64_t bdesc = sm100::make_smem_desc(sB, cbytes >> 1, 128u);
            if (SHAPE == 0) {
                // the kernel's shape: whole warp walks, one elected lane loops
                if (sm100::elect_one()) {
                    for (int j = 0; j < nk; ++j) {
                        sm100::mma_i8(dcol, adesc, bdesc, idesc, j > 0 ? 1u : 0u);
                        adesc += 4096u >> 4;
                        bdesc += cbytes >> 4;
                    }
                }
                __syncwarp();
            } else if (SHAPE == 1) {
                // lane 0 loops (no elect)
                if (threadIdx.x == 0) {
                    for (int j = 0; j < nk; ++j) {
                        sm100::mma_i8(dcol, adesc, bdesc, idesc, j > 0 ? 1u : 0u);
                        adesc += 4096u >> 4;
                        bdesc += cbytes >> 4;
                    }
                }
                __syncwarp();
            } else if (SHAPE == 2) {
                // whole warp loops, elect per MMA
                for (int j = 0; j < nk; ++j) {
                    if (sm100::elect_one())
                        sm100::mma_i8(dcol, adesc, bdesc, idesc, j > 0 ? 1u : 0u);
                    __syncwarp();
                    adesc += 4096u >> 4;
                    bdesc += cbytes >> 4;
                }
            } else {
                // SHAPE 3: predicate from one elect, every lane executes the
                // (predicated) tcgen05.mma so the loop stays warp-uniform
                uint32_t lead = sm100::elect_one() ? 1u : 0u;
                for (int j = 0; j < nk; ++j) {
                    asm volatile(
                        "{\n\t.reg .pred p, q;\n\t"
                        "setp.ne.b32 p, %4, 0;\n\t"
                        "setp.ne.b32 q, %5, 0;\n\t"
                        "@q tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dcol),
                        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(j > 0 ? 1u : 0u), "r"(lead)
                        : "memory");
                    adesc += 4096u >> 4;
                    bdesc += cbytes >> 4;
                }
                __syncwarp();
            }
            if (sm100::elect_one())
                sm100::mma_commit(&bar);
            __syncwarp();
            sm100::mbar_wait(&bar, ph);
            ph ^= 1u;
            sm100::tc_fence_after();
        }
        if (threadIdx.x == 0) {
            out[blockIdx.x] = clock64() - t0;
            stop = 1;
        }
    } else if (sts) {
        // warps 1-3 stream st.shared.v4 into a region the MMAs do not read
        // (an epilogue writing the next tile's one-hot while the MMAs run)
        const uint32_t base = sm100::smem_u32(smem) + 144 * 1024 + (warp - 1) * 4096 + (threadIdx.x & 31) * 16;
        while (!stop)
            for (int r = 0; r < 8; ++r)
                sm100::st_shared_v4(base + (r & 7) * 512, r, r, r, r);
    }
    __syncwarp();
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    if (warp == 0)
        sm100::tmem_dealloc(tmem, 512);
}

template <int SHAPE, int NK>
static void run(const char *name, int N, int nk, int sts = 0) {
    long long *d_out, h_out[148];
    cudaMalloc(&d_out, sizeof(h_out));
    cudaFuncSetAttribute(issue<SHAPE, NK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const int rounds = 256;
    issue<SHAPE, NK><<<148, 128, 160 * 1024>>>(rounds, nk, N, d_out, sts);
    if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("error\n");
        return;
    }
    cudaMemcpy(h_out, d_out, sizeof(h_out), cudaMemcpyDeviceToHost);
    double tot = 0;
    for (int g = 0; g < 148; ++g)
        tot += h_out[g];
    tot /= 148.0 * rounds;
    printf("{\"shape\": \"%s\", \"N\": %d, \"k_steps\": %d, \"sts_warps\": %d, \"cycles_per_round\": %.0f, "
           "\"cycles_per_mma\": %.1f, \"floor\": %.0f}\n",
           name, N, nk, sts ? 3 : 0, tot, tot / nk, 128.0 * N / 256.0);
    cudaFree(d_out);
}

int main(int argc, char **argv) {
    if (argc > 1 && std::string(argv[1]) == "sts") {
        for (int N : {32, 128, 256})
            for (int sts : {0, 1})
                run<0, 16>("elect+loop, 16 unrolled", N, 16, sts);
        return 0;
    }
    for (int N : {32, 128}) {
        for (int nk : {4, 16}) {
            run<0, 0>("elect+loop (kernel)", N, nk);
            run<1, 0>("lane0 loop", N, nk);
            run<2, 0>("elect per mma", N, nk);
            run<3, 0>("predicated, uniform loop", N, nk);
        }
        run<0, 16>("elect+loop, 16 unrolled", N, 16);
        run<3, 16>("predicated, 16 unrolled", N, 16);
    }
    return 0;
}
