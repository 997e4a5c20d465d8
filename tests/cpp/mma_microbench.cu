// mma_microbench.cu — measures the issue-to-completion cost of back-to-back
// tcgen05.mma.kind::i8 (M=128, K=32) from shared-memory operands for several
// N and smem layouts (SWIZZLE_NONE interleave vs 128B swizzle).  Diagnostic
// only; results go to profiles/.  Build: see tests/cpp/Makefile (mma_microbench).
#include <cstdio>
#include <cstdint>
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

int main() {
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
    return 0;
}
