// launch_spec.cuh — one kernel launch described as data (function, grid,
// block, dynamic shared memory, its single by-value argument struct), so the
// zero-copy lanes can replay it from a per-lane CUDA graph
// (bida_gpu.cu lane_launch) instead of a stream launch.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstring>

namespace bida_gpu {

struct KernelLaunch {
    const void *func = nullptr;
    dim3 grid, block;
    size_t smem = 0;
    alignas(16) unsigned char args[4096];
    size_t args_size = 0;
    void *argv[1] = {nullptr};

    template <class A>
    void set_args(const A &a) {
        static_assert(sizeof(A) <= sizeof(args), "kernel argument struct too large");
        std::memcpy(args, &a, sizeof(A));
        args_size = sizeof(A);
        argv[0] = args;
    }
};

} // namespace bida_gpu
