// common.cuh — shared constants for the sm_100a evaluator kernels.
#pragma once
#include <cstdint>

namespace bida_gpu {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kSTP2 = 2, kSTP3 = 3, kSTP4 = 4, kRC = 100;

// Per-launch error flags: err[k] = 1 (plain idempotent store) into a small
// mapped host array, one word per kind; decoded into bida_status by the host.
constexpr int kErrDistribution = 0; // ClassDistribution::validate would throw
constexpr int kErrState = 1;        // packed state encodes outside [0, F)
constexpr int kErrWords = 4;

__device__ __forceinline__ void raise_error(int *err, int kind) {
    reinterpret_cast<volatile int *>(err)[kind] = 1;
}

constexpr int kMaxClasses = 256;    // 8 class slots per lane

// Threshold of quantile_class: cum >= q - 1e-12 (heuristic.hpp:116).
struct Readout {
    double thr;   // q - 1e-12, computed on the host exactly as the reference does
    int classes;  // C
};

} // namespace bida_gpu
