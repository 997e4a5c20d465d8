// mlp.cuh — BMLP1 integer MLP ensemble on tcgen05 tensor cores (see mlp.cu).
#pragma once
#include <atomic>
#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "launch_spec.cuh"
#include "pdb.cuh"

namespace bida_gpu {

struct MlpModel;

struct MlpShape {
    int F = 0, C = 0, E = 0, L = 0;
    int H[8] = {0};
};

// Parses a BMLP1 image, uploads it to the current device; returns a
// bida_status (0 = OK) and fills *err on failure.
int mlp_create(const unsigned char *blob, size_t len, int F, double thr, int num_sms,
               MlpModel **out, MlpShape *shape, std::string *err);
// Enqueues the fused encode + MLP + readout on `st`; returns 0 or nonzero
// (message in mlp_last_error()).
int mlp_launch(MlpModel *m, int domain, const void *d_packed, int64_t n, int32_t *d_h,
               double *d_logits, int *err_dev, unsigned long long *replays, cudaStream_t st,
               std::atomic<int64_t> *launches, const PdbArgs *pdb = nullptr);
// The same launch as data for graph replay; returns 0 when the model's
// schedule is one plain kernel launch (fused schedules without clusters), 1
// otherwise (wide schedule: scratch-pool ordering; CTA pairs).
int mlp_prepare(MlpModel *m, int domain, const void *d_packed, int64_t n, int32_t *d_h, int *err_dev,
                unsigned long long *replays, const PdbArgs *pdb, KernelLaunch *out);
void mlp_destroy(MlpModel *m);
// Debug: record a per-warp clock64 timeline of CTA 0 into dev_buf ([10 warps][mlp_trace_slots()]).
void mlp_set_trace(MlpModel *m, long long *dev_buf);
int mlp_trace_slots();
const char *mlp_last_error();

} // namespace bida_gpu
