// bida_gpu.cu — host side of the C-ABI (include/bida_gpu.h) and kernel
// dispatch.  One handle = one model resident on one device, plus a pair of
// pinned staging slots and streams so host<->device copies of chunk i+1
// overlap the kernel of chunk i.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing without a tool attached

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bida_gpu.h"
#include "common.cuh"
#include "linear.cuh"
#include "linear_thread.cuh"
#include "mlp.cuh"
#include "pdb.cuh"

using namespace bida_gpu;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                             \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return fail(BIDA_ERR_CUDA, std::string(#expr " failed: ") + cudaGetErrorString(e_)); \
    } while (0)

int feature_length(int domain) {
    switch (domain) {
    case BIDA_DOMAIN_STP2: return 16;
    case BIDA_DOMAIN_STP3: return 81;
    case BIDA_DOMAIN_STP4: return 256;
    case BIDA_DOMAIN_RC: return 480;
    default: return -1;
    }
}
int packed_bytes(int domain) {
    if (domain == BIDA_DOMAIN_RC)
        return 16;
    return feature_length(domain) > 0 ? 8 : -1;
}

} // namespace

namespace bida_gpu {
std::string &last_error_ref() { return g_last_error; }
int pdb_build_device(int domain, const uint8_t *pattern, int m, uint8_t **d_out, uint64_t *n_out);
} // namespace bida_gpu

// Host<->device pipelining of large batches: kSlots chunks of up to kMaxSlot
// states in flight on kSlots streams, so the H2D copy of chunk i+1.. overlaps
// the kernel of chunk i and the D2H of chunk i-1 (copy engines are full duplex).
constexpr int kSlots = 4;
constexpr int kZcLanes = 8;
// Error channels: each zero-copy lane, the pipelined path and the device path
// own kErrWords mapped words, so a bad state in one call is reported by that
// call only (concurrent agents share a handle).
constexpr int kChanPipe = kZcLanes;
constexpr int kChanDevice = kZcLanes + 1;
constexpr int kChannels = kZcLanes + 2;

struct bida_gpu_evaluator {
    int kind = 0, domain = 0, F = 0, C = 0, E = 0, device = 0;
    double q = 0.5, thr = 0.0;
    float uLo = 0.0f, uHi = 0.0f;
    int num_sms = 148;

    // linear model: thread-per-state kernel (linear_thread.cuh) when C <= 96
    // and every weight is finite, else the warp-per-state kernel (linear.cuh)
    bool lin_thread = false;
    float *d_Wthr = nullptr;  // [E][F+1][Cp]
    int Cp = 0, lin_cm = 0;
    float *d_Wt = nullptr;
    uint8_t *d_rowflag = nullptr;
    int any_rowflag = 0;
    int w_in_smem = 0;
    size_t lin_smem = 0;
    int lin_grid_cap = 0;
    unsigned long long *d_replays = nullptr;  // readouts that took the exact float64 replay

    // MLP model
    MlpModel *mlp = nullptr;
    int hidden_layers = 0;
    int hidden[8] = {0};

    std::mutex mu;
    cudaStream_t stream[kSlots] = {};
    cudaEvent_t done[kSlots] = {};
    int64_t slot_cap = 0;
    void *h_in[kSlots] = {};
    int32_t *h_h[kSlots] = {};
    void *d_in[kSlots] = {};
    int32_t *d_h[kSlots] = {};
    int *err_host = nullptr; // mapped pinned, kChannels x kErrWords ints
    int *err_dev = nullptr;
    // small-batch zero-copy path: mapped pinned in/out read/written by the
    // kernel, kZcLanes independent lanes (own lock, stream and buffers) so
    // concurrent callers on one handle (the ring evaluator's agents,
    // include/bida_ring_evaluator.hpp) keep several batches on the device
    // A lane is owned by one call at a time (busy flag); the asynchronous
    // submit / wait pair (bida_gpu_submit) keeps it across calls.
    struct ZcLane {
        std::atomic<int> busy{0};
        cudaStream_t st = nullptr;
        cudaEvent_t done = nullptr;
        void *in = nullptr, *in_dev = nullptr;
        int32_t *out = nullptr, *out_dev = nullptr;
        int64_t n = 0;
        bida_gpu_evaluator *owner = nullptr;
        // one-kernel graph replayed for every launch on this lane
        // (lane_launch); the node's parameters are rewritten per call
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t gexec = nullptr;
        cudaGraphNode_t gnode = nullptr;
        const void *gfunc = nullptr;
    } zc[kZcLanes];
    std::atomic<int64_t> graph_launches{0};
    std::atomic<unsigned> zc_next{0};
    std::mutex err_mu;
    std::atomic<int64_t> zc_calls{0};
    // PDB correction (bida_gpu_attach_pdb)
    uint8_t *d_pdb = nullptr;
    PdbArgs pdb{};
    std::atomic<int64_t> launches{0};
};

namespace {

constexpr int64_t kMaxSlotDefault = int64_t(1) << 18;
constexpr int64_t kMinChunk = int64_t(1) << 16;
// BIDA_GPU_CHUNK_LOG2 (experiments): largest pipelined chunk 2^k states, 12..22
int64_t max_slot() {
    static const int64_t v = [] {
        const char *s = std::getenv("BIDA_GPU_CHUNK_LOG2");
        const int k = s ? std::atoi(s) : 0;
        return k >= 12 && k <= 22 ? int64_t(1) << k : kMaxSlotDefault;
    }();
    return v;
}
// Pipelined chunk for `remaining` states: the slot capacity (2^18 states, the
// measured best: profiles/r2_e2e_chunks.jsonl) while at least twice that
// remains, then halving down to kMinChunk, so the last kernel + D2H, which no
// H2D copy overlaps, is short: e2e 2.86 -> 2.94 G evals/s (h128, 4 M states).
// Larger caps lose (2^20: 2.65 G) although bigger copies alone move faster.
// BIDA_GPU_CHUNK_FIXED=1: fixed chunks.
int64_t chunk_for(int64_t remaining, int64_t cap) {
    static const bool fixed = [] {
        const char *s = std::getenv("BIDA_GPU_CHUNK_FIXED");
        return s && s[0] == '1';
    }();
    int64_t c = cap;
    if (!fixed)
        while (c > kMinChunk && c * 2 > remaining)
            c >>= 1;
    return std::min(c, remaining);
}
// Batches up to this size skip the copy engines: the kernel reads the packed
// states from mapped pinned memory and writes h straight back into it (one
// launch + one stream sync per call; search batches are 1-8K states).
constexpr int64_t kZeroCopyMax = int64_t(1) << 15;
// linear thread kernel: at or below this many states the weights are not
// staged in shared memory (profiles/r2_latency_breakdown_linear.jsonl)
constexpr int64_t kLinSmallBatch = int64_t(1) << 12;

template <int DOMAIN, int CS>
int launch_linear_t(bida_gpu_evaluator *ev, const LinearArgs &a, cudaStream_t st) {
    const int64_t groups = (a.n + 31) / 32;
    const int64_t want = (groups + kLinearWarps - 1) / kLinearWarps;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, ev->lin_grid_cap)));
    linear_eval_kernel<DOMAIN, CS><<<grid, kLinearThreads, ev->lin_smem, st>>>(a);
    ev->launches.fetch_add(1, std::memory_order_relaxed);
    CUDA_TRY(cudaGetLastError());
    return BIDA_OK;
}

template <int DOMAIN>
int launch_linear_d(bida_gpu_evaluator *ev, const LinearArgs &a, cudaStream_t st) {
    const int cs = (ev->C + 31) / 32;
    switch (cs) {
    case 1: return launch_linear_t<DOMAIN, 1>(ev, a, st);
    case 2: return launch_linear_t<DOMAIN, 2>(ev, a, st);
    case 3: return launch_linear_t<DOMAIN, 3>(ev, a, st);
    case 4: return launch_linear_t<DOMAIN, 4>(ev, a, st);
    default: return launch_linear_t<DOMAIN, 8>(ev, a, st);
    }
}

// Thread-per-state linear kernel (linear_thread.cuh): one instantiation per
// (domain, class-slot count).
template <int DOMAIN, int CM>
void *linear_thread_fn() {
    return reinterpret_cast<void *>(linear_thread_kernel<DOMAIN, CM>);
}

template <int DOMAIN>
void *linear_thread_fn_cm(int cm) {
    switch (cm) {
    case 8: return linear_thread_fn<DOMAIN, 8>();
    case 16: return linear_thread_fn<DOMAIN, 16>();
    case 24: return linear_thread_fn<DOMAIN, 24>();
    case 32: return linear_thread_fn<DOMAIN, 32>();
    case 64: return linear_thread_fn<DOMAIN, 64>();
    default: return linear_thread_fn<DOMAIN, 96>();
    }
}

void *linear_thread_kernel_for(int domain, int cm) {
    switch (domain) {
    case BIDA_DOMAIN_STP2: return linear_thread_fn_cm<kSTP2>(cm);
    case BIDA_DOMAIN_STP3: return linear_thread_fn_cm<kSTP3>(cm);
    case BIDA_DOMAIN_STP4: return linear_thread_fn_cm<kSTP4>(cm);
    default: return linear_thread_fn_cm<kRC>(cm);
    }
}

void prepare_linear_thread(bida_gpu_evaluator *ev, const void *d_packed, int64_t n, int32_t *d_h,
                           double *d_logits, int *err, KernelLaunch *kl) {
    LinearThreadArgs a;
    a.packed = d_packed;
    a.n = n;
    a.h_out = d_h;
    a.logits_out = d_logits;
    a.W = ev->d_Wthr;
    a.E = ev->E;
    a.C = ev->C;
    a.Cp = ev->Cp;
    a.rk.thr = ev->thr;
    a.rk.uLo = ev->uLo;
    a.rk.uHi = ev->uHi;
    // small batches (the search's zero-copy regime) read the weights through
    // L1/L2 instead of staging the whole table into every CTA's shared memory
    const bool small = n <= kLinSmallBatch;
    a.w_in_smem = small ? 0 : ev->w_in_smem;
    a.err = err;
    a.replays = ev->d_replays;
    a.pdb = ev->pdb;
    if (!ev->d_pdb)
        a.pdb.entries = nullptr;
    const int64_t want = (n + kLinThreads - 1) / kLinThreads;
    kl->func = linear_thread_kernel_for(ev->domain, ev->lin_cm);
    kl->grid = dim3(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, ev->lin_grid_cap))));
    kl->block = dim3(kLinThreads);
    kl->smem = small ? 0 : ev->lin_smem;
    kl->set_args(a);
}

int launch_linear_thread(bida_gpu_evaluator *ev, const void *d_packed, int64_t n, int32_t *d_h,
                         double *d_logits, cudaStream_t st, int *err) {
    KernelLaunch kl;
    prepare_linear_thread(ev, d_packed, n, d_h, d_logits, err, &kl);
    CUDA_TRY(cudaLaunchKernel(kl.func, kl.grid, kl.block, kl.argv, kl.smem, st));
    ev->launches.fetch_add(1, std::memory_order_relaxed);
    return BIDA_OK;
}

int launch(bida_gpu_evaluator *ev, const void *d_packed, int64_t n, int32_t *d_h, double *d_logits,
           cudaStream_t st, int *err) {
    if (n <= 0)
        return BIDA_OK;
    if (ev->kind == BIDA_MODEL_MLP)
        return mlp_launch(ev->mlp, ev->domain, d_packed, n, d_h, d_logits, err, ev->d_replays, st,
                          &ev->launches, ev->d_pdb ? &ev->pdb : nullptr)
                   ? fail(BIDA_ERR_CUDA, mlp_last_error())
                   : BIDA_OK;
    if (ev->lin_thread)
        return launch_linear_thread(ev, d_packed, n, d_h, d_logits, st, err);
    LinearArgs a;
    a.packed = d_packed;
    a.n = n;
    a.h_out = d_h;
    a.logits_out = d_logits;
    a.Wt = ev->d_Wt;
    a.rowflag = ev->d_rowflag;
    a.E = ev->E;
    a.C = ev->C;
    a.thr = ev->thr;
    a.uLo = ev->uLo;
    a.uHi = ev->uHi;
    a.w_in_smem = ev->w_in_smem;
    a.any_rowflag = ev->any_rowflag;
    a.err = err;
    a.replays = ev->d_replays;
    a.pdb = ev->pdb;
    if (!ev->d_pdb)
        a.pdb.entries = nullptr;
    switch (ev->domain) {
    case BIDA_DOMAIN_STP2: return launch_linear_d<kSTP2>(ev, a, st);
    case BIDA_DOMAIN_STP3: return launch_linear_d<kSTP3>(ev, a, st);
    case BIDA_DOMAIN_STP4: return launch_linear_d<kSTP4>(ev, a, st);
    default: return launch_linear_d<kRC>(ev, a, st);
    }
}

int *chan_err(bida_gpu_evaluator *ev, int ch) { return ev->err_dev + ch * kErrWords; }

// BIDA_GPU_GRAPHS=0 turns the lane graphs off (A/B, debugging)
bool graphs_enabled() {
    static const bool on = [] {
        const char *s = std::getenv("BIDA_GPU_GRAPHS");
        return !(s && s[0] == '0');
    }();
    return on;
}

void drop_lane_graph(bida_gpu_evaluator::ZcLane *ln) {
    if (ln->gexec) cudaGraphExecDestroy(ln->gexec);
    if (ln->graph) cudaGraphDestroy(ln->graph);
    ln->gexec = nullptr;
    ln->graph = nullptr;
    ln->gnode = nullptr;
    ln->gfunc = nullptr;
}

// One launch on a zero-copy lane. The lane's buffers never move, so the
// launch is a one-node CUDA graph built at the lane's first use and replayed
// afterwards with the node's parameters (n, grid, PDB, the argument struct)
// rewritten in place: cudaGraphLaunch of an updated exec costs ~3.5 us less
// per call than cudaLaunchKernel + the launch's own bookkeeping on the
// search's small batches (profiles/r2_latency_breakdown_graph.jsonl).
// Schedules that are not one plain launch (the wide MLP's scratch pool,
// CTA-pair clusters, the warp-per-state linear kernel) launch directly.
int lane_launch(bida_gpu_evaluator *ev, bida_gpu_evaluator::ZcLane *ln, int64_t n, int ch) {
    if (n <= 0)
        return BIDA_OK;
    KernelLaunch kl;
    bool graphable = false;
    if (graphs_enabled()) {
        if (ev->kind == BIDA_MODEL_MLP)
            graphable = mlp_prepare(ev->mlp, ev->domain, ln->in_dev, n, ln->out_dev, chan_err(ev, ch),
                                    ev->d_replays, ev->d_pdb ? &ev->pdb : nullptr, &kl) == 0;
        else if (ev->lin_thread) {
            prepare_linear_thread(ev, ln->in_dev, n, ln->out_dev, nullptr, chan_err(ev, ch), &kl);
            graphable = true;
        }
    }
    if (!graphable)
        return launch(ev, ln->in_dev, n, ln->out_dev, nullptr, ln->st, chan_err(ev, ch));
    cudaKernelNodeParams kp = {};
    kp.func = const_cast<void *>(kl.func);
    kp.gridDim = kl.grid;
    kp.blockDim = kl.block;
    kp.sharedMemBytes = static_cast<unsigned>(kl.smem);
    kp.kernelParams = kl.argv;
    kp.extra = nullptr;
    cudaError_t e = cudaSuccess;
    if (ln->gexec && ln->gfunc == kl.func) {
        e = cudaGraphExecKernelNodeSetParams(ln->gexec, ln->gnode, &kp);
    } else {
        drop_lane_graph(ln);
        e = cudaGraphCreate(&ln->graph, 0);
        if (e == cudaSuccess)
            e = cudaGraphAddKernelNode(&ln->gnode, ln->graph, nullptr, 0, &kp);
        if (e == cudaSuccess)
            e = cudaGraphInstantiate(&ln->gexec, ln->graph, 0);
        if (e == cudaSuccess)
            ln->gfunc = kl.func;
    }
    if (e == cudaSuccess)
        e = cudaGraphLaunch(ln->gexec, ln->st);
    if (e != cudaSuccess) {
        // a graph-path failure is not fatal: drop the graph, clear the
        // sticky-free error and launch directly
        drop_lane_graph(ln);
        (void)cudaGetLastError();
        return launch(ev, ln->in_dev, n, ln->out_dev, nullptr, ln->st, chan_err(ev, ch));
    }
    ev->launches.fetch_add(1, std::memory_order_relaxed);
    ev->graph_launches.fetch_add(1, std::memory_order_relaxed);
    return BIDA_OK;
}

// First free zero-copy lane from a rotating start; spins (then yields) while
// every lane is busy.
bida_gpu_evaluator::ZcLane *acquire_lane(bida_gpu_evaluator *ev) {
    const unsigned start = ev->zc_next.fetch_add(1, std::memory_order_relaxed);
    for (unsigned spins = 0;; ++spins) {
        for (int k = 0; k < kZcLanes; ++k) {
            auto &cand = ev->zc[(start + k) % kZcLanes];
            int idle = 0;
            if (cand.busy.load(std::memory_order_relaxed) == 0 &&
                cand.busy.compare_exchange_strong(idle, 1, std::memory_order_acquire))
                return &cand;
        }
        if (spins > 64)
            std::this_thread::yield();
    }
}
void release_lane(bida_gpu_evaluator::ZcLane *ln) { ln->busy.store(0, std::memory_order_release); }

// Exclusive use of the whole handle (PDB attach): the pipelined path's mutex
// plus every lane.
struct HandleLock {
    explicit HandleLock(bida_gpu_evaluator *e) : ev(e), lk(e->mu) {
        for (auto &ln : ev->zc) {
            int idle = 0;
            while (!ln.busy.compare_exchange_weak(idle, 1, std::memory_order_acquire)) {
                idle = 0;
                std::this_thread::yield();
            }
        }
    }
    ~HandleLock() {
        for (auto &ln : ev->zc)
            release_lane(&ln);
    }
    bida_gpu_evaluator *ev;
    std::lock_guard<std::mutex> lk;
};

// Decodes and clears one channel's error words.  Channels other than the
// device path are owned by the call holding their lock; the device path's
// words may be collected by any thread (bida_gpu_stream_status).
int collect_errors(bida_gpu_evaluator *ev, int ch) {
    std::unique_lock<std::mutex> lk(ev->err_mu, std::defer_lock);
    if (ch == kChanDevice)
        lk.lock();
    volatile int *e = ev->err_host + ch * kErrWords;
    int rc = BIDA_OK;
    if (e[kErrState])
        rc = fail(BIDA_ERR_STATE, "packed state encodes a feature outside [0, F)");
    else if (e[kErrDistribution])
        rc = fail(BIDA_ERR_DISTRIBUTION, "ClassDistribution: probabilities must sum to 1");
    for (int k = 0; k < kErrWords; ++k)
        e[k] = 0;
    return rc;
}

int ensure_slots(bida_gpu_evaluator *ev, int64_t n) {
    const int64_t want = std::min<int64_t>(std::max<int64_t>(n, 1024), max_slot());
    if (ev->slot_cap >= want)
        return BIDA_OK;
    int64_t cap = 1024;
    while (cap < want)
        cap <<= 1;
    const int pb = packed_bytes(ev->domain);
    for (int s = 0; s < kSlots; ++s) {
        if (ev->h_in[s]) cudaFreeHost(ev->h_in[s]);
        if (ev->h_h[s]) cudaFreeHost(ev->h_h[s]);
        if (ev->d_in[s]) cudaFree(ev->d_in[s]);
        if (ev->d_h[s]) cudaFree(ev->d_h[s]);
        ev->h_in[s] = ev->h_h[s] = nullptr;
        ev->d_in[s] = ev->d_h[s] = nullptr;
        CUDA_TRY(cudaHostAlloc(&ev->h_in[s], cap * pb, cudaHostAllocDefault));
        CUDA_TRY(cudaHostAlloc(reinterpret_cast<void **>(&ev->h_h[s]), cap * 4, cudaHostAllocDefault));
        CUDA_TRY(cudaMalloc(&ev->d_in[s], cap * pb));
        CUDA_TRY(cudaMalloc(reinterpret_cast<void **>(&ev->d_h[s]), cap * 4));
    }
    ev->slot_cap = cap;
    return BIDA_OK;
}

int common_init(bida_gpu_evaluator *ev, int device) {
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "device index out of range");
    ev->device = device;
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(BIDA_ERR_CUDA, std::string("this library is built for sm_100a (B200); device is ") +
                                       prop.name);
    ev->num_sms = prop.multiProcessorCount;
    for (int s = 0; s < kSlots; ++s) {
        CUDA_TRY(cudaStreamCreateWithFlags(&ev->stream[s], cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&ev->done[s], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaHostAlloc(reinterpret_cast<void **>(&ev->err_host), kChannels * kErrWords * sizeof(int),
                           cudaHostAllocMapped));
    std::memset(ev->err_host, 0, kChannels * kErrWords * sizeof(int));
    CUDA_TRY(cudaMalloc(reinterpret_cast<void **>(&ev->d_replays), sizeof(unsigned long long)));
    CUDA_TRY(cudaMemset(ev->d_replays, 0, sizeof(unsigned long long)));
    CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void **>(&ev->err_dev), ev->err_host, 0));
    for (auto &ln : ev->zc) {
        ln.owner = ev;
        CUDA_TRY(cudaEventCreateWithFlags(&ln.done, cudaEventDisableTiming));
        CUDA_TRY(cudaStreamCreateWithFlags(&ln.st, cudaStreamNonBlocking));
        CUDA_TRY(cudaHostAlloc(&ln.in, kZeroCopyMax * 16, cudaHostAllocMapped | cudaHostAllocWriteCombined));
        CUDA_TRY(cudaHostGetDevicePointer(&ln.in_dev, ln.in, 0));
        CUDA_TRY(cudaHostAlloc(reinterpret_cast<void **>(&ln.out), kZeroCopyMax * 4, cudaHostAllocMapped));
        CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void **>(&ln.out_dev), ln.out, 0));
    }
    return BIDA_OK;
}

void release(bida_gpu_evaluator *ev) {
    if (!ev)
        return;
    cudaSetDevice(ev->device);
    for (int s = 0; s < kSlots; ++s) {
        if (ev->stream[s]) cudaStreamSynchronize(ev->stream[s]);
        if (ev->h_in[s]) cudaFreeHost(ev->h_in[s]);
        if (ev->h_h[s]) cudaFreeHost(ev->h_h[s]);
        if (ev->d_in[s]) cudaFree(ev->d_in[s]);
        if (ev->d_h[s]) cudaFree(ev->d_h[s]);
        if (ev->done[s]) cudaEventDestroy(ev->done[s]);
        if (ev->stream[s]) cudaStreamDestroy(ev->stream[s]);
    }
    if (ev->err_host) cudaFreeHost(ev->err_host);
    for (auto &ln : ev->zc) {
        if (ln.st) cudaStreamSynchronize(ln.st);
        drop_lane_graph(&ln);
        if (ln.done) cudaEventDestroy(ln.done);
        if (ln.in) cudaFreeHost(ln.in);
        if (ln.out) cudaFreeHost(ln.out);
        if (ln.st) cudaStreamDestroy(ln.st);
    }
    if (ev->d_Wt) cudaFree(ev->d_Wt);
    if (ev->d_Wthr) cudaFree(ev->d_Wthr);
    if (ev->d_replays) cudaFree(ev->d_replays);
    if (ev->d_rowflag) cudaFree(ev->d_rowflag);
    if (ev->d_pdb) cudaFree(ev->d_pdb);
    if (ev->mlp) mlp_destroy(ev->mlp);
    delete ev;
}

bool direct_enabled() {
    static const bool on = [] {
        const char *s = std::getenv("BIDA_GPU_DIRECT");
        return !(s && s[0] == '0');
    }();
    return on;
}

bool is_pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

int check_quantile(double q) {
    if (!(q > 0.0 && q <= 1.0))
        return fail(BIDA_ERR_INVALID_ARGUMENT, "quantile_class: q must be in (0, 1]");
    return BIDA_OK;
}

bool read_file(const char *path, std::vector<unsigned char> &out) {
    std::ifstream f(path, std::ios::binary);
    if (!f)
        return false;
    out.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
    return true;
}

uint32_t rd_u32(const unsigned char *b) {
    return uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 | uint32_t(b[3]) << 24;
}

int linear_create_impl(int device, int domain, const float *weights, int E, int C, double q,
                       bida_gpu_evaluator **out) {
    if (!out)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "out handle pointer is NULL");
    *out = nullptr;
    const int F = feature_length(domain);
    if (F < 0)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "unknown domain");
    if (E <= 0)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "LinearModelBackend: empty ensemble");
    if (C <= 0)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "LinearModelBackend: need at least one class");
    if (C > kMaxClasses)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "classes > 256 are not supported by the GPU readout");
    if (!weights)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "LinearModelBackend: weight matrix size mismatch");
    if (int rc = check_quantile(q))
        return rc;

    auto *ev = new bida_gpu_evaluator();
    ev->kind = BIDA_MODEL_LINEAR;
    ev->domain = domain;
    ev->F = F;
    ev->C = C;
    ev->E = E;
    ev->q = q;
    ev->thr = q - 1e-12;
    {
        const double u = 1.0 - ev->thr, eps64 = (4.0 * C + 16.0) * std::ldexp(1.0, -53);
        ev->uLo = std::nextafter(static_cast<float>(u - eps64), 0.0f);
        ev->uHi = std::nextafter(static_cast<float>(u + eps64), INFINITY);
    }
    if (int rc = common_init(ev, device)) {
        release(ev);
        return rc;
    }
    // Transpose [E][C][F] -> [E][F][C] so class lanes read consecutive floats.
    const size_t nw = static_cast<size_t>(E) * F * C;
    std::vector<float> wt(nw);
    std::vector<uint8_t> flag(static_cast<size_t>(E) * C, 0);
    for (int m = 0; m < E; ++m)
        for (int c = 0; c < C; ++c)
            for (int j = 0; j < F; ++j) {
                const float w = weights[(static_cast<size_t>(m) * C + c) * F + j];
                wt[(static_cast<size_t>(m) * F + j) * C + c] = w;
                if (!std::isfinite(w)) {
                    flag[static_cast<size_t>(m) * C + c] = 1;
                    ev->any_rowflag = 1;
                }
            }
    auto bail = [&](int rc) {
        release(ev);
        return rc;
    };
    if (C > kLinMaxClasses || ev->any_rowflag) {  // warp-per-state kernel's layout
        cudaError_t e = cudaMalloc(&ev->d_Wt, nw * sizeof(float));
        if (e == cudaSuccess)
            e = cudaMemcpy(ev->d_Wt, wt.data(), nw * sizeof(float), cudaMemcpyHostToDevice);
        if (e == cudaSuccess)
            e = cudaMalloc(&ev->d_rowflag, flag.size());
        if (e == cudaSuccess)
            e = cudaMemcpy(ev->d_rowflag, flag.data(), flag.size(), cudaMemcpyHostToDevice);
        if (e != cudaSuccess)
            return bail(fail(BIDA_ERR_CUDA, std::string("weight upload: ") + cudaGetErrorString(e)));
    }
    if (C <= kLinMaxClasses && !ev->any_rowflag) {
        // thread-per-state kernel: [E][F+1][Cp], zero pad columns and a zero row F
        ev->lin_thread = true;
        // row stride in 16-byte chunks made odd: the quarter-warp of a
        // float4 load then spreads over all 8 bank groups (an even stride
        // reaches only 4; profiles/r2_linear.txt: 72% LSU wavefront load)
        ev->Cp = (C + 3) & ~3;
        if ((ev->Cp / 4) % 2 == 0)
            ev->Cp += 4;
        ev->lin_cm = C <= 8 ? 8 : C <= 16 ? 16 : C <= 24 ? 24 : C <= 32 ? 32 : C <= 64 ? 64 : 96;
        const size_t per = static_cast<size_t>(F + 1) * ev->Cp;
        std::vector<float> w3(per * E, 0.0f);
        for (int m = 0; m < E; ++m)
            for (int c = 0; c < C; ++c)
                for (int j = 0; j < F; ++j)
                    w3[m * per + static_cast<size_t>(j) * ev->Cp + c] =
                        weights[(static_cast<size_t>(m) * C + c) * F + j];
        cudaError_t e = cudaMalloc(&ev->d_Wthr, w3.size() * sizeof(float));
        if (e == cudaSuccess)
            e = cudaMemcpy(ev->d_Wthr, w3.data(), w3.size() * sizeof(float), cudaMemcpyHostToDevice);
        if (e != cudaSuccess)
            return bail(fail(BIDA_ERR_CUDA, std::string("weight upload: ") + cudaGetErrorString(e)));
        const size_t wbytes = w3.size() * sizeof(float);
        ev->w_in_smem = wbytes <= 200 * 1024 ? 1 : 0;
        ev->lin_smem = ev->w_in_smem ? wbytes : 0;
        void *fn = linear_thread_kernel_for(domain, ev->lin_cm);
        if (ev->lin_smem > 48 * 1024) {
            e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ev->lin_smem));
            if (e != cudaSuccess)
                return bail(fail(BIDA_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e)));
        }
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kLinThreads, ev->lin_smem);
        if (e != cudaSuccess || per_sm < 1)
            return bail(fail(BIDA_ERR_CUDA, "linear kernel does not fit on an SM"));
        ev->lin_grid_cap = ev->num_sms * per_sm;
        *out = ev;
        return BIDA_OK;
    }
    const int cpad = (C + 1) & ~1;
    const size_t extra = static_cast<size_t>(kLinearWarps) * cpad * 8 + kLinearWarps * 32 * 4;
    const size_t wbytes = (nw * 4 + 15) & ~size_t(15);
    ev->w_in_smem = (wbytes + extra <= 200 * 1024) ? 1 : 0;
    ev->lin_smem = (ev->w_in_smem ? wbytes : 0) + extra;
    if (ev->lin_smem > 48 * 1024) {
        // once per handle (the kernel instance depends on the domain and C)
        cudaError_t e = cudaSuccess;
        switch (domain) {
#define BIDA_SET_ATTR(D)                                                                                   \
    e = [&] {                                                                                              \
        const int cs = (C + 31) / 32;                                                                      \
        const void *fn = cs == 1   ? reinterpret_cast<const void *>(linear_eval_kernel<D, 1>)              \
                         : cs == 2 ? reinterpret_cast<const void *>(linear_eval_kernel<D, 2>)              \
                         : cs == 3 ? reinterpret_cast<const void *>(linear_eval_kernel<D, 3>)              \
                         : cs == 4 ? reinterpret_cast<const void *>(linear_eval_kernel<D, 4>)              \
                                   : reinterpret_cast<const void *>(linear_eval_kernel<D, 8>);             \
        return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,                      \
                                    static_cast<int>(ev->lin_smem));                                       \
    }();                                                                                                   \
    break;
        case BIDA_DOMAIN_STP2: BIDA_SET_ATTR(kSTP2)
        case BIDA_DOMAIN_STP3: BIDA_SET_ATTR(kSTP3)
        case BIDA_DOMAIN_STP4: BIDA_SET_ATTR(kSTP4)
        default: BIDA_SET_ATTR(kRC)
#undef BIDA_SET_ATTR
        }
        if (e != cudaSuccess)
            return bail(fail(BIDA_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e)));
    }
    // Resident CTAs per SM from the smem budget (228 KB/SM, 1 KB reserved per CTA).
    const size_t per_cta = ev->lin_smem + 1024;
    int per_sm = static_cast<int>(std::min<size_t>(8, (228 * 1024) / per_cta));
    per_sm = std::max(per_sm, 1);
    ev->lin_grid_cap = ev->num_sms * per_sm;
    *out = ev;
    return BIDA_OK;
}

int parse_blin1(const unsigned char *b, size_t len, int F, const std::string &name,
                std::vector<float> &w, int &C, int &E) {
    if (len < 5 || std::memcmp(b, "BLIN1", 5) != 0)
        return fail(BIDA_ERR_RUNTIME, "not a BLIN1 file: " + name);
    if (len < 17)
        return fail(BIDA_ERR_RUNTIME, "BLIN1 header does not match domain: " + name);
    const uint32_t flen = rd_u32(b + 5), classes = rd_u32(b + 9), ens = rd_u32(b + 13);
    if (flen != static_cast<uint32_t>(F) || ens == 0)
        return fail(BIDA_ERR_RUNTIME, "BLIN1 header does not match domain: " + name);
    const size_t count = static_cast<size_t>(flen) * classes * ens;
    if (len < 17 + count * 4)
        return fail(BIDA_ERR_RUNTIME, "truncated BLIN1 file: " + name);
    w.resize(count);
    std::memcpy(w.data(), b + 17, count * 4);
    C = static_cast<int>(classes);
    E = static_cast<int>(ens);
    return BIDA_OK;
}

} // namespace

extern "C" {

int bida_gpu_abi_version(void) { return BIDA_GPU_ABI_VERSION; }
const char *bida_gpu_last_error(void) { return g_last_error.c_str(); }

int bida_gpu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess)
        return 0;
    return n;
}

int bida_gpu_feature_length(int domain) { return feature_length(domain); }
int bida_gpu_packed_bytes(int domain) { return packed_bytes(domain); }

int bida_gpu_linear_create(int device, int domain, const float *weights, int ensemble, int classes,
                           double quantile, bida_gpu_evaluator **out) {
    return linear_create_impl(device, domain, weights, ensemble, classes, quantile, out);
}

int bida_gpu_linear_create_blin1(int device, int domain, const void *blob, size_t len,
                                 double quantile, bida_gpu_evaluator **out) {
    if (out)
        *out = nullptr;
    const int F = feature_length(domain);
    if (F < 0)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "unknown domain");
    std::vector<float> w;
    int C = 0, E = 0;
    if (int rc = parse_blin1(static_cast<const unsigned char *>(blob), blob ? len : 0, F,
                             "<memory>", w, C, E))
        return rc;
    return linear_create_impl(device, domain, w.data(), E, C, quantile, out);
}

int bida_gpu_linear_load(int device, int domain, const char *path, double quantile,
                         bida_gpu_evaluator **out) {
    if (out)
        *out = nullptr;
    const int F = feature_length(domain);
    if (F < 0)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "unknown domain");
    std::vector<unsigned char> buf;
    if (!path || !read_file(path, buf))
        return fail(BIDA_ERR_RUNTIME, std::string("cannot open weights file: ") + (path ? path : ""));
    std::vector<float> w;
    int C = 0, E = 0;
    if (int rc = parse_blin1(buf.data(), buf.size(), F, path, w, C, E))
        return rc;
    return linear_create_impl(device, domain, w.data(), E, C, quantile, out);
}

int bida_gpu_mlp_create_bmlp1(int device, int domain, const void *blob, size_t len,
                              double quantile, bida_gpu_evaluator **out) {
    if (!out)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "out handle pointer is NULL");
    *out = nullptr;
    const int F = feature_length(domain);
    if (F < 0)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "unknown domain");
    if (int rc = check_quantile(quantile))
        return rc;
    auto *ev = new bida_gpu_evaluator();
    ev->kind = BIDA_MODEL_MLP;
    ev->domain = domain;
    ev->F = F;
    ev->q = quantile;
    ev->thr = quantile - 1e-12;
    if (int rc = common_init(ev, device)) {
        release(ev);
        return rc;
    }
    MlpShape shape;
    std::string err;
    const int rc = mlp_create(static_cast<const unsigned char *>(blob), blob ? len : 0, F,
                              ev->thr, ev->num_sms, &ev->mlp, &shape, &err);
    if (rc) {
        release(ev);
        return fail(rc, err);
    }
    ev->C = shape.C;
    ev->E = shape.E;
    ev->hidden_layers = shape.L;
    for (int l = 0; l < shape.L && l < 8; ++l)
        ev->hidden[l] = shape.H[l];
    *out = ev;
    return BIDA_OK;
}

int bida_gpu_mlp_load(int device, int domain, const char *path, double quantile,
                      bida_gpu_evaluator **out) {
    if (out)
        *out = nullptr;
    std::vector<unsigned char> buf;
    if (!path || !read_file(path, buf))
        return fail(BIDA_ERR_RUNTIME, std::string("cannot open weights file: ") + (path ? path : ""));
    return bida_gpu_mlp_create_bmlp1(device, domain, buf.data(), buf.size(), quantile, out);
}

} // extern "C"

namespace {
struct NvtxRange {  // SURVEY §5 tracing: one range per C-ABI evaluate call
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
} // namespace

extern "C" {

int bida_gpu_evaluate_logits(bida_gpu_evaluator *ev, const void *packed, int64_t n, int32_t *h_out,
                             double *logits_out) {
    NvtxRange nvtx(n <= kZeroCopyMax && !logits_out ? "bida_gpu_evaluate/zero_copy" : "bida_gpu_evaluate/staged");
    if (!ev)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "NULL evaluator");
    if (n < 0 || (n > 0 && (!packed || !h_out)))
        return fail(BIDA_ERR_INVALID_ARGUMENT, "bad batch arguments");
    if (n == 0)
        return BIDA_OK;
    CUDA_TRY(cudaSetDevice(ev->device));
    if (n <= kZeroCopyMax && !logits_out) {
        bida_gpu_evaluator::ZcLane *ln = acquire_lane(ev);
        const int pbz = packed_bytes(ev->domain);
        std::memcpy(ln->in, packed, static_cast<size_t>(n) * pbz);
        const int ch = static_cast<int>(ln - ev->zc);
        int rc = lane_launch(ev, ln, n, ch);
        if (rc == BIDA_OK) {
            const cudaError_t e = cudaStreamSynchronize(ln->st);
            if (e != cudaSuccess)
                rc = fail(BIDA_ERR_CUDA, std::string("evaluate: ") + cudaGetErrorString(e));
        }
        ev->zc_calls.fetch_add(1, std::memory_order_relaxed);
        if (rc != BIDA_OK) {
            std::fill(h_out, h_out + n, 0);
            collect_errors(ev, ch);
            release_lane(ln);
            return rc;
        }
        std::memcpy(h_out, ln->out, static_cast<size_t>(n) * 4);
        rc = collect_errors(ev, ch);
        release_lane(ln);
        return rc;
    }
    // Page-locked caller buffers are mapped into the device's address space
    // (unified addressing): the kernel reads the packed states over PCIe and
    // writes h straight back, one launch for the whole batch -- no chunked
    // copies, no per-copy overhead, no pipeline fill or drain
    // (BIDA_GPU_DIRECT=0: always the chunked copy pipeline).
    if (!logits_out && direct_enabled()) {
        void *dp = nullptr, *dh = nullptr;
        if (is_pinned(packed) && is_pinned(h_out) &&
            cudaHostGetDevicePointer(&dp, const_cast<void *>(packed), 0) == cudaSuccess &&
            cudaHostGetDevicePointer(&dh, h_out, 0) == cudaSuccess &&
            reinterpret_cast<uintptr_t>(dp) % 16 == 0 && reinterpret_cast<uintptr_t>(dh) % 4 == 0) {
            NvtxRange nvtx_d("bida_gpu_evaluate/direct");
            std::lock_guard<std::mutex> lk(ev->mu);
            int rc = launch(ev, dp, n, static_cast<int32_t *>(dh), nullptr, ev->stream[0], chan_err(ev, kChanPipe));
            if (rc == BIDA_OK) {
                const cudaError_t e = cudaStreamSynchronize(ev->stream[0]);
                if (e != cudaSuccess)
                    rc = fail(BIDA_ERR_CUDA, std::string("evaluate: ") + cudaGetErrorString(e));
            }
            if (rc != BIDA_OK) {
                std::fill(h_out, h_out + n, 0);
                collect_errors(ev, kChanPipe);
                return rc;
            }
            return collect_errors(ev, kChanPipe);
        }
        (void)cudaGetLastError();  // a pointer that is not mapped: the copy pipeline below
    }
    std::lock_guard<std::mutex> lk(ev->mu);
    if (int rc = ensure_slots(ev, n)) {
        std::fill(h_out, h_out + n, 0);
        return rc;
    }
    const int pb = packed_bytes(ev->domain);
    const size_t per_logits = static_cast<size_t>(ev->E) * ev->C;
    double *d_logits = nullptr;
    if (logits_out)
        CUDA_TRY(cudaMalloc(&d_logits, static_cast<size_t>(std::min<int64_t>(n, ev->slot_cap)) *
                                           per_logits * sizeof(double)));
    const char *src = static_cast<const char *>(packed);
    // Caller buffers that are already page-locked (cudaHostAlloc /
    // cudaHostRegister / torch pin_memory) are DMA'd directly; pageable ones
    // go through the handle's pinned staging slots.
    const bool in_pinned = is_pinned(packed);
    const bool out_pinned = is_pinned(h_out);
    int64_t pend_off[kSlots], pend_n[kSlots];
    for (int k = 0; k < kSlots; ++k) {
        pend_off[k] = -1;
        pend_n[k] = 0;
    }
    int rc = BIDA_OK;
    auto drain = [&](int s) -> int {
        if (pend_off[s] < 0)
            return BIDA_OK;
        cudaError_t e = cudaEventSynchronize(ev->done[s]);
        if (e != cudaSuccess)
            return fail(BIDA_ERR_CUDA, std::string("evaluate: ") + cudaGetErrorString(e));
        if (!out_pinned)
            std::memcpy(h_out + pend_off[s], ev->h_h[s], pend_n[s] * 4);
        pend_off[s] = -1;
        return BIDA_OK;
    };
    int slot = 0;
    for (int64_t i0 = 0, m = 0; i0 < n && rc == BIDA_OK; i0 += m, slot = (slot + 1) % kSlots) {
        m = chunk_for(n - i0, ev->slot_cap);
        if ((rc = drain(slot)))
            break;
        const void *h2d_src = src + i0 * pb;
        if (!in_pinned) {
            std::memcpy(ev->h_in[slot], src + i0 * pb, m * pb);
            h2d_src = ev->h_in[slot];
        }
        cudaStream_t st = ev->stream[slot];
        cudaError_t e = cudaMemcpyAsync(ev->d_in[slot], h2d_src, m * pb, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) {
            rc = fail(BIDA_ERR_CUDA, std::string("H2D: ") + cudaGetErrorString(e));
            break;
        }
        if ((rc = launch(ev, ev->d_in[slot], m, ev->d_h[slot], d_logits, st, chan_err(ev, kChanPipe))))
            break;
        e = cudaMemcpyAsync(out_pinned ? static_cast<void *>(h_out + i0) : static_cast<void *>(ev->h_h[slot]),
                            ev->d_h[slot], m * 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess)
            e = cudaEventRecord(ev->done[slot], st);
        if (e != cudaSuccess) {
            rc = fail(BIDA_ERR_CUDA, std::string("D2H: ") + cudaGetErrorString(e));
            break;
        }
        pend_off[slot] = i0;
        pend_n[slot] = m;
        if (d_logits) {
            // diagnostics path: serialise so the single logits buffer is reused safely
            e = cudaMemcpyAsync(logits_out + i0 * per_logits, d_logits,
                                m * per_logits * sizeof(double), cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess)
                e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) {
                rc = fail(BIDA_ERR_CUDA, std::string("logits D2H: ") + cudaGetErrorString(e));
                break;
            }
        }
    }
    for (int s = 0; s < kSlots; ++s) {  // oldest pending chunk first
        const int r = drain((slot + s) % kSlots) ? BIDA_ERR_CUDA : BIDA_OK;
        if (rc == BIDA_OK)
            rc = r;
    }
    // make sure no stream still writes staging before we return
    for (int s = 0; s < kSlots; ++s)
        cudaStreamSynchronize(ev->stream[s]);
    if (d_logits)
        cudaFree(d_logits);
    if (rc != BIDA_OK) {
        std::fill(h_out, h_out + n, 0);
        collect_errors(ev, kChanPipe);
        return rc;
    }
    return collect_errors(ev, kChanPipe);
}

int bida_gpu_evaluate(bida_gpu_evaluator *ev, const void *packed, int64_t n, int32_t *h_out) {
    return bida_gpu_evaluate_logits(ev, packed, n, h_out, nullptr);
}

int bida_gpu_batch_begin(bida_gpu_evaluator *ev, int64_t n, bida_gpu_batch **out, void **in_host) {
    if (!out || !in_host)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "out pointers are NULL");
    *out = nullptr;
    *in_host = nullptr;
    if (!ev)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "NULL evaluator");
    if (n < 0)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "bad batch arguments");
    if (n > kZeroCopyMax)
        return fail(BIDA_ERR_CAPACITY, "asynchronous batches hold at most 32768 states");
    bida_gpu_evaluator::ZcLane *ln = acquire_lane(ev);
    ln->n = n;
    *out = reinterpret_cast<bida_gpu_batch *>(ln);
    *in_host = ln->in;
    return BIDA_OK;
}

int bida_gpu_batch_launch(bida_gpu_batch *b) {
    if (!b)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "NULL batch");
    auto *ln = reinterpret_cast<bida_gpu_evaluator::ZcLane *>(b);
    bida_gpu_evaluator *ev = ln->owner;
    const int ch = static_cast<int>(ln - ev->zc);
    int rc = BIDA_OK;
    cudaError_t e = cudaSetDevice(ev->device);
    if (e != cudaSuccess)
        rc = fail(BIDA_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e));
    if (rc == BIDA_OK)
        rc = lane_launch(ev, ln, ln->n, ch);
    if (rc == BIDA_OK) {
        e = cudaEventRecord(ln->done, ln->st);
        if (e != cudaSuccess)
            rc = fail(BIDA_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e));
    }
    if (rc != BIDA_OK) {
        cudaStreamSynchronize(ln->st);
        collect_errors(ev, ch);
        release_lane(ln);
        return rc;
    }
    ev->zc_calls.fetch_add(1, std::memory_order_relaxed);
    return BIDA_OK;
}

int bida_gpu_submit(bida_gpu_evaluator *ev, const void *packed, int64_t n, bida_gpu_batch **out) {
    NvtxRange nvtx("bida_gpu_submit");
    if (!out)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "out batch pointer is NULL");
    *out = nullptr;
    if (!ev)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "NULL evaluator");
    if (n < 0 || (n > 0 && !packed))
        return fail(BIDA_ERR_INVALID_ARGUMENT, "bad batch arguments");
    if (n > kZeroCopyMax)
        return fail(BIDA_ERR_CAPACITY, "asynchronous batches hold at most 32768 states");
    CUDA_TRY(cudaSetDevice(ev->device));
    bida_gpu_evaluator::ZcLane *ln = acquire_lane(ev);
    const int ch = static_cast<int>(ln - ev->zc);
    if (n > 0)
        std::memcpy(ln->in, packed, static_cast<size_t>(n) * packed_bytes(ev->domain));
    ln->n = n;
    int rc = lane_launch(ev, ln, n, ch);
    if (rc == BIDA_OK) {
        const cudaError_t e = cudaEventRecord(ln->done, ln->st);
        if (e != cudaSuccess)
            rc = fail(BIDA_ERR_CUDA, std::string("submit: ") + cudaGetErrorString(e));
    }
    if (rc != BIDA_OK) {
        cudaStreamSynchronize(ln->st);
        collect_errors(ev, ch);
        release_lane(ln);
        return rc;
    }
    ev->zc_calls.fetch_add(1, std::memory_order_relaxed);
    *out = reinterpret_cast<bida_gpu_batch *>(ln);
    return BIDA_OK;
}

int bida_gpu_batch_ready(bida_gpu_batch *b) {
    if (!b)
        return -fail(BIDA_ERR_INVALID_ARGUMENT, "NULL batch");
    auto *ln = reinterpret_cast<bida_gpu_evaluator::ZcLane *>(b);
    const cudaError_t e = cudaEventQuery(ln->done);
    if (e == cudaSuccess)
        return 1;
    if (e == cudaErrorNotReady)
        return 0;
    return -fail(BIDA_ERR_CUDA, std::string("batch: ") + cudaGetErrorString(e));
}

const int32_t *bida_gpu_batch_h(bida_gpu_batch *b) {
    return b ? reinterpret_cast<bida_gpu_evaluator::ZcLane *>(b)->out : nullptr;
}

int bida_gpu_batch_wait(bida_gpu_batch *b, int32_t *h_out) {
    NvtxRange nvtx("bida_gpu_batch_wait");
    if (!b)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "NULL batch");
    auto *ln = reinterpret_cast<bida_gpu_evaluator::ZcLane *>(b);
    bida_gpu_evaluator *ev = ln->owner;
    const int ch = static_cast<int>(ln - ev->zc);
    int rc = BIDA_OK;
    const cudaError_t e = cudaEventSynchronize(ln->done);
    if (e != cudaSuccess)
        rc = fail(BIDA_ERR_CUDA, std::string("batch wait: ") + cudaGetErrorString(e));
    const int erc = collect_errors(ev, ch);
    if (rc == BIDA_OK)
        rc = erc;
    if (h_out && ln->n > 0) {
        if (rc == BIDA_OK)
            std::memcpy(h_out, ln->out, static_cast<size_t>(ln->n) * 4);
        else
            std::fill(h_out, h_out + ln->n, 0);
    }
    release_lane(ln);
    return rc;
}

int bida_gpu_evaluate_device(bida_gpu_evaluator *ev, const void *d_packed, int64_t n, int32_t *d_h,
                             double *d_logits, void *stream) {
    NvtxRange nvtx("bida_gpu_evaluate_device");
    if (!ev)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "NULL evaluator");
    if (n < 0 || (n > 0 && (!d_packed || !d_h)))
        return fail(BIDA_ERR_INVALID_ARGUMENT, "bad batch arguments");
    CUDA_TRY(cudaSetDevice(ev->device));
    return launch(ev, d_packed, n, d_h, d_logits, static_cast<cudaStream_t>(stream), chan_err(ev, kChanDevice));
}

int bida_gpu_stream_status(bida_gpu_evaluator *ev) {
    if (!ev)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "NULL evaluator");
    return collect_errors(ev, kChanDevice);
}

int bida_gpu_info(const bida_gpu_evaluator *ev, bida_gpu_model_info *out) {
    if (!ev || !out)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "NULL argument");
    std::memset(out, 0, sizeof(*out));
    out->kind = ev->kind;
    out->domain = ev->domain;
    out->features = ev->F;
    out->classes = ev->C;
    out->ensemble = ev->E;
    out->hidden_layers = ev->hidden_layers;
    for (int l = 0; l < 8; ++l)
        out->hidden[l] = ev->hidden[l];
    out->quantile = ev->q;
    out->device = ev->device;
    out->weights_in_smem = ev->w_in_smem;
    return BIDA_OK;
}

} // extern "C"

namespace {
// Installs a device table (ownership passes to the handle); the caller holds
// every lock of the handle.
void install_pdb(bida_gpu_evaluator *ev, const uint8_t *pattern, int pattern_len, uint8_t *d, uint64_t n_entries,
                 int mode) {
    const int n = ev->domain == BIDA_DOMAIN_RC ? 8 : ev->domain * ev->domain;
    PdbArgs a{};
    a.n = n_entries;
    a.m = pattern_len;
    a.mode = mode;
    for (int i = 0; i < pattern_len; ++i) {
        a.pat[i] = pattern[i];
        unsigned long long w = 1;  // partial_perm_rank weight (ranking.hpp:43-45)
        for (int k = 0; k < pattern_len - i - 1; ++k)
            w *= static_cast<unsigned long long>(n - i - 1 - k);
        a.w[i] = w;
    }
    if (ev->d_pdb)
        cudaFree(ev->d_pdb);
    ev->d_pdb = d;
    a.entries = d;
    ev->pdb = a;
}
} // namespace

extern "C" {

int bida_gpu_attach_pdb(bida_gpu_evaluator *ev, const uint8_t *pattern, int pattern_len,
                        const uint8_t *entries, uint64_t n_entries, int mode) {
    if (!ev)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "NULL evaluator");
    HandleLock all(ev);
    CUDA_TRY(cudaSetDevice(ev->device));
    if (mode == BIDA_PDB_OFF) {
        if (ev->d_pdb)
            cudaFree(ev->d_pdb);
        ev->d_pdb = nullptr;
        ev->pdb = PdbArgs{};
        return BIDA_OK;
    }
    if (mode != BIDA_PDB_MIN && mode != BIDA_PDB_REPLACE)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "unknown PDB mode");
    if (!pattern || pattern_len <= 0 || pattern_len > kPdbMaxPattern || !entries)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "PDB pattern must have 1..8 labels");
    const int n = ev->domain == BIDA_DOMAIN_RC ? 8 : ev->domain * ev->domain;
    for (int i = 0; i < pattern_len; ++i) {
        if (pattern[i] >= n)
            return fail(BIDA_ERR_INVALID_ARGUMENT, ev->domain == BIDA_DOMAIN_RC
                                                       ? "RubiksCube::Abstraction: only corner labels 0..7 supported"
                                                       : "TilePuzzle::Abstraction: label out of range");
        for (int j = 0; j < i; ++j)
            if (pattern[j] == pattern[i])
                return fail(BIDA_ERR_INVALID_ARGUMENT, "PDB pattern repeats a label");
    }
    // Abstraction::size (stp.hpp:204-206, rubiks.hpp:240-245)
    uint64_t expect = 1;
    for (int i = 0; i < pattern_len; ++i)
        expect *= static_cast<uint64_t>(n - i);
    if (ev->domain == BIDA_DOMAIN_RC)
        for (int i = 0; i < pattern_len; ++i)
            expect *= 3;
    if (n_entries != expect)
        return fail(BIDA_ERR_RUNTIME, "PDB entry count does not match pattern");
    uint8_t *d = nullptr;
    CUDA_TRY(cudaMalloc(&d, n_entries));
    const cudaError_t e = cudaMemcpy(d, entries, n_entries, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(d);
        return fail(BIDA_ERR_CUDA, std::string("PDB upload: ") + cudaGetErrorString(e));
    }
    install_pdb(ev, pattern, pattern_len, d, n_entries, mode);
    return BIDA_OK;
}

int bida_gpu_attach_pdb_built(bida_gpu_evaluator *ev, const uint8_t *pattern, int pattern_len, int mode) {
    if (!ev)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "NULL evaluator");
    if (mode != BIDA_PDB_MIN && mode != BIDA_PDB_REPLACE)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "unknown PDB mode");
    CUDA_TRY(cudaSetDevice(ev->device));
    uint8_t *d = nullptr;
    uint64_t n = 0;
    if (int rc = bida_gpu::pdb_build_device(ev->domain, pattern, pattern_len, &d, &n))
        return rc;
    HandleLock all(ev);
    install_pdb(ev, pattern, pattern_len, d, n, mode);
    return BIDA_OK;
}

int bida_gpu_attach_pdb_file(bida_gpu_evaluator *ev, const char *path, int mode) {
    // BPDB1 (pdb.hpp:78-138): "BPDB1", tag ('S' / 'R'), board (N*N / 0), u8 plen,
    // pattern, u64 entry count (little-endian), entries.
    if (!ev)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "NULL evaluator");
    std::vector<unsigned char> b;
    if (!path || !read_file(path, b))
        return fail(BIDA_ERR_RUNTIME, std::string("cannot open PDB file: ") + (path ? path : ""));
    if (b.size() < 5 || std::memcmp(b.data(), "BPDB1", 5) != 0)
        return fail(BIDA_ERR_RUNTIME, std::string("not a BPDB1 file: ") + path);
    if (b.size() < 8)
        return fail(BIDA_ERR_RUNTIME, std::string("corrupt PDB header: ") + path);
    const bool rc = ev->domain == BIDA_DOMAIN_RC;
    const int tag = b[5], board = b[6], plen = b[7];
    if (tag != (rc ? 'R' : 'S') || board != (rc ? 0 : ev->domain * ev->domain))
        return fail(BIDA_ERR_RUNTIME, std::string("PDB domain mismatch: ") + path);
    if (plen <= 0 || b.size() < 8 + static_cast<size_t>(plen) + 8)
        return fail(BIDA_ERR_RUNTIME, std::string("corrupt PDB header: ") + path);
    uint64_t cnt = 0;
    for (int i = 0; i < 8; ++i)
        cnt |= static_cast<uint64_t>(b[8 + plen + i]) << (8 * i);
    const size_t off = 8 + plen + 8;
    if (b.size() < off + cnt)
        return fail(BIDA_ERR_RUNTIME, std::string("truncated PDB file: ") + path);
    return bida_gpu_attach_pdb(ev, b.data() + 8, plen, b.data() + off, cnt, mode);
}

int bida_gpu_debug_trace(bida_gpu_evaluator *ev, long long *dev_buf) {
    if (!ev || ev->kind != BIDA_MODEL_MLP)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "debug trace needs an MLP evaluator");
#if !defined(BIDA_MLP_TRACE) || !BIDA_MLP_TRACE
    if (dev_buf)
        return fail(BIDA_ERR_STATE, "tracing is compiled into libbida_gpu_trace.so only (build.py trace=True)");
#endif
    mlp_set_trace(ev->mlp, dev_buf);
    return BIDA_OK;
}

int bida_gpu_trace_slots(void) { return mlp_trace_slots(); }

int bida_gpu_exact_replays(bida_gpu_evaluator *ev, int64_t *out) {
    if (!ev || !out)
        return fail(BIDA_ERR_INVALID_ARGUMENT, "NULL argument");
    CUDA_TRY(cudaSetDevice(ev->device));
    unsigned long long v = 0;
    CUDA_TRY(cudaMemcpy(&v, ev->d_replays, sizeof(v), cudaMemcpyDeviceToHost));
    *out = static_cast<int64_t>(v);
    return BIDA_OK;
}

int64_t bida_gpu_launch_count(const bida_gpu_evaluator *ev) {
    return ev ? ev->launches.load(std::memory_order_relaxed) : 0;
}

int64_t bida_gpu_graph_launch_count(const bida_gpu_evaluator *ev) {
    return ev ? ev->graph_launches.load(std::memory_order_relaxed) : 0;
}

int bida_gpu_destroy(bida_gpu_evaluator *ev) {
    release(ev);
    return BIDA_OK;
}

} // extern "C"
