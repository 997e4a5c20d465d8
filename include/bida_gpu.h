/*
 * bida_gpu.h — C-ABI of the B200 batched heuristic evaluator.
 *
 * This is the drop-in boundary for the reference's evaluator backend
 * (/root/reference/proj/include/bida/batch_eval.hpp:45-51,
 *  `EvaluatorBackend<D>::evaluate(span<const BatchItem<D>>, span<int32_t>)`).
 * Plain pointers and sizes only; no C++ or torch types.  The C++ adapter
 * `bida_gpu::GpuBackend<D>` (include/bida_gpu_backend.hpp) wraps it into a
 * `bida::EvaluatorBackend<D>`; INTEGRATION.md shows the bindings.
 *
 * States cross the boundary PACKED exactly as the reference packs them:
 *   STP N=2..4 : one little-endian u64, 4 bits per cell (stp.hpp:121-126)
 *   Rubik's    : {u64 lo, u64 hi} = RubiksCube::Packed (rubiks.hpp:121-137)
 * The one-hot encode (stp.hpp:141-146, rubiks.hpp:155-166) happens on the
 * device, so the backend reports needs_features() == false.
 *
 * Every entry point returns a status (BIDA_OK == 0); on failure the message
 * is available from bida_gpu_last_error() (thread-local).  Nothing throws.
 * Handles are safe to use from several host threads at once (the agent thread
 * and evaluate_single / evaluate_sync callers of batch_eval.hpp:241,261).
 */
#ifndef BIDA_GPU_H
#define BIDA_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BIDA_GPU_ABI_VERSION 1

/* Domains: TilePuzzle<N> (stp.hpp:19-286) and RubiksCube (rubiks.hpp:19-383). */
enum bida_domain {
    BIDA_DOMAIN_STP2 = 2,
    BIDA_DOMAIN_STP3 = 3,
    BIDA_DOMAIN_STP4 = 4,
    BIDA_DOMAIN_RC = 100
};

/* Status codes.  INVALID_ARGUMENT / RUNTIME mirror the std::invalid_argument /
 * std::runtime_error the reference throws from the same call. */
enum bida_status {
    BIDA_OK = 0,
    BIDA_ERR_INVALID_ARGUMENT = 1, /* ctor checks, batch_eval.hpp:87-93       */
    BIDA_ERR_RUNTIME = 2,          /* BLIN1 load errors, batch_eval.hpp:111-129 */
    BIDA_ERR_CUDA = 3,             /* device / driver failure                 */
    BIDA_ERR_DISTRIBUTION = 4,     /* ClassDistribution::validate, heuristic.hpp:95-104 */
    BIDA_ERR_STATE = 5,            /* packed state encodes outside [0, F)     */
    BIDA_ERR_CAPACITY = 6          /* batch larger than the handle allows     */
};

enum bida_model_kind { BIDA_MODEL_LINEAR = 1, BIDA_MODEL_MLP = 2 };

typedef struct bida_gpu_evaluator bida_gpu_evaluator;

typedef struct bida_gpu_model_info {
    int32_t kind;           /* bida_model_kind                 */
    int32_t domain;         /* bida_domain                     */
    int32_t features;       /* F = D::feature_length()         */
    int32_t classes;        /* C                               */
    int32_t ensemble;       /* E                               */
    int32_t hidden_layers;  /* MLP only, else 0                */
    int32_t hidden[8];      /* MLP widths                      */
    double quantile;        /* q of quantile_class             */
    int32_t device;
    int32_t weights_in_smem;
} bida_gpu_model_info;

int bida_gpu_abi_version(void);
const char *bida_gpu_last_error(void);
int bida_gpu_device_count(void);
/* D::feature_length() (stp.hpp:139, rubiks.hpp:153); -1 for unknown domain. */
int bida_gpu_feature_length(int domain);
/* bytes of one packed state (8 or 16); -1 for unknown domain. */
int bida_gpu_packed_bytes(int domain);

/* LinearModelBackend(member_weights, classes, quantile) (batch_eval.hpp:85-94).
 * weights: ensemble * classes * F floats, member-major, each member row-major
 * [C][F] as in the reference.  q is validated here (the reference validates it
 * in quantile_class, heuristic.hpp:110-111, at evaluate time). */
int bida_gpu_linear_create(int device, int domain, const float *weights, int ensemble,
                           int classes, double quantile, bida_gpu_evaluator **out);

/* LinearModelBackend::load(path, quantile) (batch_eval.hpp:109-131) from an
 * in-memory BLIN1 image, and from a file path with the reference's messages. */
int bida_gpu_linear_create_blin1(int device, int domain, const void *blob, size_t len,
                                 double quantile, bida_gpu_evaluator **out);
int bida_gpu_linear_load(int device, int domain, const char *path, double quantile,
                         bida_gpu_evaluator **out);

/* BMLP1 integer MLP ensemble (project format; the reference has
 * no MLP).  Same readout as the linear model.  Hidden widths 1..4096 (the
 * kernel schedule -- weights resident in shared memory, streamed, or wide
 * with activations in L2-resident scratch -- is chosen at load time), up to 4
 * hidden layers, C <= 256 classes, E <= 8 members. */
int bida_gpu_mlp_create_bmlp1(int device, int domain, const void *blob, size_t len,
                              double quantile, bida_gpu_evaluator **out);
int bida_gpu_mlp_load(int device, int domain, const char *path, double quantile,
                      bida_gpu_evaluator **out);

/* EvaluatorBackend<D>::evaluate (batch_eval.hpp:49): n packed HOST states ->
 * n int32 h-values in HOST memory.  Synchronous; any n >= 0 (batches larger
 * than the internal staging are pipelined in chunks).  On error every h_out[i]
 * is still written (0). */
int bida_gpu_evaluate(bida_gpu_evaluator *ev, const void *packed, int64_t n, int32_t *h_out);

/* Same, also returning the per-member logits as float64 [n][E][C]
 * (diagnostics / parity; may be NULL). */
int bida_gpu_evaluate_logits(bida_gpu_evaluator *ev, const void *packed, int64_t n,
                             int32_t *h_out, double *logits_out);

/* Asynchronous submit / complete (SURVEY §8(b) optional extra): bida_gpu_submit
 * copies n <= 32768 packed HOST states into one of the handle's 8 zero-copy
 * lanes (mapped pinned memory) and launches the evaluation; the GPU writes the
 * int32 h-values straight into mapped host memory at bida_gpu_batch_h(b),
 * readable once bida_gpu_batch_ready(b) returns 1 (0: not yet; < 0: -status).
 * bida_gpu_batch_wait(b, h_out) waits, copies h (h_out may be NULL), reports
 * this batch's errors only, and releases the lane (b is invalid afterwards).
 * A lane is held from submit to wait: at most 8 batches per handle in flight;
 * a ninth submit waits for a lane. */
typedef struct bida_gpu_batch bida_gpu_batch;
int bida_gpu_submit(bida_gpu_evaluator *ev, const void *packed, int64_t n, bida_gpu_batch **out);
/* The same in two steps, without the staging copy: bida_gpu_batch_begin
 * reserves a lane for n <= 32768 states and returns its mapped (write-combined)
 * host input buffer; the caller packs the states straight into it, then
 * bida_gpu_batch_launch starts the evaluation (ready / h / wait as above). */
int bida_gpu_batch_begin(bida_gpu_evaluator *ev, int64_t n, bida_gpu_batch **out, void **in_host);
int bida_gpu_batch_launch(bida_gpu_batch *b);
int bida_gpu_batch_ready(bida_gpu_batch *b);
const int32_t *bida_gpu_batch_h(bida_gpu_batch *b);
int bida_gpu_batch_wait(bida_gpu_batch *b, int32_t *h_out);

/* Device-resident variant: d_packed / d_h / d_logits are DEVICE pointers on
 * the handle's device, `stream` a cudaStream_t (NULL = legacy default).
 * Asynchronous: returns after enqueueing; call bida_gpu_stream_status() after
 * synchronising the stream to collect a deferred per-state error. */
int bida_gpu_evaluate_device(bida_gpu_evaluator *ev, const void *d_packed, int64_t n,
                             int32_t *d_h, double *d_logits, void *stream);
int bida_gpu_stream_status(bida_gpu_evaluator *ev);

/* PDB correction in the readout (north star "admissible class-argmax/PDB-
 * correction readout"): h = min(h_model, h_PDB) (BIDA_PDB_MIN), or h = h_PDB
 * with the model still evaluated (BIDA_PDB_REPLACE: the paper's Table-1 mode,
 * PAPER.md:407).  h_PDB = PdbTable<D>::lookup (pdb.hpp:66-69) over the rank of
 * Abstraction::rank_state (rubiks.hpp:247-267 corners, stp.hpp:208-227 tiles),
 * computed on the device.  `entries` as PdbTable::entries(); the table is
 * copied to device memory.  BIDA_PDB_OFF detaches. */
enum bida_pdb_mode { BIDA_PDB_OFF = 0, BIDA_PDB_MIN = 1, BIDA_PDB_REPLACE = 2 };
int bida_gpu_attach_pdb(bida_gpu_evaluator *ev, const uint8_t *pattern, int pattern_len,
                        const uint8_t *entries, uint64_t n_entries, int mode);
/* Same from a BPDB1 file written by PdbTable::save (pdb.hpp:78-96). */
int bida_gpu_attach_pdb_file(bida_gpu_evaluator *ev, const char *path, int mode);

/* PdbTable<D>::build(pattern, D::solved()) (pdb.hpp:30-64) as a level-
 * synchronous breadth-first search on the GPU; the table is byte-identical to
 * the reference's (BFS distances are unique).  `max_entries` (0 = the
 * reference's default cap 2^28, pdb.hpp kDefaultPdbEntryCap) mirrors the
 * reference's size check and message.  *n_entries is set before the capacity
 * check, so a call with entries_out == NULL sizes the buffer. */
int bida_gpu_pdb_build(int device, int domain, const uint8_t *pattern, int pattern_len, uint64_t max_entries,
                       uint8_t *entries_out, uint64_t out_cap, uint64_t *n_entries, int *max_depth);
/* Same, written to `path` in the BPDB1 format of PdbTable::save (pdb.hpp:78-96),
 * so the reference's PdbTable::load reads it. */
int bida_gpu_pdb_build_save(int device, int domain, const uint8_t *pattern, int pattern_len, const char *path);
/* Builds the table on the evaluator's device and attaches it (no host copy). */
int bida_gpu_attach_pdb_built(bida_gpu_evaluator *ev, const uint8_t *pattern, int pattern_len, int mode);

/* Synthetic benchmark input: n packed non-retracting random-walk
 * scrambles from the solved state, state i of len_min + i % (len_max - len_min
 * + 1) moves (the distribution of random_walk_instance, instance.hpp:36-57; a
 * counter-based RNG, not mt19937_64), written to DEVICE memory d_out on
 * `stream` (asynchronous). */
int bida_gpu_random_walks(int device, int domain, int64_t n, int len_min, int len_max, uint64_t seed,
                          void *d_out, void *stream);

int bida_gpu_info(const bida_gpu_evaluator *ev, bida_gpu_model_info *out);
/* Diagnostics (MLP handles): record a clock64 timeline of CTA 0's warps into
 * the DEVICE buffer `dev_buf` (int64 [32 warps][bida_gpu_trace_slots()]) on every
 * subsequent launch; NULL switches it off. */
int bida_gpu_debug_trace(bida_gpu_evaluator *ev, long long *dev_buf);
int bida_gpu_trace_slots(void);
/* Parity diagnostics: number of (state, member) readouts so far whose
 * certified float32 softmax bound could not decide the class and that replayed
 * the reference's float64 sequence (batch_eval.hpp:159-166,
 * heuristic.hpp:95-120) instead.  Synchronous; counts completed work only. */
int bida_gpu_exact_replays(bida_gpu_evaluator *ev, int64_t *out);
/* Number of kernel launches issued by this handle so far (bench evidence). */
int64_t bida_gpu_launch_count(const bida_gpu_evaluator *ev);
/* How many of those launches were replays of a zero-copy lane's CUDA graph
 * (small batches; BIDA_GPU_GRAPHS=0 disables the graphs). */
int64_t bida_gpu_graph_launch_count(const bida_gpu_evaluator *ev);
int bida_gpu_destroy(bida_gpu_evaluator *ev);

#ifdef __cplusplus
}
#endif
#endif /* BIDA_GPU_H */
