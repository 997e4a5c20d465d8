/*
 * bida_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the reference's batched heuristic evaluation path,
 * used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg to
 * check the CUDA evaluator.  Nothing in paper_2507_11916_b200/ links this.
 *
 * Every function cites the reference (/root/reference/proj/...) line it
 * restates.  The restatement is pinned against the reference itself: the
 * reference headers are compiled unchanged into oracle/_ref/libbida_ref.so by
 * oracle/Makefile, and tests/test_oracle.py checks this file against that
 * library and against the golden vectors in tests/golden/.
 *
 * Parity of the MLP ("BMLP1") path is pinned only by construction: the
 * reference has no MLP; this file is its definition.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "bida_oracle.h"

/* ---------------------------------------------------------------- domains */

int orc_feature_length(int domain) {
    switch (domain) {
    case ORC_STP2: return 16;   /* stp.hpp:139 kCells*kCells */
    case ORC_STP3: return 81;
    case ORC_STP4: return 256;
    case ORC_RC: return 480;    /* rubiks.hpp:153 8*24 + 12*24 */
    default: return -1;
    }
}

int orc_packed_bytes(int domain) {
    /* stp.hpp:121-126 packs into one u64; rubiks.hpp:121-137 into {lo, hi}. */
    if (domain == ORC_RC) return 16;
    if (domain >= ORC_STP2 && domain <= ORC_STP4) return 8;
    return -1;
}

int orc_active_features(int domain) {
    if (domain == ORC_RC) return 20;
    if (domain >= ORC_STP2 && domain <= ORC_STP4) return domain * domain;
    return -1;
}

/* Active one-hot indices of one packed state, in ascending index order.
 * STP: x[cell*N^2 + tiles[cell]] = 1 (stp.hpp:141-146); ascending in cell.
 * RC : x[cp[p]*24 + p*3 + co[p]] and x[192 + ep[p]*24 + p*2 + eo[p]]
 *      (rubiks.hpp:155-166); ascending means ordered by cubie id, so the
 *      position is found through the inverse permutation.  Packed layout is
 *      rubiks.hpp:126-137: lo = cp (3b each) | co (2b each) << 24 |
 *      eo (1b each) << 40, hi = ep (4b each). */
int orc_active_indices(int domain, const void *packed, int *idx) {
    if (domain >= ORC_STP2 && domain <= ORC_STP4) {
        const int N = domain, K = N * N;
        uint64_t v;
        memcpy(&v, packed, 8);
        for (int cell = 0; cell < K; ++cell)
            idx[cell] = cell * K + (int)((v >> (4 * cell)) & 0xF);
        return K;
    }
    if (domain == ORC_RC) {
        uint64_t lo, hi;
        memcpy(&lo, packed, 8);
        memcpy(&hi, (const char *)packed + 8, 8);
        int k = 0;
        for (int c = 0; c < 8; ++c)
            for (int p = 0; p < 8; ++p)
                if ((int)((lo >> (3 * p)) & 7) == c)
                    idx[k++] = c * 24 + p * 3 + (int)((lo >> (24 + 2 * p)) & 3);
        for (int e = 0; e < 12; ++e)
            for (int p = 0; p < 12; ++p)
                if ((int)((hi >> (4 * p)) & 0xF) == e)
                    idx[k++] = 192 + e * 24 + p * 2 + (int)((lo >> (40 + p)) & 1);
        return k;
    }
    return -1;
}

/* D::encode (stp.hpp:141-146, rubiks.hpp:155-166): dense float one-hot row. */
int orc_encode(int domain, const void *packed, int64_t n, float *out) {
    const int F = orc_feature_length(domain), pb = orc_packed_bytes(domain);
    if (F < 0) return ORC_ERR_ARG;
    int idx[32];
    for (int64_t i = 0; i < n; ++i) {
        float *x = out + i * F;
        for (int j = 0; j < F; ++j) x[j] = 0.0f;
        const int k = orc_active_indices(domain, (const char *)packed + i * pb, idx);
        for (int a = 0; a < k; ++a) x[idx[a]] = 1.0f;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------ the readout */

/* ClassDistribution::validate (heuristic.hpp:95-104) followed by
 * quantile_class (heuristic.hpp:109-120).  Returns the class, or -1 with
 * *err set where the reference throws std::invalid_argument. */
int orc_quantile_class(const double *p, int C, double q, int *err) {
    if (q <= 0.0 || q > 1.0) { *err = ORC_ERR_QUANTILE; return -1; }
    double sum = 0.0;
    for (int c = 0; c < C; ++c) {
        if (p[c] < 0.0) { *err = ORC_ERR_DISTRIBUTION; return -1; }
        sum += p[c];
    }
    if (fabs(sum - 1.0) > 1e-9) { *err = ORC_ERR_DISTRIBUTION; return -1; }
    double cum = 0.0;
    for (int c = 0; c < C; ++c) {
        cum += p[c];
        if (cum >= q - 1e-12) return c;
    }
    return C - 1;
}

/* Softmax of LinearModelBackend::score (batch_eval.hpp:159-166):
 * max_element, exp(l - mx) accumulated into z in class order, p = l / z.
 * std::max_element keeps the first maximum and compares with operator<. */
void orc_softmax(const double *logits, int C, double *p) {
    double mx = logits[0];
    for (int c = 1; c < C; ++c)
        if (mx < logits[c]) mx = logits[c];
    double z = 0.0;
    for (int c = 0; c < C; ++c) {
        p[c] = exp(logits[c] - mx);
        z += p[c];
    }
    for (int c = 0; c < C; ++c) p[c] = p[c] / z;
}

/* ------------------------------------------------------- linear ensemble */

/* LinearModelBackend::evaluate + score (batch_eval.hpp:98-105, 148-168):
 * per member m, logit[c] = sum_{j=0..F-1} (double)W_m[c*F+j] * (double)x[j]
 * in ascending j over the dense one-hot row; then softmax, quantile_class and
 * ensemble_min (heuristic.hpp:122-126). logits_out (optional) is [n][E][C]. */
int orc_linear_evaluate(int domain, const float *W, int E, int C, double q, const void *packed,
                        int64_t n, int32_t *h_out, double *logits_out) {
    const int F = orc_feature_length(domain), pb = orc_packed_bytes(domain);
    if (F < 0 || E < 1 || C < 1) return ORC_ERR_ARG;
    float *x = (float *)malloc(sizeof(float) * (size_t)F);
    double *lg = (double *)malloc(sizeof(double) * (size_t)C);
    double *p = (double *)malloc(sizeof(double) * (size_t)C);
    int rc = ORC_OK;
    for (int64_t i = 0; i < n && rc == ORC_OK; ++i) {
        orc_encode(domain, (const char *)packed + i * pb, 1, x);
        int best = 0;
        for (int m = 0; m < E; ++m) {
            const float *w = W + (size_t)m * C * F;
            for (int c = 0; c < C; ++c) {
                double dot = 0.0;
                const float *row = w + (size_t)c * F;
                for (int j = 0; j < F; ++j) dot += (double)row[j] * (double)x[j];
                lg[c] = dot;
            }
            if (logits_out) memcpy(logits_out + ((size_t)i * E + m) * C, lg, sizeof(double) * C);
            orc_softmax(lg, C, p);
            int err = ORC_OK;
            const int h = orc_quantile_class(p, C, q, &err);
            if (err != ORC_OK) { rc = err; break; }
            if (m == 0 || h < best) best = h;
        }
        h_out[i] = best;
    }
    free(x);
    free(lg);
    free(p);
    return rc;
}

/* BLIN1 (batch_eval.hpp:107-131): "BLIN1", u32 F, u32 C, u32 E little-endian,
 * then E*C*F f32 row-major.  Returns a malloc'd weight array. */
int orc_blin1_parse(const void *blob, size_t len, int F_expected, int *C, int *E, float **W) {
    const unsigned char *b = (const unsigned char *)blob;
    if (len < 5 || memcmp(b, "BLIN1", 5) != 0) return ORC_ERR_FORMAT;
    if (len < 17) return ORC_ERR_FORMAT;
    uint32_t h[3];
    for (int k = 0; k < 3; ++k)
        h[k] = (uint32_t)b[5 + 4 * k] | (uint32_t)b[6 + 4 * k] << 8 | (uint32_t)b[7 + 4 * k] << 16 |
               (uint32_t)b[8 + 4 * k] << 24;
    if (h[0] != (uint32_t)F_expected || h[2] == 0) return ORC_ERR_FORMAT;
    const size_t count = (size_t)h[0] * h[1] * h[2];
    if (len < 17 + count * 4) return ORC_ERR_TRUNCATED;
    *W = (float *)malloc(count * 4 + 4);
    memcpy(*W, b + 17, count * 4);
    *C = (int)h[1];
    *E = (int)h[2];
    return ORC_OK;
}

/* ----------------------------------------------------------- BMLP1 model */
/*
 * The reference has no MLP; BMLP1 is this project's
 * multi-layer extension of BLIN1, defined here and in DESIGN.md §4.  It is an
 * integer-quantised classifier ensemble so that any summation order gives the
 * same logits (bit-exact h on tensor cores by construction):
 *
 *   "BMLP1", u32 F, u32 C, u32 E, u32 L (hidden layers), u32 H[L]; then per
 *   member, per layer l = 0..L (in = l ? H[l-1] : F, out = l < L ? H[l] : C):
 *       i8  W[out][in]   row-major
 *       i32 bias[out]
 *       u32 shift        (hidden layers only)
 *   and per member one f32 out_scale.
 *
 *   hidden: a'[o] = clamp((bias[o] + sum_i W[o][i]*a[i]) >> shift, 0, 255)
 *           (arithmetic shift = floor division by 2^shift; a is u8 0..255)
 *   output: logit[c] = (double)(bias[c] + sum_i W[c][i]*a[i]) * (double)out_scale
 * followed by the reference readout (softmax, quantile_class, ensemble_min).
 * Layer 0's input is the one-hot encode (a = x in {0,1}).
 */
int orc_bmlp1_parse(const void *blob, size_t len, int F_expected, orc_mlp *m) {
    const unsigned char *b = (const unsigned char *)blob;
    memset(m, 0, sizeof(*m));
    if (len < 21 || memcmp(b, "BMLP1", 5) != 0) return ORC_ERR_FORMAT;
    size_t off = 5;
#define RD32(dst)                                                                               \
    do {                                                                                        \
        if (off + 4 > len) return ORC_ERR_TRUNCATED;                                            \
        dst = (uint32_t)b[off] | (uint32_t)b[off + 1] << 8 | (uint32_t)b[off + 2] << 16 |       \
              (uint32_t)b[off + 3] << 24;                                                       \
        off += 4;                                                                               \
    } while (0)
    uint32_t F, C, E, L;
    RD32(F);
    RD32(C);
    RD32(E);
    RD32(L);
    if (F != (uint32_t)F_expected || C == 0 || E == 0 || L == 0 || L > ORC_MLP_MAX_LAYERS)
        return ORC_ERR_FORMAT;
    m->F = (int)F;
    m->C = (int)C;
    m->E = (int)E;
    m->L = (int)L;
    for (uint32_t l = 0; l < L; ++l) {
        uint32_t h;
        RD32(h);
        if (h == 0 || h > 65536) return ORC_ERR_FORMAT;
        m->H[l] = (int)h;
    }
    m->layers = (orc_mlp_layer *)calloc((size_t)E * (L + 1), sizeof(orc_mlp_layer));
    m->out_scale = (float *)calloc(E, sizeof(float));
    for (uint32_t e = 0; e < E; ++e) {
        for (uint32_t l = 0; l <= L; ++l) {
            orc_mlp_layer *ly = &m->layers[e * (L + 1) + l];
            ly->in = l ? m->H[l - 1] : (int)F;
            ly->out = l < L ? m->H[l] : (int)C;
            const size_t nw = (size_t)ly->in * ly->out;
            if (off + nw > len) { orc_mlp_free(m); return ORC_ERR_TRUNCATED; }
            ly->W = (int8_t *)malloc(nw);
            memcpy(ly->W, b + off, nw);
            off += nw;
            if (l == 0) {
                ly->WT = (int8_t *)malloc(nw);
                for (int o = 0; o < ly->out; ++o)
                    for (int i = 0; i < ly->in; ++i)
                        ly->WT[(size_t)i * ly->out + o] = ly->W[(size_t)o * ly->in + i];
            }
            if (off + 4 * (size_t)ly->out > len) { orc_mlp_free(m); return ORC_ERR_TRUNCATED; }
            ly->bias = (int32_t *)malloc(4 * (size_t)ly->out);
            memcpy(ly->bias, b + off, 4 * (size_t)ly->out);
            off += 4 * (size_t)ly->out;
            if (l < L) {
                uint32_t s;
                if (off + 4 > len) { orc_mlp_free(m); return ORC_ERR_TRUNCATED; }
                s = (uint32_t)b[off] | (uint32_t)b[off + 1] << 8 | (uint32_t)b[off + 2] << 16 |
                    (uint32_t)b[off + 3] << 24;
                off += 4;
                if (s > 31) { orc_mlp_free(m); return ORC_ERR_FORMAT; }
                ly->shift = (int)s;
            }
        }
        if (off + 4 > len) { orc_mlp_free(m); return ORC_ERR_TRUNCATED; }
        memcpy(&m->out_scale[e], b + off, 4);
        off += 4;
    }
#undef RD32
    return ORC_OK;
}

void orc_mlp_free(orc_mlp *m) {
    if (m->layers) {
        for (int i = 0; i < m->E * (m->L + 1); ++i) {
            free(m->layers[i].W);
            free(m->layers[i].WT);
            free(m->layers[i].bias);
        }
    }
    free(m->layers);
    free(m->out_scale);
    memset(m, 0, sizeof(*m));
}

static int mlp_eval_range(const orc_mlp *m, int domain, double q, const void *packed, int64_t lo,
                          int64_t hi, int32_t *h_out, double *logits_out) {
    const int pb = orc_packed_bytes(domain);
    int maxw = m->F;
    for (int l = 0; l < m->L; ++l)
        if (m->H[l] > maxw) maxw = m->H[l];
    if (m->C > maxw) maxw = m->C;
    uint8_t *a = (uint8_t *)malloc(maxw);  /* hidden activations, 0..255 */
    int32_t *nx = (int32_t *)malloc(sizeof(int32_t) * maxw);
    int32_t *nx2 = (int32_t *)malloc(sizeof(int32_t) * maxw);
    double *lg = (double *)malloc(sizeof(double) * m->C);
    double *p = (double *)malloc(sizeof(double) * m->C);
    int idx[32];
    int rc = ORC_OK;
    for (int64_t i = lo; i < hi && rc == ORC_OK; ++i) {
        int k = orc_active_indices(domain, (const char *)packed + i * pb, idx);
        /* the one-hot row sets each x[j] once: sort, drop repeats */
        for (int s = 1; s < k; ++s)
            for (int t = s; t > 0 && idx[t - 1] > idx[t]; --t) {
                const int tmp = idx[t];
                idx[t] = idx[t - 1];
                idx[t - 1] = tmp;
            }
        int u = 0;
        for (int t = 0; t < k; ++t)
            if (t == 0 || idx[t] != idx[t - 1]) idx[u++] = idx[t];
        k = u;
        for (int t = 0; t < k; ++t)
            if (idx[t] < 0 || idx[t] >= m->F) rc = ORC_ERR_ARG; /* packed state encodes outside [0, F) */
        if (rc != ORC_OK) break;
        int best = 0;
        for (int e = 0; e < m->E; ++e) {
            for (int l = 0; l <= m->L; ++l) {
                const orc_mlp_layer *ly = &m->layers[e * (m->L + 1) + l];
                if (l == 0) {
                    /* x is one-hot: W x = the sum of the active columns (exact
                     * integers, so identical to the dense product) */
                    for (int o = 0; o < ly->out; ++o) nx[o] = ly->bias[o];
                    for (int t = 0; t < k; ++t) {
                        const int8_t *col = ly->WT + (size_t)idx[t] * ly->out;
                        for (int o = 0; o < ly->out; ++o) nx[o] += col[o];
                    }
                }
                for (int o = 0; o < ly->out; ++o) {
                    int32_t acc = nx[o];
                    if (l > 0) {
                        const int8_t *w = ly->W + (size_t)o * ly->in;
                        int32_t dot = 0;
                        for (int t = 0; t < ly->in; ++t) dot += (int32_t)w[t] * (int32_t)a[t];
                        acc = ly->bias[o] + dot;
                    }
                    if (l < m->L) {
                        int32_t v = acc >> ly->shift; /* arithmetic: floor division */
                        nx2[o] = v < 0 ? 0 : (v > 255 ? 255 : v);
                    } else {
                        lg[o] = (double)acc * (double)m->out_scale[e];
                    }
                }
                if (l < m->L)
                    for (int o = 0; o < ly->out; ++o) a[o] = (uint8_t)nx2[o];
            }
            if (logits_out) memcpy(logits_out + ((size_t)i * m->E + e) * m->C, lg, sizeof(double) * m->C);
            orc_softmax(lg, m->C, p);
            int err = ORC_OK;
            const int h = orc_quantile_class(p, m->C, q, &err);
            if (err != ORC_OK) { rc = err; break; }
            if (e == 0 || h < best) best = h;
        }
        h_out[i] = best;
    }
    free(a);
    free(nx);
    free(nx2);
    free(lg);
    free(p);
    return rc;
}

typedef struct {
    const orc_mlp *m;
    int domain;
    double q;
    const void *packed;
    int64_t lo, hi;
    int32_t *h;
    double *logits;
    int rc;
} mlp_job;

static void *mlp_job_run(void *arg) {
    mlp_job *j = (mlp_job *)arg;
    j->rc = mlp_eval_range(j->m, j->domain, j->q, j->packed, j->lo, j->hi, j->h, j->logits);
    return NULL;
}

/* Whole-batch BMLP1 evaluation, split over `threads` pthreads (contiguous
 * shards); threads <= 1 runs inline. */
int orc_mlp_evaluate(const orc_mlp *m, int domain, double q, const void *packed, int64_t n,
                     int32_t *h_out, double *logits_out, int threads) {
    if (orc_feature_length(domain) != m->F) return ORC_ERR_ARG;
    if (q <= 0.0 || q > 1.0) return ORC_ERR_QUANTILE;
    if (threads <= 1 || n < threads)
        return mlp_eval_range(m, domain, q, packed, 0, n, h_out, logits_out);
    mlp_job *jobs = (mlp_job *)calloc(threads, sizeof(mlp_job));
    pthread_t *th = (pthread_t *)calloc(threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (mlp_job){m, domain, q, packed, n * t / threads, n * (t + 1) / threads, h_out,
                            logits_out, 0};
        pthread_create(&th[t], NULL, mlp_job_run, &jobs[t]);
    }
    int rc = ORC_OK;
    for (int t = 0; t < threads; ++t) {
        pthread_join(th[t], NULL);
        if (jobs[t].rc != ORC_OK) rc = jobs[t].rc;
    }
    free(jobs);
    free(th);
    return rc;
}

/* Convenience for ctypes: parse + evaluate + free in one call. */
int orc_mlp_evaluate_blob(const void *blob, size_t len, int domain, double q, const void *packed,
                          int64_t n, int32_t *h_out, double *logits_out, int threads) {
    orc_mlp m;
    int rc = orc_bmlp1_parse(blob, len, orc_feature_length(domain), &m);
    if (rc != ORC_OK) return rc;
    rc = orc_mlp_evaluate(&m, domain, q, packed, n, h_out, logits_out, threads);
    orc_mlp_free(&m);
    return rc;
}

/* ------------------------------------------------------------ utilities */

/* ManhattanHeuristic<N>::lookup (heuristic.hpp:76-89) on packed states. */
int orc_manhattan(int domain, const void *packed, int64_t n, int32_t *out) {
    if (domain < ORC_STP2 || domain > ORC_STP4) return ORC_ERR_ARG;
    const int N = domain, K = N * N;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t v;
        memcpy(&v, (const char *)packed + i * 8, 8);
        int sum = 0;
        for (int cell = 0; cell < K; ++cell) {
            const int t = (int)((v >> (4 * cell)) & 0xF);
            if (t == 0) continue;
            sum += abs(cell / N - t / N) + abs(cell % N - t % N);
        }
        out[i] = sum;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ PDBs */

/* partial_perm_rank (ranking.hpp:26-51): lexicographic rank of seq[0..m) among
 * length-m sequences of distinct values from {0..n-1}.  -1 on repeats. */
int64_t orc_partial_perm_rank(const int *seq, int m, int n) {
    int64_t rank = 0;
    for (int i = 0; i < m; ++i) {
        int smaller = 0;
        for (int j = 0; j < i; ++j) {
            if (seq[j] == seq[i]) return -1;
            if (seq[j] < seq[i]) ++smaller;
        }
        if (seq[i] < 0 || seq[i] >= n) return -1;
        const int idx = seq[i] - smaller; /* index among the still-available values */
        int64_t w = 1;
        for (int a = 0; a < m - i - 1; ++a) w *= (int64_t)(n - i - 1 - a);
        rank += (int64_t)idx * w;
    }
    return rank;
}

/* Abstraction::rank_state: RubiksCube corners (rubiks.hpp:247-267: pos/ori of
 * each pattern corner, partial_perm_rank(pos, 8) then *3 + ori per corner) and
 * TilePuzzle (stp.hpp:208-227: cell of each pattern tile, partial_perm_rank(pos,
 * N*N)).  The last matching position wins, as in project().  -1 if invalid. */
int64_t orc_pdb_rank(int domain, const uint8_t *pattern, int m, const void *packed) {
    int pos[16], ori[16];
    if (domain == ORC_RC) {
        uint64_t lo;
        memcpy(&lo, packed, 8);
        for (int i = 0; i < m; ++i) {
            pos[i] = -1;
            ori[i] = 0;
            for (int p = 0; p < 8; ++p)
                if ((int)((lo >> (3 * p)) & 7) == pattern[i]) {
                    pos[i] = p;
                    ori[i] = (int)((lo >> (24 + 2 * p)) & 3);
                }
        }
        int64_t r = orc_partial_perm_rank(pos, m, 8);
        if (r < 0) return -1;
        for (int i = 0; i < m; ++i) r = r * 3 + ori[i];
        return r;
    }
    if (domain >= ORC_STP2 && domain <= ORC_STP4) {
        const int K = domain * domain;
        uint64_t v;
        memcpy(&v, packed, 8);
        for (int i = 0; i < m; ++i) {
            pos[i] = -1;
            for (int cell = 0; cell < K; ++cell)
                if ((int)((v >> (4 * cell)) & 0xF) == pattern[i]) pos[i] = cell;
        }
        return orc_partial_perm_rank(pos, m, K);
    }
    return -1;
}

/* PdbTable::lookup (pdb.hpp:66-69): unreachable entries (0xFF) read as 0. */
int orc_pdb_lookup(int domain, const uint8_t *pattern, int m, const uint8_t *entries, uint64_t n_entries,
                   const void *packed, int64_t n, int32_t *out) {
    const int pb = orc_packed_bytes(domain);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t r = orc_pdb_rank(domain, pattern, m, (const char *)packed + i * pb);
        if (r < 0 || (uint64_t)r >= n_entries) return ORC_ERR_ARG;
        const uint8_t e = entries[r];
        out[i] = e == 0xFF ? 0 : e;
    }
    return ORC_OK;
}
