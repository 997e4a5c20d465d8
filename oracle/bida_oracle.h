/* bida_oracle.h — TEST INFRASTRUCTURE ONLY: CPU restatement of the reference
 * evaluator path (see bida_oracle.c).  Never linked by the product. */
#pragma once
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_STP2 = 2, ORC_STP3 = 3, ORC_STP4 = 4, ORC_RC = 100 };
enum {
    ORC_OK = 0,
    ORC_ERR_ARG = 1,
    ORC_ERR_QUANTILE = 2,
    ORC_ERR_DISTRIBUTION = 3,
    ORC_ERR_FORMAT = 4,
    ORC_ERR_TRUNCATED = 5,
};

#define ORC_MLP_MAX_LAYERS 8

typedef struct {
    int in, out, shift;
    int8_t *W;
    int32_t *bias;
    int8_t *WT; /* layer 0 only: W transposed [in][out] (sparse one-hot input) */
} orc_mlp_layer;

typedef struct {
    int F, C, E, L;
    int H[ORC_MLP_MAX_LAYERS];
    orc_mlp_layer *layers; /* [E][L+1] */
    float *out_scale;      /* [E] */
} orc_mlp;

int orc_feature_length(int domain);
int orc_packed_bytes(int domain);
int orc_active_features(int domain);
int orc_active_indices(int domain, const void *packed, int *idx);
int orc_encode(int domain, const void *packed, int64_t n, float *out);
int orc_quantile_class(const double *p, int C, double q, int *err);
void orc_softmax(const double *logits, int C, double *p);
int orc_linear_evaluate(int domain, const float *W, int E, int C, double q, const void *packed,
                        int64_t n, int32_t *h_out, double *logits_out);
int orc_blin1_parse(const void *blob, size_t len, int F_expected, int *C, int *E, float **W);
int orc_bmlp1_parse(const void *blob, size_t len, int F_expected, orc_mlp *m);
void orc_mlp_free(orc_mlp *m);
int orc_mlp_evaluate(const orc_mlp *m, int domain, double q, const void *packed, int64_t n,
                     int32_t *h_out, double *logits_out, int threads);
int orc_mlp_evaluate_blob(const void *blob, size_t len, int domain, double q, const void *packed,
                          int64_t n, int32_t *h_out, double *logits_out, int threads);
int orc_manhattan(int domain, const void *packed, int64_t n, int32_t *out);

#ifdef __cplusplus
}
#endif

#ifdef __cplusplus
extern "C" {
#endif
int64_t orc_partial_perm_rank(const int *seq, int m, int n);
int64_t orc_pdb_rank(int domain, const uint8_t *pattern, int m, const void *packed);
int orc_pdb_lookup(int domain, const uint8_t *pattern, int m, const uint8_t *entries, uint64_t n_entries,
                   const void *packed, int64_t n, int32_t *out);
#ifdef __cplusplus
}
#endif
