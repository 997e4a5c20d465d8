// mlp.cu — placeholder until the tcgen05 MLP kernel lands.
#include "mlp.cuh"

namespace bida_gpu {

struct MlpModel {};
static thread_local std::string g_mlp_err;

int mlp_create(const unsigned char *, size_t, int, double, int, MlpModel **out, MlpShape *,
               std::string *err) {
    *out = nullptr;
    *err = "BMLP1 evaluator not built yet";
    return 2;
}
int mlp_launch(MlpModel *, int, const void *, int64_t, int32_t *, double *, int *, cudaStream_t,
               std::atomic<int64_t> *) {
    g_mlp_err = "BMLP1 evaluator not built yet";
    return 1;
}
void mlp_destroy(MlpModel *m) { delete m; }
const char *mlp_last_error() { return g_mlp_err.c_str(); }

} // namespace bida_gpu
