// bida_search.cpp — the builder's search driver: the reference's own Batch
// IDA* / AIDA* (search.hpp:101-247, unchanged) with evaluators chosen per run:
//   gpu : bida_gpu::GpuBackend<D> (include/bida_gpu_backend.hpp) per evaluator
//   cpu : the reference's LinearModelBackend (BLIN1); BMLP1 on the CPU only in
//         the test build (-DBIDA_WITH_ORACLE, tests/cpp/bin/search_parity),
//         where the oracle's C restatement stands in (the reference has no MLP)
//   pdb : the reference's PdbTable lookups only (AIDA* baseline)
// It prints one JSON line per (instance, backend): cost, status, threshold
// history, per-iteration counts, nodes/s, evals/s.  tools/bin/bida_search is
// the product build (no oracle linked); tests/test_gpu_search.py drives the
// test build to check GPU and CPU searches agree.
//
//   search_parity --domain stp4 --instances korf10.txt --model linear:w.blin --q 0.5 \
//                 --threads 8 --work-num 16 --batch 4096 --timeout-us 200 --evaluators 1 --mode both
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "bida/search.hpp"
#include "bida_gpu_backend.hpp"
#ifdef BIDA_WITH_ORACLE
#include "../oracle/bida_oracle.h"
#endif

using namespace bida;

namespace {

struct Args {
    std::string domain = "stp4", instances, model, mode = "both";
    std::string walks;  // n:len_min:len_max:seed
    double q = 0.5, time_limit = 0.0;
    int threads = 4, work_num = 4, evaluators = 1, d_init = -1, first = 0, count = 1 << 30;
    std::size_t batch = 1024;
    long long timeout_us = 200;
    int gpus = 1;
    bool immediate = false;  // AIDA*: evaluate inline on the searcher threads
    int table1_corners = 0;  // >0: "Table-1" mode with an N-corner PDB (Rubik's)
    bool gpu_pdb = false;    // Table-1 on the GPU: PDB lookup fused into the device readout
    std::string algo = "batch-idastar";  // or "batch-astar" (search.hpp:350-503)
};

// Table-1 mode: the network is evaluated for
// every node (its cost is real) but the search is guided by the admissible
// PDB value, so CPU and GPU runs expand identical trees.  `pdb_only` skips the
// network (the AIDA*-with-PDB baseline).
template <class D>
class Table1Backend final : public EvaluatorBackend<D> {
public:
    Table1Backend(std::unique_ptr<EvaluatorBackend<D>> nn, std::shared_ptr<const Heuristic<D>> pdb)
        : nn_(std::move(nn)), pdb_(std::move(pdb)) {}
    bool needs_features() const override { return nn_ && nn_->needs_features(); }
    void evaluate(std::span<const BatchItem<D>> batch, std::span<std::int32_t> out) override {
        if (nn_)
            nn_->evaluate(batch, out);  // h_NN computed (and discarded, as in the paper)
        for (std::size_t i = 0; i < batch.size(); ++i)
            out[i] = static_cast<std::int32_t>(pdb_->lookup(batch[i].state));
    }

private:
    std::unique_ptr<EvaluatorBackend<D>> nn_;
    std::shared_ptr<const Heuristic<D>> pdb_;
};

inline std::string corner_pdb_path(int corners) {
    return "/tmp/bida_rc_corner" + std::to_string(corners) + ".pdb";
}

bool g_pdb_build_gpu = false;  // --pdb-build gpu

template <class D>
std::shared_ptr<const Heuristic<D>> corner_pdb(int corners) {
    if constexpr (std::is_same_v<D, RubiksCube>) {
        std::vector<std::uint8_t> pat;
        for (int c = 0; c < corners; ++c)
            pat.push_back(static_cast<std::uint8_t>(c));
        const std::string cache = corner_pdb_path(corners);
        std::shared_ptr<const PdbTable<D>> t;
        try {
            t = std::make_shared<const PdbTable<D>>(PdbTable<D>::load(cache));
        } catch (const std::exception &) {
            if (g_pdb_build_gpu) {
                // PdbTable<D>::build on the GPU (bida_gpu_pdb_build_save): the same
                // bytes in ~0.6 s instead of ~700 s for 8 corners; the reference's
                // PdbTable::load reads it back (and checks the goal entry)
                if (bida_gpu_pdb_build_save(0, BIDA_DOMAIN_RC, pat.data(), static_cast<int>(pat.size()),
                                            cache.c_str()) != BIDA_OK)
                    throw std::runtime_error(std::string("GPU PDB build: ") + bida_gpu_last_error());
                t = std::make_shared<const PdbTable<D>>(PdbTable<D>::load(cache));
            } else {
                auto built = PdbTable<D>::build(pat, D::solved());
                built.save(cache);
                t = std::make_shared<const PdbTable<D>>(std::move(built));
            }
        }
        return std::make_shared<const PdbHeuristic<D>>(t);
    } else {
        throw std::runtime_error("--table1-pdb needs --domain rc");
    }
}

std::vector<unsigned char> read_all(const std::string &p) {
    std::ifstream f(p, std::ios::binary);
    if (!f)
        throw std::runtime_error("cannot open " + p);
    return std::vector<unsigned char>(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}

#ifdef BIDA_WITH_ORACLE
// CPU BMLP1 backend over the oracle restatement (test infrastructure).
template <class D>
class OracleMlpBackend final : public EvaluatorBackend<D> {
public:
    OracleMlpBackend(const std::string &path, double q) : q_(q) {
        blob_ = read_all(path);
        if (orc_bmlp1_parse(blob_.data(), blob_.size(), D::feature_length(), &m_) != ORC_OK)
            throw std::runtime_error("bad BMLP1 file " + path);
    }
    ~OracleMlpBackend() override { orc_mlp_free(&m_); }
    void evaluate(std::span<const BatchItem<D>> batch, std::span<std::int32_t> out) override {
        std::vector<unsigned char> packed(batch.size() * bida_gpu::DomainOf<D>::packed_bytes);
        for (std::size_t i = 0; i < batch.size(); ++i)
            bida_gpu::DomainOf<D>::pack(batch[i].state, packed.data() + i * bida_gpu::DomainOf<D>::packed_bytes);
        orc_mlp_evaluate(&m_, bida_gpu::DomainOf<D>::id, q_, packed.data(), static_cast<int64_t>(batch.size()),
                         out.data(), nullptr, 1);
    }

private:
    std::vector<unsigned char> blob_;
    orc_mlp m_{};
    double q_;
};
#endif

template <class D>
std::vector<std::unique_ptr<EvaluatorBackend<D>>> make_backends(const Args &a, bool gpu);

template <class D>
std::vector<std::unique_ptr<EvaluatorBackend<D>>> make_mode_backends(const Args &a, const std::string &mode) {
    if (a.table1_corners <= 0)
        return make_backends<D>(a, mode == "gpu");
    const auto pdb = corner_pdb<D>(a.table1_corners);
    std::vector<std::unique_ptr<EvaluatorBackend<D>>> v;
    if (mode == "pdb") {
        for (int e = 0; e < a.evaluators; ++e)
            v.push_back(std::make_unique<Table1Backend<D>>(nullptr, pdb));
        return v;
    }
    if (mode == "gpu" && a.gpu_pdb) {
        // the network and the PDB lookup both run in the device readout
        for (auto &b : make_backends<D>(a, true)) {
            static_cast<bida_gpu::GpuBackend<D> *>(b.get())->attach_pdb_file(corner_pdb_path(a.table1_corners),
                                                                             BIDA_PDB_REPLACE);
            v.push_back(std::move(b));
        }
        return v;
    }
    for (auto &b : make_backends<D>(a, mode == "gpu"))
        v.push_back(std::make_unique<Table1Backend<D>>(std::move(b), pdb));
    return v;
}

template <class D>
std::vector<std::unique_ptr<EvaluatorBackend<D>>> make_backends(const Args &a, bool gpu) {
    const auto colon = a.model.find(':');
    const std::string kind = a.model.substr(0, colon), path = a.model.substr(colon + 1);
    std::vector<std::unique_ptr<EvaluatorBackend<D>>> v;
    for (int e = 0; e < a.evaluators; ++e) {
        const int dev = e % std::max(1, a.gpus);
        if (kind == "linear") {
            if (gpu)
                v.push_back(bida_gpu::GpuBackend<D>::load_linear(dev, path, a.q));
            else
                v.push_back(std::make_unique<LinearModelBackend<D>>(LinearModelBackend<D>::load(path, a.q)));
        } else if (kind == "mlp") {
            if (gpu)
                v.push_back(bida_gpu::GpuBackend<D>::load_mlp(dev, path, a.q));
            else
#ifdef BIDA_WITH_ORACLE
                v.push_back(std::make_unique<OracleMlpBackend<D>>(path, a.q));
#else
                throw std::runtime_error("BMLP1 on the CPU needs the test build (tests/cpp/bin/search_parity)");
#endif
        } else {
            throw std::runtime_error("model must be linear:PATH or mlp:PATH");
        }
    }
    return v;
}

template <class D>
std::vector<Instance<D>> get_instances(const Args &a) {
    if (!a.instances.empty())
        return load_instances<D>(a.instances);
    int n = 0, lmin = 0, lmax = 0;
    unsigned long long seed = 0;
    if (std::sscanf(a.walks.c_str(), "%d:%d:%d:%llu", &n, &lmin, &lmax, &seed) != 4)
        throw std::runtime_error("--walks n:len_min:len_max:seed");
    std::vector<Instance<D>> v;
    for (int i = 0; i < n; ++i)
        v.push_back(random_walk_instance<D>(D::solved(), lmin + i % (lmax - lmin + 1), seed + i));
    return v;
}

#ifdef BIDA_RING_EVALUATOR
constexpr const char *kEvaluatorImpl = "ring"; // include/bida_ring_evaluator.hpp
#else
constexpr const char *kEvaluatorImpl = "reference"; // batch_eval.hpp:193-473
#endif
#ifdef BIDA_FAST_CBDFS
constexpr const char *kSearchImpl = "fast"; // include/bida_fast_cbdfs.hpp
#else
constexpr const char *kSearchImpl = "reference"; // cbdfs.hpp:254-415
#endif

const char *status_name(SearchStatus s) {
    switch (s) {
    case SearchStatus::Solved: return "solved";
    case SearchStatus::TimedOut: return "timeout";
    default: return "budget";
    }
}

template <class D>
int run(const Args &a) {
    const auto insts = get_instances<D>(a);
    SearchConfig cfg;
    cfg.threads = a.threads;
    cfg.work_num = a.work_num;
    cfg.batch_size = a.batch;
    cfg.timeout_us = a.timeout_us;
    cfg.evaluators = a.evaluators;
    cfg.d_init = a.d_init;
    cfg.time_limit_s = a.time_limit;
    std::vector<std::string> modes;
    if (a.mode == "both" || a.mode == "cpu")
        modes.push_back("cpu");
    if (a.mode == "both" || a.mode == "gpu")
        modes.push_back("gpu");
    if (a.mode == "pdb")
        modes.push_back("pdb");
    for (const std::string &mode : modes) {
        EvaluatorGroup<D> group(make_mode_backends<D>(a, mode), a.batch, a.timeout_us, a.immediate);
        for (int i = a.first; i < static_cast<int>(insts.size()) && i < a.first + a.count; ++i) {
            const SearchResult<D> r = a.algo == "batch-astar"
                                          ? batch_astar<D>(insts[static_cast<std::size_t>(i)], group, cfg)
                                          : batch_idastar<D>(insts[static_cast<std::size_t>(i)], group, cfg);
            const SearchStats &s = r.stats;
            std::ostringstream js;
            js << "{\"instance\": " << i << ", \"mode\": \"" << mode << "\", \"status\": \"" << status_name(r.status)
               << "\", \"cost\": " << r.cost << ", \"expanded\": " << s.expanded << ", \"generated\": " << s.generated
               << ", \"batches\": " << s.batches << ", \"batch_items\": " << s.batch_items
               << ", \"sync_evaluations\": " << s.sync_evaluations << ", \"forced_flushes\": " << s.forced_flushes
               << ", \"assertion_violations\": " << s.assertion_violations << ", \"wall_s\": " << s.wall_seconds
               << ", \"nodes_per_s\": " << (s.wall_seconds > 0 ? s.generated / s.wall_seconds : 0.0)
               << ", \"evals_per_s\": " << (s.wall_seconds > 0 ? s.batch_items / s.wall_seconds : 0.0)
               << ", \"mean_batch\": " << s.mean_batch() << ", \"thresholds\": [";
            for (std::size_t k = 0; k < r.threshold_history.size(); ++k)
                js << (k ? ", " : "") << r.threshold_history[k];
            js << "], \"iterations\": [";
            for (std::size_t k = 0; k < s.iterations.size(); ++k) {
                const auto &it = s.iterations[k];
                js << (k ? ", " : "") << "[" << it.threshold << ", " << it.expanded << ", " << it.generated << ", "
                   << it.batches << ", " << it.batch_items << "]";
            }
            js << "], \"threads\": " << a.threads << ", \"work_num\": " << a.work_num << ", \"batch\": " << a.batch
               << ", \"timeout_us\": " << a.timeout_us << ", \"evaluators\": " << a.evaluators
               << ", \"evaluator_impl\": \"" << kEvaluatorImpl << "\""
               << ", \"search_impl\": \"" << kSearchImpl << "\"" << ", \"solution\": [";
            for (std::size_t k = 0; k < r.solution.size(); ++k)
                js << (k ? ", " : "") << static_cast<int>(r.solution[k]);
            js << "]"
               << ", \"immediate\": " << (a.immediate ? "true" : "false")
               << ", \"table1_corners\": " << a.table1_corners << ", \"gpu_pdb\": " << (a.gpu_pdb ? "true" : "false")
               << ", \"algo\": \"" << a.algo << "\"}";
            std::printf("%s\n", js.str().c_str());
            std::fflush(stdout);
        }
        group.close();
    }
    return 0;
}

} // namespace

int main(int argc, char **argv) {
    Args a;
    for (int i = 1; i < argc; ++i) {
        const std::string k = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc)
                throw std::runtime_error("missing value for " + k);
            return argv[++i];
        };
        if (k == "--domain") a.domain = val();
        else if (k == "--instances") a.instances = val();
        else if (k == "--walks") a.walks = val();
        else if (k == "--model") a.model = val();
        else if (k == "--mode") a.mode = val();
        else if (k == "--q") a.q = std::stod(val());
        else if (k == "--threads") a.threads = std::stoi(val());
        else if (k == "--work-num") a.work_num = std::stoi(val());
        else if (k == "--batch") a.batch = static_cast<std::size_t>(std::stoull(val()));
        else if (k == "--timeout-us") a.timeout_us = std::stoll(val());
        else if (k == "--evaluators") a.evaluators = std::stoi(val());
        else if (k == "--gpus") a.gpus = std::stoi(val());
        else if (k == "--d-init") a.d_init = std::stoi(val());
        else if (k == "--time-limit") a.time_limit = std::stod(val());
        else if (k == "--first") a.first = std::stoi(val());
        else if (k == "--count") a.count = std::stoi(val());
        else if (k == "--immediate") a.immediate = true;
        else if (k == "--table1-pdb") a.table1_corners = std::stoi(val());
        else if (k == "--gpu-pdb") a.gpu_pdb = true;
        else if (k == "--algo") a.algo = val();
        else if (k == "--pdb-build") g_pdb_build_gpu = val() == "gpu";
        else {
            std::fprintf(stderr, "unknown flag %s\n", k.c_str());
            return 2;
        }
    }
    try {
        if (a.domain == "stp3") return run<TilePuzzle<3>>(a);
        if (a.domain == "stp4") return run<TilePuzzle<4>>(a);
        if (a.domain == "rc") return run<RubiksCube>(a);
        std::fprintf(stderr, "unknown domain %s\n", a.domain.c_str());
        return 2;
    } catch (const std::exception &e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
