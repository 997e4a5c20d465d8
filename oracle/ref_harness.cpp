// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.
//
// Compiles the reference's own header-only library UNCHANGED (from
// $(BIDA_REF_INCLUDE), default /root/reference/proj/include) into
// oracle/_ref/libbida_ref.so and exposes a few extern "C" entry points so the
// Python tests can run the real reference evaluator on the same packed states
// and weights as the CUDA path.  Nothing here is copied from the reference;
// it only calls it.  Built by oracle/Makefile; never shipped in the product.
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "bida/batch_eval.hpp"
#include "bida/heuristic.hpp"
#include "bida/instance.hpp"
#include "bida/rubiks.hpp"
#include "bida/stp.hpp"

using namespace bida;

namespace {

template <class P>
using bare_t = std::remove_cv_t<std::remove_pointer_t<P>>;

enum { D_STP2 = 2, D_STP3 = 3, D_STP4 = 4, D_RC = 100 };
enum { RH_OK = 0, RH_ERR_ARG = 1, RH_ERR_INVALID = 2, RH_ERR_RUNTIME = 3 };

thread_local std::string g_err;

template <int N>
typename TilePuzzle<N>::State unpack(const TilePuzzle<N> *, const void *p) {
    std::uint64_t v;
    std::memcpy(&v, p, 8);
    typename TilePuzzle<N>::State s;
    for (int c = 0; c < N * N; ++c) {
        s.tiles[static_cast<std::size_t>(c)] = static_cast<std::uint8_t>((v >> (4 * c)) & 0xF);
        if (s.tiles[static_cast<std::size_t>(c)] == 0)
            s.blank = static_cast<std::uint8_t>(c);
    }
    return s;
}

RubiksCube::State unpack(const RubiksCube *, const void *p) {
    std::uint64_t lo, hi;
    std::memcpy(&lo, p, 8);
    std::memcpy(&hi, static_cast<const char *>(p) + 8, 8);
    RubiksCube::State s;
    for (int i = 0; i < 8; ++i) {
        s.cp[static_cast<std::size_t>(i)] = static_cast<std::uint8_t>((lo >> (3 * i)) & 7);
        s.co[static_cast<std::size_t>(i)] = static_cast<std::uint8_t>((lo >> (24 + 2 * i)) & 3);
    }
    for (int i = 0; i < 12; ++i) {
        s.eo[static_cast<std::size_t>(i)] = static_cast<std::uint8_t>((lo >> (40 + i)) & 1);
        s.ep[static_cast<std::size_t>(i)] = static_cast<std::uint8_t>((hi >> (4 * i)) & 0xF);
    }
    return s;
}

template <int N>
void pack_into(const typename TilePuzzle<N>::State &s, void *out) {
    const std::uint64_t v = TilePuzzle<N>::pack(s);
    std::memcpy(out, &v, 8);
}
void pack_into_rc(const RubiksCube::State &s, void *out) {
    const RubiksCube::Packed p = RubiksCube::pack(s);
    std::memcpy(out, &p.lo, 8);
    std::memcpy(static_cast<char *>(out) + 8, &p.hi, 8);
}

template <class D>
constexpr int packed_bytes() {
    if constexpr (std::is_same_v<D, RubiksCube>)
        return 16;
    else
        return 8;
}

template <class D>
void pack_state(const typename D::State &s, void *out) {
    if constexpr (std::is_same_v<D, RubiksCube>)
        pack_into_rc(s, out);
    else if constexpr (std::is_same_v<D, TilePuzzle<2>>)
        pack_into<2>(s, out);
    else if constexpr (std::is_same_v<D, TilePuzzle<3>>)
        pack_into<3>(s, out);
    else
        pack_into<4>(s, out);
}

template <class F>
int dispatch(int domain, F &&f) {
    try {
        switch (domain) {
        case D_STP2: return f(static_cast<const TilePuzzle<2> *>(nullptr));
        case D_STP3: return f(static_cast<const TilePuzzle<3> *>(nullptr));
        case D_STP4: return f(static_cast<const TilePuzzle<4> *>(nullptr));
        case D_RC: return f(static_cast<const RubiksCube *>(nullptr));
        default: g_err = "unknown domain"; return RH_ERR_ARG;
        }
    } catch (const std::invalid_argument &e) {
        g_err = e.what();
        return RH_ERR_INVALID;
    } catch (const std::exception &e) {
        g_err = e.what();
        return RH_ERR_RUNTIME;
    }
}

template <class D>
std::vector<BatchItem<D>> make_items(const void *packed, std::int64_t n) {
    std::vector<BatchItem<D>> items(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) {
        auto &it = items[static_cast<std::size_t>(i)];
        it.state = unpack(static_cast<const D *>(nullptr),
                          static_cast<const char *>(packed) + i * packed_bytes<D>());
        it.features.resize(static_cast<std::size_t>(D::feature_length()));
        D::encode(it.state, it.features.data());
    }
    return items;
}

template <class D>
int run_backend_mt(EvaluatorBackend<D> &backend, const std::vector<BatchItem<D>> &items,
                   std::int32_t *h_out, int threads) {
    const std::size_t n = items.size();
    if (threads <= 1 || n < static_cast<std::size_t>(threads)) {
        backend.evaluate(items, std::span<std::int32_t>(h_out, n));
        return RH_OK;
    }
    std::vector<std::thread> th;
    std::vector<std::string> errs(static_cast<std::size_t>(threads));
    for (int t = 0; t < threads; ++t) {
        const std::size_t lo = n * static_cast<std::size_t>(t) / static_cast<std::size_t>(threads);
        const std::size_t hi = n * static_cast<std::size_t>(t + 1) / static_cast<std::size_t>(threads);
        th.emplace_back([&, lo, hi, t] {
            try {
                backend.evaluate(std::span<const BatchItem<D>>(items.data() + lo, hi - lo),
                                 std::span<std::int32_t>(h_out + lo, hi - lo));
            } catch (const std::exception &e) {
                errs[static_cast<std::size_t>(t)] = e.what();
            }
        });
    }
    for (auto &x : th)
        x.join();
    for (auto &e : errs)
        if (!e.empty())
            throw std::invalid_argument(e);
    return RH_OK;
}

} // namespace

extern "C" {

const char *ref_last_error() { return g_err.c_str(); }

int ref_feature_length(int domain) {
    return dispatch(domain, [](auto *d) { return bare_t<decltype(d)>::feature_length(); });
}

// Seeded random walks through the reference's random_walk_instance
// (instance.hpp:36-57): state i is a walk of length len_min + i % span from
// the solved state with seed `seed + i`, packed with D::pack.
int ref_random_walk_packed(int domain, std::int64_t n, int len_min, int len_max,
                           std::uint64_t seed, void *out_packed) {
    if (len_max < len_min || len_min < 0) {
        g_err = "bad walk lengths";
        return RH_ERR_ARG;
    }
    return dispatch(domain, [&](auto *d) {
        using D = bare_t<decltype(d)>;
        const int span = len_max - len_min + 1;
        for (std::int64_t i = 0; i < n; ++i) {
            const int L = len_min + static_cast<int>(i % span);
            const Instance<D> inst =
                random_walk_instance<D>(D::solved(), L, seed + static_cast<std::uint64_t>(i));
            pack_state<D>(inst.start, static_cast<char *>(out_packed) + i * packed_bytes<D>());
        }
        return RH_OK;
    });
}

// Round trip through the reference pack: out = D::pack(unpack(in)).
int ref_repack(int domain, const void *packed, std::int64_t n, void *out) {
    return dispatch(domain, [&](auto *d) {
        using D = bare_t<decltype(d)>;
        for (std::int64_t i = 0; i < n; ++i) {
            const auto s = unpack(d, static_cast<const char *>(packed) + i * packed_bytes<D>());
            if (!D::valid(s))
                throw std::invalid_argument("packed state " + std::to_string(i) + " is not valid");
            pack_state<D>(s, static_cast<char *>(out) + i * packed_bytes<D>());
        }
        return RH_OK;
    });
}

// D::encode (stp.hpp:141-146, rubiks.hpp:155-166) into dense float rows.
int ref_encode(int domain, const void *packed, std::int64_t n, float *out) {
    return dispatch(domain, [&](auto *d) {
        using D = bare_t<decltype(d)>;
        for (std::int64_t i = 0; i < n; ++i) {
            const auto s = unpack(d, static_cast<const char *>(packed) + i * packed_bytes<D>());
            D::encode(s, out + i * D::feature_length());
        }
        return RH_OK;
    });
}

// LinearModelBackend<D>::evaluate (batch_eval.hpp:98-105) over n packed
// states, weights W[E][C][F]; `threads` > 1 splits the batch into contiguous
// shards evaluated concurrently on the same backend (the all-core CPU
// evaluator of BASELINE.md §3).
int ref_linear_evaluate(int domain, const float *W, int E, int C, double q, const void *packed,
                        std::int64_t n, std::int32_t *h_out, int threads) {
    return dispatch(domain, [&](auto *d) {
        using D = bare_t<decltype(d)>;
        const std::size_t per = static_cast<std::size_t>(C) * D::feature_length();
        std::vector<std::vector<float>> w(static_cast<std::size_t>(E));
        for (int m = 0; m < E; ++m)
            w[static_cast<std::size_t>(m)].assign(W + m * per, W + (m + 1) * per);
        LinearModelBackend<D> backend(std::move(w), C, q);
        const auto items = make_items<D>(packed, n);
        return run_backend_mt<D>(backend, items, h_out, threads);
    });
}

// The reference's own LinearModelBackend::evaluate (score's softmax,
// quantile_class, ensemble_min: batch_eval.hpp:98-105,148-168,
// heuristic.hpp:95-126) applied to ARBITRARY per-(state, member, class)
// logits of the form (double)acc * (double)scale, acc int32, scale float --
// the BMLP1 output layer, which the reference does not have.
//
// score() computes sum_j (double)w[c][j] * (double)x[j] over F float
// features.  For member m, class c we use two feature slots
// j0 = 2(mC + c), j1 = j0 + 1 holding the split acc = hi + lo
// (lo = acc & 4095, hi = acc - lo: both exact in float), and put the member's
// scale at w_m[c][j0] = w_m[c][j1]; every other weight is 0.  Both products
// are exact in double, the running sum is exactly 0 before j0, so the sum
// rounds ONCE to round(acc * scale) == (double)acc * (double)scale, and the
// later +-0.0 terms do not change it.  Needs 2*E*C <= F.
int ref_readout_scaled_logits(int domain, const std::int32_t *acc, const float *scale, int E, int C,
                              double q, std::int64_t n, std::int32_t *h_out, int threads) {
    return dispatch(domain, [&](auto *d) {
        using D = bare_t<decltype(d)>;
        const int F = D::feature_length();
        if (2 * E * C > F)
            throw std::invalid_argument("ref_readout_scaled_logits: 2*E*C exceeds the feature length");
        std::vector<std::vector<float>> w(static_cast<std::size_t>(E),
                                          std::vector<float>(static_cast<std::size_t>(C) * F, 0.0f));
        for (int m = 0; m < E; ++m)
            for (int c = 0; c < C; ++c) {
                const std::size_t j0 = static_cast<std::size_t>(2 * (m * C + c));
                w[static_cast<std::size_t>(m)][static_cast<std::size_t>(c) * F + j0] = scale[m];
                w[static_cast<std::size_t>(m)][static_cast<std::size_t>(c) * F + j0 + 1] = scale[m];
            }
        LinearModelBackend<D> backend(std::move(w), C, q);
        std::vector<BatchItem<D>> items(static_cast<std::size_t>(n));
        for (std::int64_t i = 0; i < n; ++i) {
            FeatureVector &x = items[static_cast<std::size_t>(i)].features;
            x.assign(static_cast<std::size_t>(F), 0.0f);
            for (int m = 0; m < E; ++m)
                for (int c = 0; c < C; ++c) {
                    const std::int32_t a = acc[(i * E + m) * C + c];
                    const std::int32_t lo = a & 4095;
                    const std::size_t j0 = static_cast<std::size_t>(2 * (m * C + c));
                    x[j0] = static_cast<float>(static_cast<std::int64_t>(a) - lo);
                    x[j0 + 1] = static_cast<float>(lo);
                }
        }
        return run_backend_mt<D>(backend, items, h_out, threads);
    });
}

// Same, with the encode done once up front and timed separately by the
// caller: returns an opaque prepared batch (for the CPU baseline, so the
// timed region is LinearModelBackend::evaluate only, like the GPU's kernel).
void *ref_linear_prepare(int domain, const float *W, int E, int C, double q, const void *packed,
                         std::int64_t n);
int ref_linear_run(void *prepared, std::int32_t *h_out, int threads);
void ref_linear_release(void *prepared);

// BLIN1 I/O through the reference (batch_eval.hpp:109-145).
int ref_blin1_save(int domain, const char *path, const float *W, int E, int C) {
    return dispatch(domain, [&](auto *d) {
        using D = bare_t<decltype(d)>;
        const std::size_t per = static_cast<std::size_t>(C) * D::feature_length();
        std::vector<std::vector<float>> w(static_cast<std::size_t>(E));
        for (int m = 0; m < E; ++m)
            w[static_cast<std::size_t>(m)].assign(W + m * per, W + (m + 1) * per);
        LinearModelBackend<D>::save(path, w, C);
        return RH_OK;
    });
}

int ref_blin1_load_evaluate(int domain, const char *path, double q, const void *packed,
                            std::int64_t n, std::int32_t *h_out) {
    return dispatch(domain, [&](auto *d) {
        using D = bare_t<decltype(d)>;
        LinearModelBackend<D> backend = LinearModelBackend<D>::load(path, q);
        const auto items = make_items<D>(packed, n);
        return run_backend_mt<D>(backend, items, h_out, 1);
    });
}

// quantile_class / ensemble_min (heuristic.hpp:107-126).
int ref_quantile_class(const double *p, int C, double q, int *out) {
    try {
        ClassDistribution dist;
        dist.p.assign(p, p + C);
        *out = quantile_class(dist, q);
        return RH_OK;
    } catch (const std::invalid_argument &e) {
        g_err = e.what();
        return RH_ERR_INVALID;
    }
}

int ref_ensemble_min(const int *v, int n, int *out) {
    try {
        *out = ensemble_min(std::span<const int>(v, static_cast<std::size_t>(n)));
        return RH_OK;
    } catch (const std::invalid_argument &e) {
        g_err = e.what();
        return RH_ERR_INVALID;
    }
}

// ManhattanHeuristic<N>::lookup (heuristic.hpp:76-89).
int ref_manhattan(int domain, const void *packed, std::int64_t n, std::int32_t *out) {
    return dispatch(domain, [&](auto *d) {
        using D = bare_t<decltype(d)>;
        if constexpr (std::is_same_v<D, RubiksCube>) {
            throw std::invalid_argument("manhattan is only defined for tile puzzles");
            return RH_ERR_ARG;
        } else {
            constexpr int N = [] {
                if constexpr (std::is_same_v<D, TilePuzzle<2>>) return 2;
                else if constexpr (std::is_same_v<D, TilePuzzle<3>>) return 3;
                else return 4;
            }();
            ManhattanHeuristic<N> mh;
            for (std::int64_t i = 0; i < n; ++i)
                out[i] = mh.lookup(unpack(d, static_cast<const char *>(packed) + i * 8));
            return RH_OK;
        }
    });
}

// load_instances<D> (instance.hpp:165-171): packs up to `cap` instance
// starts; returns the count through *count.
int ref_load_instances(int domain, const char *path, void *out_packed, std::int64_t cap,
                       std::int64_t *count) {
    return dispatch(domain, [&](auto *d) {
        using D = bare_t<decltype(d)>;
        const auto inst = load_instances<D>(path);
        std::int64_t k = 0;
        for (const auto &x : inst) {
            if (k >= cap)
                break;
            pack_state<D>(x.start, static_cast<char *>(out_packed) + k * packed_bytes<D>());
            ++k;
        }
        *count = static_cast<std::int64_t>(inst.size());
        return RH_OK;
    });
}

} // extern "C"

// ---- prepared batches for the timed CPU baseline ----
namespace {
struct PreparedBase {
    virtual ~PreparedBase() = default;
    virtual int run(std::int32_t *h, int threads) = 0;
};
template <class D>
struct Prepared final : PreparedBase {
    LinearModelBackend<D> backend;
    std::vector<BatchItem<D>> items;
    Prepared(std::vector<std::vector<float>> w, int C, double q) : backend(std::move(w), C, q) {}
    int run(std::int32_t *h, int threads) override {
        return run_backend_mt<D>(backend, items, h, threads);
    }
};
} // namespace

extern "C" void *ref_linear_prepare(int domain, const float *W, int E, int C, double q,
                                    const void *packed, std::int64_t n) {
    PreparedBase *out = nullptr;
    dispatch(domain, [&](auto *d) {
        using D = bare_t<decltype(d)>;
        const std::size_t per = static_cast<std::size_t>(C) * D::feature_length();
        std::vector<std::vector<float>> w(static_cast<std::size_t>(E));
        for (int m = 0; m < E; ++m)
            w[static_cast<std::size_t>(m)].assign(W + m * per, W + (m + 1) * per);
        auto *p = new Prepared<D>(std::move(w), C, q);
        p->items = make_items<D>(packed, n);
        out = p;
        return RH_OK;
    });
    return out;
}

extern "C" int ref_linear_run(void *prepared, std::int32_t *h_out, int threads) {
    try {
        return static_cast<PreparedBase *>(prepared)->run(h_out, threads);
    } catch (const std::exception &e) {
        g_err = e.what();
        return RH_ERR_INVALID;
    }
}

extern "C" void ref_linear_release(void *prepared) { delete static_cast<PreparedBase *>(prepared); }

// ---- pattern databases (pdb.hpp:30-69), built and looked up by the reference ----
extern "C" int ref_pdb_build(int domain, const std::uint8_t *pattern, int m, std::uint8_t *entries_out,
                             std::uint64_t cap, std::uint64_t *n_out) {
    return dispatch(domain, [&](auto *d) {
        using D = bare_t<decltype(d)>;
        std::vector<std::uint8_t> pat(pattern, pattern + m);
        const PdbTable<D> t = PdbTable<D>::build(pat, D::solved());
        *n_out = t.size();
        if (t.size() > cap)
            throw std::invalid_argument("PDB larger than the output buffer");
        std::memcpy(entries_out, t.entries().data(), t.size());
        return RH_OK;
    });
}

extern "C" int ref_pdb_lookup_file(int domain, const char *path, const void *packed, std::int64_t n,
                                   std::int32_t *out) {
    return dispatch(domain, [&](auto *d) {
        using D = bare_t<decltype(d)>;
        const PdbTable<D> t = PdbTable<D>::load(path);
        for (std::int64_t i = 0; i < n; ++i)
            out[i] = t.lookup(unpack(d, static_cast<const char *>(packed) + i * packed_bytes<D>()));
        return RH_OK;
    });
}

extern "C" int ref_pdb_build_save(int domain, const std::uint8_t *pattern, int m, const char *path) {
    return dispatch(domain, [&](auto *d) {
        using D = bare_t<decltype(d)>;
        std::vector<std::uint8_t> pat(pattern, pattern + m);
        PdbTable<D>::build(pat, D::solved()).save(path);
        return RH_OK;
    });
}
