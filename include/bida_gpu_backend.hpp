// bida_gpu_backend.hpp — C++ drop-in for the reference's evaluator backend.
//
//   bida::EvaluatorBackend<D>  (/root/reference/proj/include/bida/batch_eval.hpp:45-51)
//     virtual void evaluate(std::span<const BatchItem<D>>, std::span<std::int32_t>) = 0;
//     virtual bool needs_features() const;
//
// GpuBackend<D> implements it over the C-ABI in bida_gpu.h, so the
// reference's Evaluator / EvaluatorGroup / batch_idastar / aidastar use the
// B200 evaluator unchanged:
//
//   std::vector<std::unique_ptr<bida::EvaluatorBackend<D>>> backends;
//   for (int g = 0; g < n_gpus; ++g)
//       backends.push_back(bida_gpu::GpuBackend<D>::load_linear(g, "w.blin", 0.5));
//   bida::EvaluatorGroup<D> group(std::move(backends), batch, timeout_us);
//
// Contract: needs_features() is false — states are packed
// with the reference's own D::pack and one-hot encoded on the device; every
// out[i] is written; evaluate() never throws (an exception on the agent thread
// would std::terminate), errors are counted and the last message kept.
// Construction errors throw std::invalid_argument / std::runtime_error like
// LinearModelBackend's constructor and load() (batch_eval.hpp:87-93, 111-129).
// Calls may come concurrently from the agent thread and evaluate_single /
// evaluate_sync callers; the C-ABI handle is re-entrant.
#pragma once

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "bida/batch_eval.hpp"
#include "bida/rubiks.hpp"
#include "bida/stp.hpp"
#include "bida_gpu.h"

namespace bida_gpu {

// Packing the agent does for every state of every batch (the wire format is
// exactly D::pack's).  With BMI2 (checked at run time) each byte-array field is
// gathered by one PEXT instead of a shift-or per element; a state with a byte
// outside its field's range (never produced by the search) takes D::pack, whose
// OR of overlapping fields the masked gather would not reproduce.
namespace pack_detail {
inline bool has_bmi2() {
#if defined(__x86_64__)
    static const bool yes = __builtin_cpu_supports("bmi2");
    return yes;
#else
    return false;
#endif
}
inline std::uint64_t rd64(const std::uint8_t *p) {
    std::uint64_t v;
    std::memcpy(&v, p, 8);
    return v;
}
inline std::uint32_t rd32(const std::uint8_t *p) {
    std::uint32_t v;
    std::memcpy(&v, p, 4);
    return v;
}
#if defined(__x86_64__)
__attribute__((target("bmi2"))) inline std::uint64_t pext(std::uint64_t v, std::uint64_t m) {
    return __builtin_ia32_pext_di(v, m);
}
#endif
}  // namespace pack_detail

template <class D>
struct DomainOf;
template <int N>
struct DomainOf<bida::TilePuzzle<N>> {
    static constexpr int id = N;  // BIDA_DOMAIN_STP2..4
    static constexpr int packed_bytes = 8;
    static void pack(const typename bida::TilePuzzle<N>::State &s, unsigned char *out) {
#if defined(__x86_64__)
        if constexpr (N == 4) {
            if (pack_detail::has_bmi2()) {
                const std::uint64_t a = pack_detail::rd64(s.tiles.data()), b = pack_detail::rd64(s.tiles.data() + 8);
                if (((a | b) & 0xF0F0F0F0F0F0F0F0ull) == 0) {
                    const std::uint64_t v = pack_detail::pext(a, 0x0F0F0F0F0F0F0F0Full) |
                                            pack_detail::pext(b, 0x0F0F0F0F0F0F0F0Full) << 32;
                    std::memcpy(out, &v, 8);
                    return;
                }
            }
        }
#endif
        const std::uint64_t v = bida::TilePuzzle<N>::pack(s);  // stp.hpp:121-126
        std::memcpy(out, &v, 8);
    }
};
template <>
struct DomainOf<bida::RubiksCube> {
    static constexpr int id = BIDA_DOMAIN_RC;
    static constexpr int packed_bytes = 16;
    static void pack(const bida::RubiksCube::State &s, unsigned char *out) {
#if defined(__x86_64__)
        if (pack_detail::has_bmi2()) {
            using namespace pack_detail;
            const std::uint64_t cp = rd64(s.cp.data()), co = rd64(s.co.data());
            const std::uint64_t ep0 = rd64(s.ep.data()), eo0 = rd64(s.eo.data());
            const std::uint32_t ep1 = rd32(s.ep.data() + 8), eo1 = rd32(s.eo.data() + 8);
            const bool in_range = (cp & 0xF8F8F8F8F8F8F8F8ull) == 0 && (co & 0xFCFCFCFCFCFCFCFCull) == 0 &&
                                  (eo0 & 0xFEFEFEFEFEFEFEFEull) == 0 && (eo1 & 0xFEFEFEFEu) == 0 &&
                                  (ep0 & 0xF0F0F0F0F0F0F0F0ull) == 0 && (ep1 & 0xF0F0F0F0u) == 0;
            if (in_range) {
                const std::uint64_t lo = pext(cp, 0x0707070707070707ull) | pext(co, 0x0303030303030303ull) << 24 |
                                         pext(eo0, 0x0101010101010101ull) << 40 | pext(eo1, 0x01010101ull) << 48;
                const std::uint64_t hi = pext(ep0, 0x0F0F0F0F0F0F0F0Full) | pext(ep1, 0x0F0F0F0Full) << 32;
                std::memcpy(out, &lo, 8);
                std::memcpy(out + 8, &hi, 8);
                return;
            }
        }
#endif
        const bida::RubiksCube::Packed p = bida::RubiksCube::pack(s);  // rubiks.hpp:126-137
        std::memcpy(out, &p.lo, 8);
        std::memcpy(out + 8, &p.hi, 8);
    }
};

inline void throw_status(int rc, const char *what) {
    const std::string msg = std::string(what) + ": " + bida_gpu_last_error();
    if (rc == BIDA_ERR_INVALID_ARGUMENT)
        throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

template <class D>
class GpuBackend final : public bida::EvaluatorBackend<D>
#ifdef BIDA_RING_EVALUATOR
    , public bida::ConcurrentBackend  // the C-ABI handle is re-entrant (8 zero-copy lanes)
    , public bida::AsyncEvaluatorBackend<D>  // bida_gpu_submit / bida_gpu_batch_wait
    , public bida::GatherEvaluatorBackend<D>  // ring ranges packed in place into a lane
    , public bida::PackedGatherBackend<D>     // submitters pre-pack; packed runs copied into a lane
#endif
{
public:
    using Traits = DomainOf<D>;

    // LinearModelBackend(member_weights, classes, quantile) on `device`.
    GpuBackend(int device, const std::vector<std::vector<float>> &member_weights, int classes,
               double quantile) {
        if (member_weights.empty())
            throw std::invalid_argument("LinearModelBackend: empty ensemble");
        const std::size_t per = static_cast<std::size_t>(classes) * D::feature_length();
        std::vector<float> flat;
        for (const auto &w : member_weights) {
            if (w.size() != per)
                throw std::invalid_argument("LinearModelBackend: weight matrix size mismatch");
            flat.insert(flat.end(), w.begin(), w.end());
        }
        bida_gpu_evaluator *h = nullptr;
        const int rc = bida_gpu_linear_create(device, Traits::id, flat.data(),
                                              static_cast<int>(member_weights.size()), classes, quantile, &h);
        if (rc)
            throw_status(rc, "GpuBackend");
        handle_ = h;
    }

    // LinearModelBackend::load(path, quantile) (BLIN1) on `device`.
    static std::unique_ptr<GpuBackend> load_linear(int device, const std::string &path, double quantile) {
        bida_gpu_evaluator *h = nullptr;
        const int rc = bida_gpu_linear_load(device, Traits::id, path.c_str(), quantile, &h);
        if (rc)
            throw_status(rc, "GpuBackend::load_linear");
        return std::unique_ptr<GpuBackend>(new GpuBackend(h));
    }

    // BMLP1 integer MLP ensemble on `device`.
    static std::unique_ptr<GpuBackend> load_mlp(int device, const std::string &path, double quantile) {
        bida_gpu_evaluator *h = nullptr;
        const int rc = bida_gpu_mlp_load(device, Traits::id, path.c_str(), quantile, &h);
        if (rc)
            throw_status(rc, "GpuBackend::load_mlp");
        return std::unique_ptr<GpuBackend>(new GpuBackend(h));
    }

    // PDB correction in the device readout (bida_gpu_attach_pdb_file):
    // BIDA_PDB_MIN -> min(h_model, h_PDB); BIDA_PDB_REPLACE -> h_PDB with the
    // model still evaluated (PAPER.md:407 Table-1 mode).  BPDB1 file from
    // PdbTable::save (pdb.hpp:78-96).
    void attach_pdb_file(const std::string &path, int mode) {
        if (const int rc = bida_gpu_attach_pdb_file(handle_, path.c_str(), mode))
            throw_status(rc, "GpuBackend::attach_pdb_file");
    }

    ~GpuBackend() override {
#ifdef BIDA_RING_EVALUATOR
        if (bida::ring_detail::profile_on() && calls_.load() > 0)
            std::fprintf(stderr, "{\"gpu_backend_profile\": {\"calls\": %llu, \"items\": %llu, \"pack_s\": %.3f, "
                                 "\"launch_wait_s\": %.3f}}\n",
                         (unsigned long long)calls_.load(), (unsigned long long)items_.load(),
                         prof_pack_ns_.load() * 1e-9, prof_gpu_ns_.load() * 1e-9);
#endif
        if (handle_)
            bida_gpu_destroy(handle_);
    }
    GpuBackend(const GpuBackend &) = delete;
    GpuBackend &operator=(const GpuBackend &) = delete;

    bool needs_features() const override { return false; }
#ifdef BIDA_RING_EVALUATOR
    int max_concurrent_calls() const override { return 8; }  // one per zero-copy lane
    // Asynchronous path (ring agents keep several batches in flight each):
    // the packed batch is copied into a zero-copy lane at submit; the GPU writes
    // h into mapped host memory; complete() waits, copies and releases the lane.
    int max_in_flight() const override { return 8; }  // zero-copy lanes per handle (bida_gpu.cu)
    void *submit(std::span<const bida::BatchItem<D>> batch) override {
        if (batch.size() > 32768)
            return nullptr;  // larger than a lane: the caller uses evaluate()
        thread_local std::vector<unsigned char> staging;
        const std::size_t n = batch.size();
        staging.resize(n * Traits::packed_bytes);
        for (std::size_t i = 0; i < n; ++i)
            Traits::pack(batch[i].state, staging.data() + i * Traits::packed_bytes);
        bida_gpu_batch *b = nullptr;
        const int rc = bida_gpu_submit(handle_, staging.data(), static_cast<std::int64_t>(n), &b);
        if (rc) {
            note_error();
            return nullptr;  // fall back to the synchronous path, which zero-fills on error
        }
        calls_.fetch_add(1, std::memory_order_relaxed);
        items_.fetch_add(n, std::memory_order_relaxed);
        return b;
    }
    std::size_t packed_bytes() const override { return Traits::packed_bytes; }
    void pack_state(const D::State &st, unsigned char *dst) const override { Traits::pack(st, dst); }
    void pack_states(const D::State *st, std::size_t n, unsigned char *dst) const override {
        for (std::size_t i = 0; i < n; ++i)
            Traits::pack(st[i], dst + i * Traits::packed_bytes);
    }
    // The ring agent's claimed runs of pre-packed states, copied into one zero-copy lane.
    void evaluate_packed(std::span<const std::span<const unsigned char>> parts, std::size_t n,
                         std::span<std::int32_t> out) override {
        const bool prof = bida::ring_detail::profile_on();
        const std::int64_t t0 = prof ? bida::ring_detail::now_ns() : 0;
        bida_gpu_batch *b = nullptr;
        void *in = nullptr;
        int rc = BIDA_ERR_INVALID_ARGUMENT;
        if (n > 0 && n <= 32768 && bida_gpu_batch_begin(handle_, static_cast<std::int64_t>(n), &b, &in) == BIDA_OK) {
            auto *dst = static_cast<unsigned char *>(in);
            for (const auto &part : parts) {
                std::memcpy(dst, part.data(), part.size());
                dst += part.size();
            }
            const std::int64_t t1 = prof ? bida::ring_detail::now_ns() : 0;
            rc = bida_gpu_batch_launch(b);
            if (rc == BIDA_OK)
                rc = bida_gpu_batch_wait(b, out.data());  // zero-fills out on error
            if (prof) {
                prof_pack_ns_.fetch_add(t1 - t0, std::memory_order_relaxed);
                prof_gpu_ns_.fetch_add(bida::ring_detail::now_ns() - t1, std::memory_order_relaxed);
            }
        } else if (n > 0) {  // larger than a lane: one contiguous staging copy
            thread_local std::vector<unsigned char> staging;
            staging.clear();
            for (const auto &part : parts)
                staging.insert(staging.end(), part.begin(), part.end());
            rc = bida_gpu_evaluate(handle_, staging.data(), static_cast<std::int64_t>(n), out.data());
        } else {
            return;
        }
        calls_.fetch_add(1, std::memory_order_relaxed);
        items_.fetch_add(n, std::memory_order_relaxed);
        if (rc) {
            for (auto &v : out)
                v = 0;
            note_error();
        }
    }
    // The ring agent's claimed ranges, packed in place into one zero-copy lane.
    void evaluate_parts(std::span<const std::span<const bida::BatchItem<D>>> parts, std::size_t n,
                        std::span<std::int32_t> out) override {
        if (n > 0 && n <= 32768) {
            bida_gpu_batch *b = nullptr;
            void *in = nullptr;
            const bool prof = bida::ring_detail::profile_on();
            const std::int64_t t0 = prof ? bida::ring_detail::now_ns() : 0;
            if (bida_gpu_batch_begin(handle_, static_cast<std::int64_t>(n), &b, &in) == BIDA_OK) {
                auto *dst = static_cast<unsigned char *>(in);
                for (const auto &part : parts)
                    for (const auto &it : part) {
                        Traits::pack(it.state, dst);
                        dst += Traits::packed_bytes;
                    }
                const std::int64_t t1 = prof ? bida::ring_detail::now_ns() : 0;
                int rc = bida_gpu_batch_launch(b);
                if (rc == BIDA_OK)
                    rc = bida_gpu_batch_wait(b, out.data());  // zero-fills out on error
                if (prof) {
                    prof_pack_ns_.fetch_add(t1 - t0, std::memory_order_relaxed);
                    prof_gpu_ns_.fetch_add(bida::ring_detail::now_ns() - t1, std::memory_order_relaxed);
                }
                calls_.fetch_add(1, std::memory_order_relaxed);
                items_.fetch_add(n, std::memory_order_relaxed);
                if (rc) {
                    for (auto &v : out)
                        v = 0;
                    note_error();
                }
                return;
            }
        }
        std::vector<bida::BatchItem<D>> flat;  // larger than a lane: one contiguous batch
        flat.reserve(n);
        for (const auto &part : parts)
            for (const auto &it : part)
                flat.push_back(bida::BatchItem<D>{nullptr, it.state, {}});
        evaluate(flat, out);
    }
    bool ready(void *token) override { return bida_gpu_batch_ready(static_cast<bida_gpu_batch *>(token)) != 0; }
    void complete(void *token, std::span<std::int32_t> out) override {
        if (bida_gpu_batch_wait(static_cast<bida_gpu_batch *>(token), out.data()) != BIDA_OK)
            note_error();  // out[] zero-filled: frames never block forever
    }
#endif

    void evaluate(std::span<const bida::BatchItem<D>> batch, std::span<std::int32_t> out) override {
        const std::size_t n = batch.size();
        if (n > 0 && n <= 32768) {
            // pack straight into a zero-copy lane's mapped input (no staging copy)
            bida_gpu_batch *b = nullptr;
            void *in = nullptr;
            if (bida_gpu_batch_begin(handle_, static_cast<std::int64_t>(n), &b, &in) == BIDA_OK) {
                auto *dst = static_cast<unsigned char *>(in);
                for (std::size_t i = 0; i < n; ++i)
                    Traits::pack(batch[i].state, dst + i * Traits::packed_bytes);
                int rc = bida_gpu_batch_launch(b);
                if (rc == BIDA_OK)
                    rc = bida_gpu_batch_wait(b, out.data());  // zero-fills out on error
                calls_.fetch_add(1, std::memory_order_relaxed);
                items_.fetch_add(n, std::memory_order_relaxed);
                if (rc) {
                    for (auto &v : out)
                        v = 0;
                    note_error();
                }
                return;
            }
        }
        thread_local std::vector<unsigned char> staging;
        staging.resize(n * Traits::packed_bytes);
        for (std::size_t i = 0; i < n; ++i)
            Traits::pack(batch[i].state, staging.data() + i * Traits::packed_bytes);
        const int rc = bida_gpu_evaluate(handle_, staging.data(), static_cast<std::int64_t>(n), out.data());
        calls_.fetch_add(1, std::memory_order_relaxed);
        items_.fetch_add(n, std::memory_order_relaxed);
        if (rc) {
            for (auto &v : out)
                v = 0;  // h >= 0 keeps frames from blocking forever (cbdfs.hpp:262-265)
            note_error();
        }
    }

    std::uint64_t errors() const { return errors_.load(std::memory_order_relaxed); }
    std::uint64_t calls() const { return calls_.load(std::memory_order_relaxed); }
    std::uint64_t items() const { return items_.load(std::memory_order_relaxed); }
    std::string last_error() const {
        std::lock_guard<std::mutex> lk(err_m_);
        return last_error_;
    }
    bida_gpu_evaluator *handle() const { return handle_; }

private:
    explicit GpuBackend(bida_gpu_evaluator *h) : handle_(h) {}

    void note_error() {
        errors_.fetch_add(1, std::memory_order_relaxed);
        std::lock_guard<std::mutex> lk(err_m_);
        last_error_ = bida_gpu_last_error();
    }

    bida_gpu_evaluator *handle_ = nullptr;
    std::atomic<std::uint64_t> errors_{0}, calls_{0}, items_{0};
    std::atomic<std::int64_t> prof_pack_ns_{0}, prof_gpu_ns_{0};  // BIDA_RING_PROFILE (ring builds)
    mutable std::mutex err_m_;
    std::string last_error_;
};

} // namespace bida_gpu
