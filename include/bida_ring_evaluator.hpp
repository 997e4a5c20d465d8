// bida_ring_evaluator.hpp — replacement of the reference's Evaluator internals
// behind the unchanged public API.
//
//   reference: bida::Evaluator<D>       /root/reference/proj/include/bida/batch_eval.hpp:193-381
//              bida::EvaluatorGroup<D>  batch_eval.hpp:385-473
//              make_table_sim_group     batch_eval.hpp:475-484
//
// The reference buffers submissions in a mutex-guarded std::vector<BatchItem>
// and runs ONE agent thread per evaluator that takes a batch, calls the
// backend synchronously and resolves the tickets before it looks at the
// buffer again.  With a B200 behind the backend that round trip (copy in,
// launch, copy out) is idle host time and caps one evaluator at ~1.9 M
// nodes/s (profiles/r1_search_rc_gpu.jsonl).  Here:
//
//   * submissions go into bounded multi-producer rings, S shards per
//     evaluator (default 8, env BIDA_EVAL_SHARDS; searcher thread i uses
//     shard i mod S): one fetch_add on the shard tail, a per-slot sequence
//     word publishes the item; no mutex, no vector growth, no notify per
//     submit, no counter shared by every searcher;
//   * K agents per evaluator (default 2, env BIDA_EVAL_AGENTS) claim
//     contiguous published ranges under a short claim lock and run backend
//     calls concurrently, so batch i+1 is staged and launched while batch i
//     is on the device (GpuBackend's C-ABI handle is re-entrant);
//   * tickets are resolved in bulk straight from the ring slots.
//
// Unchanged: Ticket / TicketSlot / poll (write-once, -1 pending), the flush
// policy (full batch, forced drain via request_flush/kick_all, close, timeout
// 0 = flush when nonempty, timeout > 0 = flush once the oldest pending item
// is timeout_us old, timeout < 0 = full or forced only), at most `capacity`
// items per backend call, evaluate_single / evaluate_sync on the caller
// thread, immediate mode, stats (one record_batch per backend batch,
// forced_flushes, sync_evaluations), submission after close throws
// std::runtime_error.  Timeout clock: the oldest pending item's age counts
// from its submission when it was its shard's head then, else from when an
// agent first saw it as the head -- as the reference restarts its clock at
// "now" after taking a full batch from a longer queue.
//
// Used by building the reference's search against include/overlay/ (see
// tools/Makefile: bida_search_ring), where bida/batch_eval.hpp is the
// reference header with these three names swapped for the ones below.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <chrono>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <deque>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <thread>
#include <vector>

#if __has_include(<nvtx3/nvToolsExt.h>)
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3 (SURVEY §5 tracing)
#define BIDA_NVTX_PUSH(name) nvtxRangePushA(name)
#define BIDA_NVTX_POP() nvtxRangePop()
#else
#define BIDA_NVTX_PUSH(name) ((void)0)
#define BIDA_NVTX_POP() ((void)0)
#endif

namespace bida {

// Opt-in marker for backends whose evaluate() may run on several agent threads
// at once (the reference's EvaluatorBackend interface is unchanged).
struct ConcurrentBackend {
    virtual ~ConcurrentBackend() = default;
    virtual int max_concurrent_calls() const = 0;
};

// Opt-in asynchronous evaluation (bida_gpu::GpuBackend: bida_gpu_submit /
// bida_gpu_batch_wait): an agent keeps up to depth batches in flight instead
// of blocking on each device round trip.
template <class D>
struct AsyncEvaluatorBackend {
    virtual ~AsyncEvaluatorBackend() = default;
    // Starts evaluating `batch` (read before returning); nullptr: not accepted,
    // the caller uses evaluate() instead.
    virtual void *submit(std::span<const BatchItem<D>> batch) = 0;
    virtual bool ready(void *token) = 0;                                  // non-blocking
    virtual void complete(void *token, std::span<std::int32_t> out) = 0;  // waits; writes every out[i]
    virtual int max_in_flight() const = 0;                                // over all callers
};

// Opt-in gather evaluation (bida_gpu::GpuBackend): the batch given as the
// agent's claimed ring ranges in place (one span per contiguous run, in
// order), so a batch spanning several shards is never moved into a scratch
// vector first.  Writes every out[i] (n = total items).
template <class D>
struct GatherEvaluatorBackend {
    virtual ~GatherEvaluatorBackend() = default;
    virtual void evaluate_parts(std::span<const std::span<const BatchItem<D>>> parts, std::size_t n,
                                std::span<std::int32_t> out) = 0;
};

// Opt-in pre-packing (bida_gpu::GpuBackend): submitters pack each state into
// the ring slot's packed bytes while the state is hot in their cache, and the
// agent hands the backend the claimed runs of packed bytes (one span per
// contiguous run).  With the gather path alone the agent packs, reading every
// state from a line another core just wrote (BIDA_RING_PROFILE measured
// ~11 ns per state there).  Writes every out[i].
template <class D>
struct PackedGatherBackend {
    virtual ~PackedGatherBackend() = default;
    virtual std::size_t packed_bytes() const = 0;
    virtual void pack_state(const typename D::State &state, unsigned char *dst) const = 0;
    // n consecutive states into n consecutive packed slots (one call per reservation run)
    virtual void pack_states(const typename D::State *states, std::size_t n, unsigned char *dst) const {
        for (std::size_t i = 0; i < n; ++i)
            pack_state(states[i], dst + i * packed_bytes());
    }
    virtual void evaluate_packed(std::span<const std::span<const unsigned char>> parts, std::size_t n,
                                 std::span<std::int32_t> out) = 0;
};

namespace ring_detail {
inline std::int64_t now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}
// BIDA_RING_PROFILE=1: agents time their phases; totals go to stderr at close()
inline bool profile_on() {
    static const bool on = [] {
        const char *s = std::getenv("BIDA_RING_PROFILE");
        return s && s[0] == '1';
    }();
    return on;
}
inline bool env_noprepack() {  // BIDA_EVAL_PREPACK=0: the agent packs (gather path)
    const char *s = std::getenv("BIDA_EVAL_PREPACK");
    return s && s[0] == '0';
}
inline int default_agents() {
    const char *s = std::getenv("BIDA_EVAL_AGENTS");
    const int k = s ? std::atoi(s) : 2;
    return std::clamp(k, 1, 16);
}
// K concurrent agents only for backends that declare concurrent evaluate()
// calls safe and useful (ConcurrentBackend, e.g. bida_gpu::GpuBackend); any
// other backend (TableSimBackend, LinearModelBackend) keeps the reference's
// one agent per evaluator, i.e. one simulated device per evaluator.
template <class B>
int agents_for(const B *backend, int requested) {
    const auto *c = dynamic_cast<const ConcurrentBackend *>(backend);
    return c ? std::clamp(requested, 1, std::max(1, c->max_concurrent_calls())) : 1;
}
inline int default_shards() {
    const char *s = std::getenv("BIDA_EVAL_SHARDS");
    const int k = s ? std::atoi(s) : 8;
    return std::clamp(k, 1, 64);
}
inline int env_inflight() {  // BIDA_EVAL_INFLIGHT: batches in flight per agent (default 1: synchronous)
    const char *s = std::getenv("BIDA_EVAL_INFLIGHT");
    return s ? std::clamp(std::atoi(s), 0, 64) : 0;
}
// a small per-thread index, so a searcher thread keeps submitting to one shard
inline std::size_t thread_slot() {
    static std::atomic<std::size_t> next{0};
    thread_local const std::size_t mine = next.fetch_add(1, std::memory_order_relaxed);
    return mine;
}
inline void relax(unsigned &spins) {
    if (++spins < 64) {
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    } else {
        std::this_thread::yield();
    }
}
} // namespace ring_detail

template <class D>
class Evaluator {
public:
    Evaluator(std::unique_ptr<EvaluatorBackend<D>> backend, std::size_t capacity, std::int64_t timeout_us,
              bool immediate = false, int agents = ring_detail::default_agents(),
              int shards = ring_detail::default_shards())
        : backend_(std::move(backend)), capacity_(capacity), timeout_us_(timeout_us), immediate_(immediate) {
        if (capacity_ == 0)
            throw std::invalid_argument("Evaluator: capacity must be >= 1");
        nshards_ = static_cast<std::size_t>(shards);
        // every shard holds at least one full batch, so a producer blocked on
        // a full shard always leaves a flushable batch behind it (timeout < 0)
        std::size_t r = 4096;
        while (r < capacity_ || r * nshards_ < 8 * capacity_)
            r <<= 1;
        ring_size_ = r;
        mask_ = r - 1;
        shards_ = std::make_unique<Shard[]>(nshards_);
        for (std::size_t k = 0; k < nshards_; ++k) {
            Shard &sh = shards_[k];
            sh.items = std::make_unique<BatchItem<D>[]>(r);
            sh.meta = std::make_unique<Meta[]>(r);
            sh.t_ns = std::make_unique<std::int64_t[]>(r);  // value-initialised: 0
            for (std::size_t i = 0; i < r; ++i)
                sh.meta[i].seq.store(i, std::memory_order_relaxed);
        }
        // a producer wakes the agents when its shard goes nonempty or crosses
        // a multiple of capacity / shards (the agents then check the total)
        wake_step_ = std::max<std::uint64_t>(1, capacity_ / nshards_);
        feats_ = backend_->needs_features();
        if (!immediate_) {
            const int k_agents = ring_detail::agents_for(backend_.get(), agents);
            // in-flight batches per agent: the backend's lanes shared by the
            // agents (so an agent blocked in submit() never waits on lanes only
            // blocked agents hold); 1 = synchronous evaluate()
            // Opt-in (BIDA_EVAL_INFLIGHT=d > 1): measured on one B200 the search is
            // bound by the agents' per-item host work, not by round trips in
            // flight (profiles/r2_search_async_sweep.jsonl), so the default stays
            // one synchronous call per agent.
            gather_ = dynamic_cast<GatherEvaluatorBackend<D> *>(backend_.get());
            packer_ = dynamic_cast<PackedGatherBackend<D> *>(backend_.get());
            async_ = dynamic_cast<AsyncEvaluatorBackend<D> *>(backend_.get());
            if (async_) {
                const int env = ring_detail::env_inflight();
                depth_ = std::min(env, std::max(1, async_->max_in_flight() / k_agents));
                if (depth_ <= 1) {
                    async_ = nullptr;
                    depth_ = 1;
                }
            }
            if (packer_ && (async_ || !gather_ || backend_->needs_features() || ring_detail::env_noprepack()))
                packer_ = nullptr;
            if (packer_) {
                pb_ = packer_->packed_bytes();
                for (std::size_t k = 0; k < nshards_; ++k)
                    shards_[k].packed = std::make_unique<unsigned char[]>(ring_size_ * pb_);
            }
            for (int k = 0; k < k_agents; ++k)
                agents_.emplace_back([this] { agent_loop(); });
        }
    }

    ~Evaluator() { close(); }

    Evaluator(const Evaluator &) = delete;
    Evaluator &operator=(const Evaluator &) = delete;

    Ticket submit(const typename D::State &state, FeatureVector features) {
        Ticket t = std::make_shared<TicketSlot>();
        if (immediate_) {
            BatchItem<D> item{t, state, std::move(features)};
            std::int32_t v = 0;
            backend_->evaluate(std::span<const BatchItem<D>>(&item, 1), std::span<std::int32_t>(&v, 1));
            resolve(*t, v);
            immediate_submitted_.fetch_add(1, std::memory_order_relaxed);
            return t;
        }
        enqueue(state, std::move(features), t, nullptr);
        return t;
    }

    // Extension for the CB-DFS overlay (include/overlay/bida/cbdfs.hpp): the
    // caller owns `slot` (value -1, address stable until it is resolved), so
    // no per-node shared_ptr is allocated.  Same batching as submit().
    void submit_slot(const typename D::State &state, FeatureVector features, TicketSlot *slot) {
        if (immediate_) {
            BatchItem<D> item{Ticket(), state, std::move(features)};
            std::int32_t v = 0;
            backend_->evaluate(std::span<const BatchItem<D>>(&item, 1), std::span<std::int32_t>(&v, 1));
            resolve(*slot, v);
            immediate_submitted_.fetch_add(1, std::memory_order_relaxed);
            return;
        }
        enqueue(state, std::move(features), Ticket(), slot);
    }

    // The children of one expansion in one reservation: one tail bump and one
    // in-flight/close handshake for all n (the per-item locked instructions
    // are a measurable share of a searcher's time per node).  Backends that
    // need features, and immediate evaluators, take the one-by-one path.
    void submit_slots(const typename D::State *states, TicketSlot *const *slots, std::size_t n) {
        if (n == 0)
            return;
        if (immediate_ || backend_->needs_features()) {
            for (std::size_t i = 0; i < n; ++i) {
                FeatureVector x;
                if (backend_->needs_features()) {
                    x.resize(static_cast<std::size_t>(D::feature_length()));
                    D::encode(states[i], x.data());
                }
                submit_slot(states[i], std::move(x), slots[i]);
            }
            return;
        }
        enqueue_n(states, slots, n);
    }

    bool needs_features() const { return backend_->needs_features(); }

    // Synchronous batch of one on the caller's thread (root nodes).
    int evaluate_single(const typename D::State &state, FeatureVector features) {
        BatchItem<D> item{std::make_shared<TicketSlot>(), state, std::move(features)};
        std::int32_t v = 0;
        backend_->evaluate(std::span<const BatchItem<D>>(&item, 1), std::span<std::int32_t>(&v, 1));
        std::lock_guard<std::mutex> lk(stats_m_);
        stats_.record_batch(1);
        return static_cast<int>(v);
    }

    // One synchronous backend call of any size; a sync evaluation, not a batch.
    std::vector<int> evaluate_sync(std::span<const typename D::State> states) {
        std::vector<BatchItem<D>> items(states.size());
        const bool feats = backend_->needs_features();
        for (std::size_t i = 0; i < states.size(); ++i) {
            items[i].state = states[i];
            if (feats) {
                items[i].features.resize(static_cast<std::size_t>(D::feature_length()));
                D::encode(states[i], items[i].features.data());
            }
        }
        std::vector<std::int32_t> vals(states.size());
        if (!states.empty())
            backend_->evaluate(items, vals);
        std::lock_guard<std::mutex> lk(stats_m_);
        ++stats_.sync_evaluations;
        return std::vector<int>(vals.begin(), vals.end());
    }

    // Flush the pending items even though no batch is full.
    void request_flush() {
        if (!pending())
            return;
        if (!force_.exchange(true, std::memory_order_acq_rel))
            wake();
    }

    // Drains everything submitted (resolving it) and joins the agents.
    void close() {
        if (closed_.exchange(true, std::memory_order_seq_cst))
            return;
        struct Report {  // after the agents joined (end of close)
            Evaluator *ev;
            ~Report() {
                if (ring_detail::profile_on() && ev->prof_batches_.load() > 0)
                    std::fprintf(stderr,
                                 "{\"ring_profile\": {\"agents\": %zu, \"batches\": %llu, \"items\": %llu, "
                                 "\"claim_s\": %.3f, \"evaluate_s\": %.3f, \"finish_s\": %.3f}}\n",
                                 ev->agents_.size(), (unsigned long long)ev->prof_batches_.load(),
                                 (unsigned long long)ev->prof_items_.load(), ev->prof_claim_ns_.load() * 1e-9,
                                 ev->prof_eval_ns_.load() * 1e-9, ev->prof_finish_ns_.load() * 1e-9);
            }
        } report{this};
        for (std::size_t k = 0; k < nshards_; ++k) {
            unsigned spins = 0;
            while (shards_[k].inflight.load(std::memory_order_seq_cst) != 0)
                ring_detail::relax(spins);
        }
        // every accepted submit is now published: agents may exit once drained
        quiesced_.store(true, std::memory_order_seq_cst);
        wake();
        for (auto &a : agents_)
            if (a.joinable())
                a.join();
    }

    SearchStats stats_snapshot() const {
        std::lock_guard<std::mutex> lk(stats_m_);
        return stats_;
    }

    std::uint64_t submitted() const {
        std::uint64_t n = immediate_submitted_.load(std::memory_order_relaxed);
        for (std::size_t k = 0; k < nshards_; ++k)
            n += shards_[k].tail.load(std::memory_order_relaxed);
        return n;
    }
    std::uint64_t resolved() const { return resolved_.load(std::memory_order_relaxed); }
    std::uint64_t double_resolutions() const { return double_resolved_.load(std::memory_order_relaxed); }
    std::size_t agent_count() const { return agents_.size(); }
    int in_flight_per_agent() const { return async_ ? depth_ : 1; }
    std::size_t shard_count() const { return nshards_; }

private:
    struct Meta {
        std::atomic<std::uint64_t> seq{0}; // == pos: free for lap pos; == pos+1: published
        TicketSlot *raw = nullptr;         // submit_slot(): resolve here instead of the item's ticket
    };
    struct Shard {
        alignas(64) std::atomic<std::uint64_t> tail{0}; // next position producers claim
        std::atomic<std::uint32_t> inflight{0};         // submits between the closed check and publish
        alignas(64) std::atomic<std::uint64_t> head{0}; // next position agents claim
        std::unique_ptr<BatchItem<D>[]> items;
        std::unique_ptr<Meta[]> meta;
        // timeout > 0: time the item became its shard's head (0: not yet); kept
        // out of Meta (16 B) since only range heads are ever stamped
        std::unique_ptr<std::int64_t[]> t_ns;
        std::unique_ptr<unsigned char[]> packed;  // pre-packing backends: pb_ bytes per slot
    };
    struct Range {
        std::size_t shard;
        std::uint64_t h;
        std::size_t n;
    };

    // enqueue() for n caller-owned slots at consecutive positions of the
    // thread's shard; items are published in order (agents claim published
    // prefixes), the last with the seq_cst store the wake check pairs with.
    void enqueue_n(const typename D::State *states, TicketSlot *const *raws, std::size_t n) {
        Shard &sh = shards_[ring_detail::thread_slot() % nshards_];
        sh.inflight.fetch_add(1, std::memory_order_seq_cst);
        if (closed_.load(std::memory_order_seq_cst)) {
            sh.inflight.fetch_sub(1, std::memory_order_release);
            throw std::runtime_error("Evaluator: submission after shutdown");
        }
        const std::uint64_t pos0 = sh.tail.fetch_add(n, std::memory_order_acq_rel);
        if (packer_) {
            // every slot of the reservation free (its previous lap consumed), then
            // one pack call per contiguous run (two if the reservation wraps)
            for (std::size_t i = 0; i < n; ++i) {
                unsigned spins = 0;
                while (sh.meta[(pos0 + i) & mask_].seq.load(std::memory_order_acquire) != pos0 + i)
                    ring_detail::relax(spins);
            }
            const std::size_t at = pos0 & mask_, first = std::min(n, ring_size_ - at);
            packer_->pack_states(states, first, &sh.packed[at * pb_]);
            if (first < n)
                packer_->pack_states(states + first, n - first, &sh.packed[0]);
        }
        for (std::size_t i = 0; i < n; ++i) {
            const std::uint64_t pos = pos0 + i;
            Meta &m = sh.meta[pos & mask_];
            unsigned spins = 0;
            while (m.seq.load(std::memory_order_acquire) != pos)
                ring_detail::relax(spins);
            if (packer_) {
                // packed above
            } else {
                BatchItem<D> &it = sh.items[pos & mask_];  // ticket and features left empty by finish()
                it.state = states[i];
            }
            m.raw = raws[i];
            if (timeout_us_ > 0)
                if (sh.head.load(std::memory_order_relaxed) == pos)
                    sh.t_ns[pos & mask_] = ring_detail::now_ns();
            if (i + 1 < n)
                m.seq.store(pos + 1, std::memory_order_release);
            else
                m.seq.store(pos + 1, std::memory_order_seq_cst);
        }
        sh.inflight.fetch_sub(1, std::memory_order_release);
        const std::uint64_t depth = pos0 + n - sh.head.load(std::memory_order_seq_cst);
        // as enqueue(): wake when the shard went non-empty or a wake step was crossed
        if (depth <= n || (depth <= ring_size_ && depth / wake_step_ != (depth - n) / wake_step_))
            wake();
    }

    void enqueue(const typename D::State &state, FeatureVector features, Ticket t, TicketSlot *raw) {
        // each searcher thread stays on one shard: the tail it bumps is
        // shared with ~threads/shards others instead of with every thread
        Shard &sh = shards_[ring_detail::thread_slot() % nshards_];
        // close() waits for in-flight submits (Dekker pairing with closed_), so
        // a submit that passed the check is always drained before the agents exit
        sh.inflight.fetch_add(1, std::memory_order_seq_cst);
        if (closed_.load(std::memory_order_seq_cst)) {
            sh.inflight.fetch_sub(1, std::memory_order_release);
            throw std::runtime_error("Evaluator: submission after shutdown");
        }
        const std::uint64_t pos = sh.tail.fetch_add(1, std::memory_order_acq_rel);
        Meta &m = sh.meta[pos & mask_];
        unsigned spins = 0;
        while (m.seq.load(std::memory_order_acquire) != pos) // shard full: wait for the lap to drain
            ring_detail::relax(spins);
        BatchItem<D> &it = sh.items[pos & mask_];
        it.ticket = std::move(t);
        it.state = state;
        if (packer_)
            packer_->pack_state(state, &sh.packed[(pos & mask_) * pb_]);
        it.features = std::move(features);
        m.raw = raw;
        // only the oldest pending item's age matters (the flush deadline): an
        // item stamps its submit time when it is its shard's head; an item
        // queued behind others is stamped by the agent when it becomes the
        // head (as the reference restarts its clock after a full batch), which
        // keeps a clock read off almost every submit
        if (timeout_us_ > 0)
            if (sh.head.load(std::memory_order_relaxed) == pos)
                sh.t_ns[pos & mask_] = ring_detail::now_ns();
        m.seq.store(pos + 1, std::memory_order_seq_cst);
        sh.inflight.fetch_sub(1, std::memory_order_release);
        const std::uint64_t depth = pos + 1 - sh.head.load(std::memory_order_seq_cst);
        if (depth == 1 || (depth <= ring_size_ && depth % wake_step_ == 0))
            wake();
    }

    bool pending() const {
        for (std::size_t k = 0; k < nshards_; ++k)
            if (shards_[k].tail.load(std::memory_order_acquire) != shards_[k].head.load(std::memory_order_acquire))
                return true;
        return false;
    }

    void wake() {
        epoch_.fetch_add(1, std::memory_order_seq_cst);
        epoch_.notify_all();
    }

    // A slot is resolved only by the agent that claimed it, so a load + release
    // store replaces the reference's exchange (batch_eval.hpp:302-306; one
    // locked instruction per node less) and still counts a second resolution.
    void resolve(TicketSlot &t, std::int32_t v) {
        const std::int32_t prev = t.value.load(std::memory_order_relaxed);
        t.value.store(v, std::memory_order_release);
        if (prev != -1)
            double_resolved_.fetch_add(1, std::memory_order_relaxed);
    }

    // published items contiguous from the shard head, at most `limit`
    std::size_t published_from(const Shard &sh, std::uint64_t h, std::size_t limit) const {
        std::size_t n = 0;
        while (n < limit && sh.meta[(h + n) & mask_].seq.load(std::memory_order_acquire) == h + n + 1)
            ++n;
        return n;
    }

    // One claimed batch from claim to resolution.
    struct Flight {
        std::vector<Range> ranges;
        std::size_t n = 0;
        bool forced_partial = false;
        bool in_place = false;
        std::vector<BatchItem<D>> scratch;  // batches spanning shards or a ring end
        std::vector<std::span<const BatchItem<D>>> parts;  // gather backends: the ranges in place
        std::vector<std::span<const unsigned char>> bytes;  // pre-packing backends: packed runs
        std::vector<std::int32_t> vals;
        void *token = nullptr;              // async backend: in flight
    };

    void agent_loop() {
        std::deque<Flight> inflight;  // async: oldest first
        std::vector<Flight> spare;
        std::vector<Range> ranges;
        std::size_t rot = 0;
        std::int64_t tp0 = ring_detail::profile_on() ? ring_detail::now_ns() : 0;
        auto finish_front = [&] {
            finish(inflight.front());
            spare.push_back(std::move(inflight.front()));
            inflight.pop_front();
        };
        for (;;) {
            // completed device batches first (resolves their tickets)
            while (!inflight.empty() && async_->ready(inflight.front().token))
                finish_front();
            if (!inflight.empty() && inflight.size() >= static_cast<std::size_t>(depth_)) {
                finish_front();  // pipeline full: wait for the oldest
                continue;
            }
            const std::uint32_t e = epoch_.load(std::memory_order_seq_cst);
            // read before the scan: once set, nothing new can be published
            const bool quiesced = quiesced_.load(std::memory_order_seq_cst);
            std::unique_lock<std::mutex> lk(claim_m_);
            // published work per shard, starting from a rotating shard so no
            // shard starves when the total exceeds one batch
            ranges.clear();
            std::size_t n = 0;
            std::int64_t oldest = INT64_MAX;
            bool drained = true;
            for (std::size_t j = 0; j < nshards_ && n < capacity_; ++j) {
                const std::size_t k = (rot + j) % nshards_;
                Shard &sh = shards_[k];
                const std::uint64_t h = sh.head.load(std::memory_order_relaxed);
                const std::size_t c = published_from(sh, h, capacity_ - n);
                if (sh.tail.load(std::memory_order_acquire) != h + c)
                    drained = false;
                if (c) {
                    ranges.push_back({k, h, c});
                    n += c;
                    if (timeout_us_ > 0) {
                        std::int64_t &ht = sh.t_ns[h & mask_];  // published: its producer is done with it
                        if (ht == 0)
                            ht = ring_detail::now_ns();
                        oldest = std::min(oldest, ht);
                    }
                }
            }
            const bool closed = closed_.load(std::memory_order_acquire);
            if (n == 0) {
                lk.unlock();
                if (!inflight.empty()) {  // nothing new: complete the oldest batch
                    finish_front();
                    continue;
                }
                if (quiesced && drained)
                    return;
                if (closed || !drained) { // a producer is mid-publish
                    std::this_thread::yield();
                    continue;
                }
                epoch_.wait(e, std::memory_order_seq_cst);
                continue;
            }
            const bool full = n >= capacity_;
            const bool force = force_.load(std::memory_order_acquire);
            bool due = full || force || closed || timeout_us_ == 0;
            if (!due && timeout_us_ > 0) {
                const std::int64_t wait_ns = oldest + timeout_us_ * 1000 - ring_detail::now_ns();
                if (wait_ns <= 0) {
                    due = true;
                } else {
                    lk.unlock();
                    if (!inflight.empty()) {  // use the wait to complete in-flight work
                        finish_front();
                        continue;
                    }
                    // one agent watches the deadline; the others park on the
                    // epoch (producers wake them) instead of spinning too
                    if (deadline_owner_.exchange(true, std::memory_order_acq_rel)) {
                        epoch_.wait(e, std::memory_order_seq_cst);
                        continue;
                    }
                    // sleep_for rounds up to the timer slack (~50 us): below
                    // that, re-check between yields so a filling batch or a
                    // short deadline is seen on time
                    if (wait_ns < 200000)
                        std::this_thread::yield();
                    else
                        std::this_thread::sleep_for(std::chrono::microseconds(100));
                    deadline_owner_.store(false, std::memory_order_release);
                    continue;
                }
            } else if (!due) {
                // timeout < 0, partial batch: producers wake us at per-shard
                // steps, which need not coincide with the total reaching
                // capacity, so re-check on a short sleep as well
                lk.unlock();
                if (!inflight.empty()) {
                    finish_front();
                    continue;
                }
                std::this_thread::sleep_for(std::chrono::microseconds(50));
                continue;
            }
            for (const Range &r : ranges)
                shards_[r.shard].head.store(r.h + r.n, std::memory_order_seq_cst);
            rot = (ranges.back().shard + 1) % nshards_;
            const bool forced_partial = force && !full;
            if (force)
                force_.store(false, std::memory_order_release);
            lk.unlock();
            // another agent may proceed with the next range right away
            if (!drained || pending())
                wake();
            Flight f;
            if (!spare.empty()) {
                f = std::move(spare.back());
                spare.pop_back();
            }
            f.ranges.assign(ranges.begin(), ranges.end());
            f.n = n;
            f.forced_partial = forced_partial;
            f.token = nullptr;
            const std::int64_t tp1 = ring_detail::profile_on() ? ring_detail::now_ns() : 0;
            if (tp1)
                prof_claim_ns_.fetch_add(tp1 - tp0, std::memory_order_relaxed);
            if (packer_) {
                // the submitters' packed bytes, run by run, straight to the backend
                f.in_place = true;
                f.bytes.clear();
                for (const Range &r : f.ranges) {
                    const std::size_t at = r.h & mask_, first = std::min(r.n, ring_size_ - at);
                    const unsigned char *base = shards_[r.shard].packed.get();
                    f.bytes.emplace_back(base + at * pb_, first * pb_);
                    if (first < r.n)
                        f.bytes.emplace_back(base, (r.n - first) * pb_);
                }
                f.vals.assign(n, 0);
                packer_->evaluate_packed(f.bytes, n, f.vals);
                const std::int64_t tp2 = tp1 ? ring_detail::now_ns() : 0;
                finish(f);
                if (tp1) {
                    const std::int64_t tp3 = ring_detail::now_ns();
                    prof_eval_ns_.fetch_add(tp2 - tp1, std::memory_order_relaxed);
                    prof_finish_ns_.fetch_add(tp3 - tp2, std::memory_order_relaxed);
                    prof_batches_.fetch_add(1, std::memory_order_relaxed);
                    prof_items_.fetch_add(n, std::memory_order_relaxed);
                    tp0 = tp3;
                }
                spare.push_back(std::move(f));
                continue;
            }
            if (gather_ && !async_) {
                // the ranges in place, straight to the backend (no staging move)
                f.in_place = true;
                f.parts.clear();
                for (const Range &r : f.ranges) {
                    const std::size_t at = r.h & mask_, first = std::min(r.n, ring_size_ - at);
                    f.parts.emplace_back(&shards_[r.shard].items[at], first);
                    if (first < r.n)
                        f.parts.emplace_back(&shards_[r.shard].items[0], r.n - first);
                }
                f.vals.assign(n, 0);
                gather_->evaluate_parts(f.parts, n, f.vals);
                const std::int64_t tp2 = tp1 ? ring_detail::now_ns() : 0;
                finish(f);
                if (tp1) {
                    const std::int64_t tp3 = ring_detail::now_ns();
                    prof_eval_ns_.fetch_add(tp2 - tp1, std::memory_order_relaxed);
                    prof_finish_ns_.fetch_add(tp3 - tp2, std::memory_order_relaxed);
                    prof_batches_.fetch_add(1, std::memory_order_relaxed);
                    prof_items_.fetch_add(n, std::memory_order_relaxed);
                    tp0 = tp3;
                }
                spare.push_back(std::move(f));
                continue;
            }
            const std::span<const BatchItem<D>> items = stage(f);
            if (async_ && (f.token = async_->submit(items)) != nullptr) {
                inflight.push_back(std::move(f));
                continue;
            }
            f.vals.assign(n, 0);
            backend_->evaluate(items, f.vals);
            finish(f);
            spare.push_back(std::move(f));
        }
    }

    // The batch's items as one span: in place in the ring, or moved into the
    // flight's scratch when it spans shards or wraps.
    std::span<const BatchItem<D>> stage(Flight &f) {
        const Range &r0 = f.ranges.front();
        f.in_place = f.ranges.size() == 1 && (r0.h & mask_) + r0.n <= ring_size_;
        if (f.in_place)
            return std::span<const BatchItem<D>>(&shards_[r0.shard].items[r0.h & mask_], f.n);
        f.scratch.clear();
        for (const Range &r : f.ranges)
            for (std::size_t i = 0; i < r.n; ++i)
                f.scratch.push_back(std::move(shards_[r.shard].items[(r.h + i) & mask_]));
        return std::span<const BatchItem<D>>(f.scratch);
    }

    // Resolves the flight's tickets (in bulk, from the ring slots), releases the
    // slots for the producers' next lap and records the batch.
    void finish(Flight &f) {
        BIDA_NVTX_PUSH(f.forced_partial ? "ring flush (forced)" : "ring flush");
        if (f.token) {
            f.vals.assign(f.n, 0);
            async_->complete(f.token, f.vals);
            f.token = nullptr;
        }
        std::size_t o = 0;
        for (const Range &r : f.ranges) {
            Shard &sh = shards_[r.shard];
            for (std::size_t i = 0; i < r.n; ++i, ++o) {
                Meta &mt = sh.meta[(r.h + i) & mask_];
                // caller-owned slots live in the searchers' caches: request the
                // line for writing a few items ahead of the resolving store
                if (i + 8 < r.n)
                    if (TicketSlot *ahead = sh.meta[(r.h + i + 8) & mask_].raw)
                        __builtin_prefetch(ahead, 1, 3);
                if (mt.raw && !feats_) {
                    // no ticket, no features: the item's line is not touched at all
                    resolve(*mt.raw, f.vals[o]);
                    continue;
                }
                BatchItem<D> &it = f.in_place ? sh.items[(r.h + i) & mask_] : f.scratch[o];
                resolve(mt.raw ? *mt.raw : *it.ticket, f.vals[o]);
                // every submit rewrites raw; caller-owned slots carry no ticket: no
                // stores to the item or meta line beyond the seq release below
                if (it.ticket)
                    it.ticket.reset();
                if (!it.features.empty())
                    FeatureVector().swap(it.features);
            }
            sh.t_ns[r.h & mask_] = 0;  // only a range's head can carry a stamp
            for (std::size_t i = 0; i < r.n; ++i)
                sh.meta[(r.h + i) & mask_].seq.store(r.h + i + ring_size_, std::memory_order_release);
        }
        resolved_.fetch_add(f.n, std::memory_order_relaxed);
        {
            std::lock_guard<std::mutex> slk(stats_m_);
            stats_.record_batch(f.n);
            if (f.forced_partial)
                ++stats_.forced_flushes;
        }
        BIDA_NVTX_POP();
    }

    std::unique_ptr<EvaluatorBackend<D>> backend_;
    std::size_t capacity_;
    std::int64_t timeout_us_;
    bool immediate_;

    std::size_t nshards_ = 1;
    std::size_t ring_size_ = 0; // per shard
    std::uint64_t mask_ = 0;
    std::uint64_t wake_step_ = 1;
    std::unique_ptr<Shard[]> shards_;
    alignas(64) std::atomic<std::uint32_t> epoch_{0};
    std::atomic<bool> force_{false};
    std::atomic<bool> closed_{false};
    std::atomic<bool> deadline_owner_{false};
    std::atomic<bool> quiesced_{false};  // close(): closed_ set and no submit in flight
    AsyncEvaluatorBackend<D> *async_ = nullptr;  // set: agents pipeline depth_ batches each
    GatherEvaluatorBackend<D> *gather_ = nullptr;  // set: synchronous batches evaluated in place
    PackedGatherBackend<D> *packer_ = nullptr;     // set: submitters pack, agents pass packed runs
    std::size_t pb_ = 0;
    bool feats_ = true;  // backend_->needs_features(), read once
    std::atomic<std::int64_t> prof_claim_ns_{0}, prof_eval_ns_{0}, prof_finish_ns_{0};  // BIDA_RING_PROFILE
    std::atomic<std::uint64_t> prof_batches_{0}, prof_items_{0};
    int depth_ = 1;
    std::mutex claim_m_;
    std::vector<std::thread> agents_;

    mutable std::mutex stats_m_;
    SearchStats stats_;

    std::atomic<std::uint64_t> immediate_submitted_{0};
    std::atomic<std::uint64_t> resolved_{0};
    std::atomic<std::uint64_t> double_resolved_{0};
};

// Searcher thread tid goes to evaluator tid % E (batch_eval.hpp:398-400).
template <class D>
class EvaluatorGroup {
public:
    EvaluatorGroup(std::vector<std::unique_ptr<EvaluatorBackend<D>>> backends, std::size_t capacity,
                   std::int64_t timeout_us, bool immediate = false) {
        if (backends.empty())
            throw std::invalid_argument("EvaluatorGroup: need at least one evaluator");
        for (auto &b : backends)
            evs_.push_back(std::make_unique<Evaluator<D>>(std::move(b), capacity, timeout_us, immediate));
    }

    std::size_t evaluator_count() const { return evs_.size(); }
    int evaluator_of(int thread_id) const { return thread_id % static_cast<int>(evs_.size()); }
    Evaluator<D> &evaluator(std::size_t i) { return *evs_[i]; }

    Ticket submit(int thread_id, const typename D::State &state, FeatureVector features) {
        return of(thread_id).submit(state, std::move(features));
    }

    Ticket submit_state(int thread_id, const typename D::State &state) {
        Evaluator<D> &e = of(thread_id);
        FeatureVector x;
        if (e.needs_features()) {
            x.resize(static_cast<std::size_t>(D::feature_length()));
            D::encode(state, x.data());
        }
        return e.submit(state, std::move(x));
    }

    // Extension (CB-DFS overlay): submit_state with a caller-owned ticket slot.
    void submit_state_slot(int thread_id, const typename D::State &state, TicketSlot *slot) {
        Evaluator<D> &e = of(thread_id);
        FeatureVector x;
        if (e.needs_features()) {
            x.resize(static_cast<std::size_t>(D::feature_length()));
            D::encode(state, x.data());
        }
        e.submit_slot(state, std::move(x), slot);
    }

    // Extension (CB-DFS overlay): one expansion's children in one reservation.
    void submit_states_slots(int thread_id, const typename D::State *states, TicketSlot *const *slots,
                             std::size_t n) {
        of(thread_id).submit_slots(states, slots, n);
    }

    bool needs_features() const { return evs_.front()->needs_features(); }

    int evaluate_single(const typename D::State &state) {
        FeatureVector x(static_cast<std::size_t>(D::feature_length()));
        D::encode(state, x.data());
        return evs_.front()->evaluate_single(state, std::move(x));
    }

    std::vector<int> evaluate_sync(std::span<const typename D::State> states) {
        return evs_.front()->evaluate_sync(states);
    }

    void kick(int thread_id) { of(thread_id).request_flush(); }
    void kick_all() {
        for (auto &e : evs_)
            e->request_flush();
    }
    void close() {
        for (auto &e : evs_)
            e->close();
    }

    SearchStats stats_snapshot() const {
        SearchStats s;
        for (const auto &e : evs_)
            s.merge(e->stats_snapshot());
        s.iterations.clear();
        return s;
    }

    std::uint64_t submitted() const { return sum(&Evaluator<D>::submitted); }
    std::uint64_t resolved() const { return sum(&Evaluator<D>::resolved); }
    std::uint64_t double_resolutions() const { return sum(&Evaluator<D>::double_resolutions); }

private:
    Evaluator<D> &of(int thread_id) { return *evs_[static_cast<std::size_t>(evaluator_of(thread_id))]; }
    std::uint64_t sum(std::uint64_t (Evaluator<D>::*f)() const) const {
        std::uint64_t n = 0;
        for (const auto &e : evs_)
            n += ((*e).*f)();
        return n;
    }

    std::vector<std::unique_ptr<Evaluator<D>>> evs_;
};

template <class D>
EvaluatorGroup<D> make_table_sim_group(std::shared_ptr<const Heuristic<D>> source, std::size_t evaluators,
                                       std::size_t capacity, std::int64_t timeout_us, std::int64_t per_call_us = 0,
                                       std::int64_t per_item_ns = 0, bool immediate = false) {
    std::vector<std::unique_ptr<EvaluatorBackend<D>>> v;
    for (std::size_t i = 0; i < evaluators; ++i)
        v.push_back(std::make_unique<TableSimBackend<D>>(source, per_call_us, per_item_ns));
    return EvaluatorGroup<D>(std::move(v), capacity, timeout_us, immediate);
}

} // namespace bida
