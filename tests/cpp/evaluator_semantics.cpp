// Evaluator semantics, restated from the reference's own unit tests
// (/root/reference/proj/tests/test_batch_eval.cpp:35-118, 120-141, 243-268;
// Catch2 is absent here, so plain checks).  Built twice by tests/cpp/Makefile:
// against the reference's batch_eval.hpp (bin/evaluator_semantics_ref, the
// control) and against the ring evaluator overlay (bin/evaluator_semantics_ring,
// include/bida_ring_evaluator.hpp).  Exit 0 = every check passed.
#include <algorithm>
#include <array>
#include <atomic>
#include <cstring>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <random>
#include <thread>
#include <vector>

#include "bida/batch_eval.hpp"
#include "bida/heuristic.hpp"
#include "bida/stp.hpp"

using namespace bida;
using D = TilePuzzle<3>;

static int failures = 0;
#define CHECK(c)                                                                \
    do {                                                                        \
        if (!(c)) {                                                             \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                         \
        }                                                                       \
    } while (0)

namespace {
D::State walk(std::mt19937_64 &rng, int steps = 30) {
    D::State s = D::solved();
    D::Action last = D::kNoAction;
    for (int i = 0; i < steps; ++i) {
        std::array<D::Action, 4> acts{};
        const int n = D::actions(s, last, true, acts);
        last = acts[static_cast<std::size_t>(std::uniform_int_distribution<int>(0, n - 1)(rng))];
        s = D::apply(s, last);
    }
    return s;
}
std::shared_ptr<const Heuristic<D>> man() { return std::make_shared<ManhattanHeuristic<3>>(); }
std::unique_ptr<EvaluatorBackend<D>> sim() { return std::make_unique<TableSimBackend<D>>(man()); }
#ifdef BIDA_RING_EVALUATOR
// A device stand-in for the ring's asynchronous path: submit() computes the
// values at once but reports them ready only `delay_us` later (a device round
// trip), so agents keep several batches in flight.
class AsyncSim final : public EvaluatorBackend<D>, public ConcurrentBackend, public AsyncEvaluatorBackend<D> {
public:
    explicit AsyncSim(int delay_us, int lanes = 8) : delay_ns_(delay_us * 1000ll), lanes_(lanes) {}
    void evaluate(std::span<const BatchItem<D>> batch, std::span<std::int32_t> out) override {
        for (std::size_t i = 0; i < batch.size(); ++i)
            out[i] = mh_.lookup(batch[i].state);
        sync_calls_.fetch_add(1);
    }
    int max_concurrent_calls() const override { return 4; }
    int max_in_flight() const override { return lanes_; }
    void *submit(std::span<const BatchItem<D>> batch) override {
        const int now_in = in_flight_.fetch_add(1) + 1;
        int peak = peak_.load();
        while (now_in > peak && !peak_.compare_exchange_weak(peak, now_in)) {
        }
        auto *t = new Token;
        t->ready_ns = now() + delay_ns_;
        for (const auto &it : batch)
            t->vals.push_back(mh_.lookup(it.state));
        return t;
    }
    bool ready(void *token) override { return now() >= static_cast<Token *>(token)->ready_ns; }
    void complete(void *token, std::span<std::int32_t> out) override {
        auto *t = static_cast<Token *>(token);
        while (now() < t->ready_ns)
            std::this_thread::yield();
        std::copy(t->vals.begin(), t->vals.end(), out.begin());
        delete t;
        in_flight_.fetch_sub(1);
    }
    int peak_in_flight() const { return peak_.load(); }
    int in_flight() const { return in_flight_.load(); }
    int sync_calls() const { return sync_calls_.load(); }

private:
    struct Token {
        std::int64_t ready_ns = 0;
        std::vector<std::int32_t> vals;
    };
    static std::int64_t now() {
        return std::chrono::duration_cast<std::chrono::nanoseconds>(
                   std::chrono::steady_clock::now().time_since_epoch())
            .count();
    }
    ManhattanHeuristic<3> mh_;
    std::int64_t delay_ns_;
    int lanes_;
    std::atomic<int> in_flight_{0}, peak_{0}, sync_calls_{0};
};
// The ring's gather path (bida_gpu::GpuBackend implements it): the claimed
// ranges arrive in place, one span per contiguous run; several agents at once.
class GatherSim final : public EvaluatorBackend<D>, public ConcurrentBackend, public GatherEvaluatorBackend<D> {
public:
    void evaluate(std::span<const BatchItem<D>> batch, std::span<std::int32_t> out) override {
        for (std::size_t i = 0; i < batch.size(); ++i)
            out[i] = mh_.lookup(batch[i].state);
        plain_.fetch_add(1);
    }
    void evaluate_parts(std::span<const std::span<const BatchItem<D>>> parts, std::size_t n,
                        std::span<std::int32_t> out) override {
        std::size_t o = 0;
        for (const auto &part : parts)
            for (const auto &it : part)
                out[o++] = mh_.lookup(it.state);
        if (o != n)
            bad_.fetch_add(1);
        gathered_.fetch_add(1);
        if (parts.size() > 1)
            multi_.fetch_add(1);
    }
    bool needs_features() const override { return false; }
    int max_concurrent_calls() const override { return 4; }
    int plain() const { return plain_.load(); }
    int gathered() const { return gathered_.load(); }
    int multi_part() const { return multi_.load(); }
    int bad() const { return bad_.load(); }

private:
    ManhattanHeuristic<3> mh_;
    std::atomic<int> plain_{0}, gathered_{0}, multi_{0}, bad_{0};
};
// The ring's pre-packing path: submitters "pack" a state into 4 bytes (here
// its Manhattan value itself), the agent hands the claimed runs back as bytes.
class PackedSim final : public EvaluatorBackend<D>, public ConcurrentBackend, public GatherEvaluatorBackend<D>,
                        public PackedGatherBackend<D> {
public:
    void evaluate(std::span<const BatchItem<D>> batch, std::span<std::int32_t> out) override {
        for (std::size_t i = 0; i < batch.size(); ++i)
            out[i] = mh_.lookup(batch[i].state);
        plain_.fetch_add(1);
    }
    void evaluate_parts(std::span<const std::span<const BatchItem<D>>>, std::size_t, std::span<std::int32_t> out) override {
        for (auto &v : out)
            v = 0;
        gathered_.fetch_add(1);  // must not be used: the packed path wins
    }
    std::size_t packed_bytes() const override { return 4; }
    void pack_state(const D::State &st, unsigned char *dst) const override {
        const std::int32_t v = mh_.lookup(st);
        std::memcpy(dst, &v, 4);
    }
    void evaluate_packed(std::span<const std::span<const unsigned char>> parts, std::size_t n,
                         std::span<std::int32_t> out) override {
        std::size_t o = 0;
        for (const auto &part : parts)
            for (std::size_t b = 0; b + 4 <= part.size(); b += 4)
                std::memcpy(&out[o++], part.data() + b, 4);
        if (o != n)
            bad_.fetch_add(1);
        packed_calls_.fetch_add(1);
        if (parts.size() > 1)
            multi_.fetch_add(1);
    }
    bool needs_features() const override { return false; }
    int max_concurrent_calls() const override { return 4; }
    int plain() const { return plain_.load(); }
    int gathered() const { return gathered_.load(); }
    int packed_calls() const { return packed_calls_.load(); }
    int multi_part() const { return multi_.load(); }
    int bad() const { return bad_.load(); }

private:
    ManhattanHeuristic<3> mh_;
    std::atomic<int> plain_{0}, gathered_{0}, packed_calls_{0}, multi_{0}, bad_{0};
};
#endif
void wait_all(const std::vector<Ticket> &ts, double seconds) {
    const auto end = std::chrono::steady_clock::now() + std::chrono::duration<double>(seconds);
    for (const auto &t : ts)
        while (poll(t) < 0 && std::chrono::steady_clock::now() < end)
            std::this_thread::yield();
}
} // namespace

int main() {
    ManhattanHeuristic<3> mh;
    { // a full buffer is exactly one flush, values equal direct lookups
        Evaluator<D> ev(sim(), 8, -1);
        std::mt19937_64 rng(1);
        std::vector<D::State> ss;
        std::vector<Ticket> ts;
        for (int i = 0; i < 8; ++i) {
            ss.push_back(walk(rng));
            ts.push_back(ev.submit(ss.back(), {}));
        }
        wait_all(ts, 2);
        for (int i = 0; i < 8; ++i)
            CHECK(poll(ts[i]) == mh.lookup(ss[i]));
        ev.close();  // tickets resolve before record_batch runs (batch_eval.hpp:350-352): join first
        const SearchStats st = ev.stats_snapshot();
        CHECK(st.batches == 1 && st.batch_items == 8 && st.max_batch_occupancy == 8);
    }
    { // timeout flushes a partial batch
        Evaluator<D> ev(sim(), 1024, 2000);
        const Ticket t = ev.submit(D::solved(), {});
        wait_all({t}, 2);
        CHECK(poll(t) == 0);
        ev.close();
        CHECK(ev.stats_snapshot().batches == 1);
    }
    { // no submissions, no flushes
        Evaluator<D> ev(sim(), 4, 100);
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
        CHECK(ev.stats_snapshot().batches == 0);
    }
    { // timeout disabled: flushes = submissions / capacity
        const std::size_t B = 16;
        Evaluator<D> ev(sim(), B, -1);
        std::mt19937_64 rng(2);
        std::vector<Ticket> ts;
        for (std::size_t i = 0; i < 10 * B; ++i)
            ts.push_back(ev.submit(walk(rng), {}));
        wait_all(ts, 5);
        ev.close();
        const SearchStats st = ev.stats_snapshot();
        CHECK(st.batches == 10 && st.batch_items == 10 * B && st.max_batch_occupancy == B);
    }
    { // close drains, then submissions throw
        Evaluator<D> ev(sim(), 1024, -1);
        std::mt19937_64 rng(3);
        std::vector<Ticket> ts;
        for (int i = 0; i < 37; ++i)
            ts.push_back(ev.submit(walk(rng), {}));
        ev.close();
        for (const auto &t : ts)
            CHECK(poll(t) >= 0);
        bool threw = false;
        try {
            ev.submit(D::solved(), {});
        } catch (const std::runtime_error &) {
            threw = true;
        }
        CHECK(threw);
    }
    { // request_flush forces one partial batch
        Evaluator<D> ev(sim(), 1024, -1);
        const Ticket t = ev.submit(D::solved(), {});
        ev.request_flush();
        wait_all({t}, 2);
        CHECK(poll(t) == 0);
        ev.close();
        CHECK(ev.stats_snapshot().forced_flushes == 1);
    }
    { // group: evaluate_single, even routing
        EvaluatorGroup<D> g = make_table_sim_group<D>(man(), 2, 8, 0);
        CHECK(g.evaluate_single(D::solved()) == 0);
        std::mt19937_64 rng(4);
        for (int i = 0; i < 50; ++i) {
            const D::State s = walk(rng);
            CHECK(g.evaluate_single(s) == mh.lookup(s));
        }
        std::array<int, 2> load{};
        for (int tid = 0; tid < 4; ++tid)
            ++load[static_cast<std::size_t>(g.evaluator_of(tid))];
        CHECK(load[0] == 2 && load[1] == 2);
        g.close();
    }
    { // liveness under randomized schedules: 200 rounds of random capacity,
      // timeout, bursts, kicks and mid-flight shutdowns
        std::mt19937_64 rng(7);
        std::uint64_t doubled = 0;
        for (int round = 0; round < 200; ++round) {
            const std::size_t B = 1 + rng() % 16;
            const std::int64_t timeout = static_cast<std::int64_t>(rng() % 3) - 1;
            Evaluator<D> ev(sim(), B, timeout);
            std::vector<Ticket> ts;
            const int count = static_cast<int>(rng() % 40);
            for (int i = 0; i < count; ++i) {
                ts.push_back(ev.submit(walk(rng, 6), {}));
                if (rng() % 8 == 0)
                    ev.request_flush();
                if (rng() % 16 == 0)
                    std::this_thread::yield();
            }
            ev.close();
            for (const auto &t : ts)
                CHECK(poll(t) >= 0);
            CHECK(ev.submitted() == ev.resolved());
            doubled += ev.double_resolutions();
        }
        CHECK(doubled == 0);
    }
    { // many producer threads into one evaluator (beyond the reference tests):
      // every ticket resolved to its own state's value, none twice
        Evaluator<D> ev(sim(), 64, 0);
        std::vector<std::thread> th;
        std::vector<std::vector<std::pair<D::State, Ticket>>> got(8);
        for (int k = 0; k < 8; ++k)
            th.emplace_back([&, k] {
                std::mt19937_64 rng(100 + k);
                for (int i = 0; i < 20000; ++i) {
                    const D::State s = walk(rng, 8);
                    got[k].emplace_back(s, ev.submit(s, {}));
                }
            });
        for (auto &t : th)
            t.join();
        ev.close();
        std::size_t n = 0;
        for (auto &v : got)
            for (auto &[s, t] : v) {
                CHECK(poll(t) == mh.lookup(s));
                ++n;
            }
        CHECK(n == 160000 && ev.submitted() == n && ev.resolved() == n && ev.double_resolutions() == 0);
        CHECK(ev.stats_snapshot().batch_items == n);
    }
#ifdef BIDA_RING_EVALUATOR
    { // ring only: more shards than 8 with a large batch and no timeout:
      // every shard holds a full batch, so a lone producer never stalls
        Evaluator<D> ev(sim(), 16384, -1, false, 1, 16);
        std::mt19937_64 rng(11);
        std::vector<Ticket> ts;
        for (int i = 0; i < 40000; ++i)
            ts.push_back(ev.submit(walk(rng, 5), {}));
        ev.request_flush();
        wait_all(ts, 10);
        ev.close();
        for (const auto &t : ts)
            CHECK(poll(t) >= 0);
        CHECK(ev.stats_snapshot().batches == 3);
    }
    { // ring only: caller-owned ticket slots (submit_slot), resolved in place
        Evaluator<D> ev(sim(), 32, 0, false, 2, 4);
        std::mt19937_64 rng(12);
        std::vector<TicketSlot> slots(5000);
        std::vector<D::State> ss;
        for (auto &sl : slots) {
            ss.push_back(walk(rng, 7));
            ev.submit_slot(ss.back(), {}, &sl);
        }
        ev.close();
        for (std::size_t i = 0; i < slots.size(); ++i)
            CHECK(slots[i].value.load() == mh.lookup(ss[i]));
        CHECK(ev.resolved() == slots.size() && ev.double_resolutions() == 0);
    }
    { // ring only: submits racing close(): every accepted submit is resolved,
      // every other one throws; nothing hangs
        for (int round = 0; round < 50; ++round) {
            Evaluator<D> ev(sim(), 8, -1, false, 2, 4);
            std::atomic<bool> go{true};
            std::vector<std::thread> th;
            std::vector<std::vector<Ticket>> got(4);
            for (int k = 0; k < 4; ++k)
                th.emplace_back([&, k] {
                    std::mt19937_64 rng(1000 * round + k);
                    while (go.load()) {
                        try {
                            got[k].push_back(ev.submit(walk(rng, 4), {}));
                        } catch (const std::runtime_error &) {
                            return;
                        }
                    }
                });
            std::this_thread::sleep_for(std::chrono::microseconds(200 + 37 * round));
            ev.close();
            go.store(false);
            for (auto &t : th)
                t.join();
            for (auto &v : got)
                for (auto &t : v)
                    CHECK(poll(t) >= 0);
            CHECK(ev.submitted() == ev.resolved());
        }
    }
    { // ring only: asynchronous backend, agents pipelining several batches each;
      // every ticket resolved to its own value once, in-flight batches drained
      // by close(), never more than the backend's lanes in flight
        // an async-capable backend with BIDA_EVAL_INFLIGHT unset: synchronous calls
        unsetenv("BIDA_EVAL_INFLIGHT");
        {
            auto sb = std::make_unique<AsyncSim>(50);
            AsyncSim *sraw = sb.get();
            Evaluator<D> sev(std::move(sb), 16, 0, false, 2, 4);
            CHECK(sev.in_flight_per_agent() == 1);
            std::mt19937_64 srng(301);
            std::vector<std::pair<D::State, Ticket>> sv;
            for (int i = 0; i < 3000; ++i) {
                const D::State s = walk(srng, 8);
                sv.emplace_back(s, sev.submit(s, {}));
            }
            sev.close();
            for (auto &[s, t] : sv)
                CHECK(poll(t) == mh.lookup(s));
            CHECK(sraw->peak_in_flight() == 0 && sraw->sync_calls() > 0);
        }
        setenv("BIDA_EVAL_INFLIGHT", "4", 1);
        auto be = std::make_unique<AsyncSim>(200);
        AsyncSim *raw = be.get();
        Evaluator<D> ev(std::move(be), 16, 0, false, 2, 4);
        CHECK(ev.in_flight_per_agent() == 4);
        std::vector<std::thread> th;
        std::vector<std::vector<std::pair<D::State, Ticket>>> got(6);
        for (int k = 0; k < 6; ++k)
            th.emplace_back([&, k] {
                std::mt19937_64 rng(300 + k);
                for (int i = 0; i < 5000; ++i) {
                    const D::State s = walk(rng, 8);
                    got[k].emplace_back(s, ev.submit(s, {}));
                }
            });
        for (auto &t : th)
            t.join();
        ev.close();
        std::size_t n = 0;
        for (auto &v : got)
            for (auto &[s, t] : v) {
                CHECK(poll(t) == mh.lookup(s));
                ++n;
            }
        CHECK(n == 30000 && ev.resolved() == n && ev.double_resolutions() == 0);
        CHECK(ev.stats_snapshot().batch_items == n);
        CHECK(raw->in_flight() == 0 && raw->peak_in_flight() > 1 && raw->peak_in_flight() <= 8);
    }
    { // ring only: asynchronous backend under the reference flush policies and
      // randomized shutdowns (liveness, as the synchronous rounds above)
        std::mt19937_64 rng(17);
        for (int round = 0; round < 100; ++round) {
            const std::size_t B = 1 + rng() % 16;
            const std::int64_t timeout = static_cast<std::int64_t>(rng() % 3) - 1;
            Evaluator<D> ev(std::make_unique<AsyncSim>(static_cast<int>(rng() % 50)), B, timeout, false,
                            1 + static_cast<int>(rng() % 3), 2);
            std::vector<Ticket> ts;
            const int count = static_cast<int>(rng() % 60);
            for (int i = 0; i < count; ++i) {
                ts.push_back(ev.submit(walk(rng, 6), {}));
                if (rng() % 8 == 0)
                    ev.request_flush();
            }
            ev.close();
            for (const auto &t : ts)
                CHECK(poll(t) >= 0);
            CHECK(ev.submitted() == ev.resolved());
            CHECK(ev.double_resolutions() == 0);
        }
    }
    { // ring only: timeout disabled with an async backend: flushes = submissions / capacity
        const std::size_t B = 16;
        Evaluator<D> ev(std::make_unique<AsyncSim>(100), B, -1, false, 2, 2);
        std::mt19937_64 rng(21);
        std::vector<Ticket> ts;
        for (std::size_t i = 0; i < 10 * B; ++i)
            ts.push_back(ev.submit(walk(rng), {}));
        wait_all(ts, 5);
        ev.close();
        const SearchStats st = ev.stats_snapshot();
        CHECK(st.batches == 10 && st.batch_items == 10 * B && st.max_batch_occupancy == B);
    }
    { // ring only: gather backend + caller-owned slots submitted an expansion at a
      // time (submit_slots: one reservation for up to 18 items), 4 agents over 8
      // shards and 6 producers; every slot resolved once to its own value
        auto gb = std::make_unique<GatherSim>();
        GatherSim *graw = gb.get();
        Evaluator<D> ev(std::move(gb), 64, 20, false, 4, 8);
        constexpr int kPer = 4000;
        std::vector<std::vector<D::State>> states(6);
        std::vector<std::unique_ptr<TicketSlot[]>> slots(6);
        std::vector<std::thread> th;
        for (int k = 0; k < 6; ++k) {
            slots[k] = std::make_unique<TicketSlot[]>(kPer);
            th.emplace_back([&, k] {
                std::mt19937_64 rng(500 + k);
                for (int i = 0; i < kPer; ++i)
                    states[k].push_back(walk(rng, 8));
                for (int i = 0; i < kPer;) {
                    const int m = std::min<int>(1 + static_cast<int>(rng() % 18), kPer - i);
                    std::vector<TicketSlot *> ps;
                    for (int j = 0; j < m; ++j)
                        ps.push_back(&slots[k][i + j]);
                    ev.submit_slots(&states[k][i], ps.data(), static_cast<std::size_t>(m));
                    i += m;
                }
            });
        }
        for (auto &t : th)
            t.join();
        ev.close();
        std::size_t n = 0;
        for (int k = 0; k < 6; ++k)
            for (int i = 0; i < kPer; ++i, ++n)
                CHECK(slots[k][i].value.load() == mh.lookup(states[k][i]));
        CHECK(n == 6u * kPer && ev.resolved() == n && ev.double_resolutions() == 0);
        CHECK(graw->gathered() > 0 && graw->plain() == 0 && graw->bad() == 0 && graw->multi_part() > 0);
        CHECK(ev.stats_snapshot().batch_items == n);
    }
    { // ring only: pre-packing backend; reservations and single submits (tickets)
      // mixed, 4 agents, 8 shards, 6 producers: every value lands in its own slot
        auto pb = std::make_unique<PackedSim>();
        PackedSim *praw = pb.get();
        Evaluator<D> ev(std::move(pb), 64, 20, false, 4, 8);
        constexpr int kPer = 4000;
        std::vector<std::vector<D::State>> states(6);
        std::vector<std::unique_ptr<TicketSlot[]>> slots(6);
        std::vector<std::vector<std::pair<D::State, Ticket>>> tickets(6);
        std::vector<std::thread> th;
        for (int k = 0; k < 6; ++k) {
            slots[k] = std::make_unique<TicketSlot[]>(kPer);
            th.emplace_back([&, k] {
                std::mt19937_64 rng(700 + k);
                for (int i = 0; i < kPer; ++i)
                    states[k].push_back(walk(rng, 8));
                for (int i = 0; i < kPer;) {
                    const int m = std::min<int>(1 + static_cast<int>(rng() % 18), kPer - i);
                    std::vector<TicketSlot *> ps;
                    for (int j = 0; j < m; ++j)
                        ps.push_back(&slots[k][i + j]);
                    ev.submit_slots(&states[k][i], ps.data(), static_cast<std::size_t>(m));
                    i += m;
                    if (rng() % 4 == 0) {
                        const D::State s = walk(rng, 8);
                        tickets[k].emplace_back(s, ev.submit(s, {}));
                    }
                }
            });
        }
        for (auto &t : th)
            t.join();
        ev.close();
        std::size_t n = 0;
        for (int k = 0; k < 6; ++k) {
            for (int i = 0; i < kPer; ++i, ++n)
                CHECK(slots[k][i].value.load() == mh.lookup(states[k][i]));
            for (auto &[s, t] : tickets[k]) {
                CHECK(poll(t) == mh.lookup(s));
                ++n;
            }
        }
        CHECK(ev.resolved() == n && ev.double_resolutions() == 0);
        CHECK(praw->packed_calls() > 0 && praw->gathered() == 0 && praw->plain() == 0 && praw->bad() == 0 &&
              praw->multi_part() > 0);
    }
    std::printf("ring evaluator: %s\n", failures ? "FAILED" : "all checks passed");
#else
    std::printf("reference evaluator: %s\n", failures ? "FAILED" : "all checks passed");
#endif
    return failures ? 1 : 0;
}
