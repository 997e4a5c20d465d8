// bida_fast_cbdfs.hpp — the reference's CB-DFS searcher loop with its
// per-node host costs removed, same public entry point.
//
//   reference: bida::cb_dfs / do_iteration / Frame / Work
//              /root/reference/proj/include/bida/cbdfs.hpp:33-52, 232-415
//
// With the ring evaluator (include/bida_ring_evaluator.hpp) the device is no
// longer the cap; the reference's searcher loop is (profiles/r1_search_ring_*):
//
//   * every child copies its parent's action path (cbdfs.hpp:318-319): a heap
//     vector per generated node, O(depth) bytes;
//   * every child heap-allocates a shared_ptr ticket (batch_eval.hpp:212) whose
//     refcount is touched by the searcher, the ring and the agent;
//   * every expansion bumps one process-wide atomic (cbdfs.hpp:289), a cache
//     line all searcher threads write.
//
// Here, with the reference's expansion order, pruning, goal test, stop
// checks, all-blocked kick and statistics unchanged:
//
//   * a frame is {state, g, h, ticket slot, last action} -- no path.  The path
//     from the work root is kept once per work in `path_`: when a frame at
//     depth d (relative to the work root) is expanded, every frame above it in
//     the DFS has already been popped, so path_[0..d-1) is still its
//     ancestors' actions and only path_[d-1] = frame.last changes.  The full
//     path is materialised only when a goal is found;
//   * ticket slots live in a per-work arena indexed by stack position (stable
//     addresses; an expansion's children get adjacent slots, reused once read)
//     and are handed to the evaluator in one reservation per expansion
//     (submit_states_slots), which resolves them in place;
//   * expansions are added to the shared counter once per round-robin cycle
//     (where the reference reads it for the budget check) instead of once per
//     node.
//
// On stop (goal, budget, deadline) frames may still be pending in the
// evaluator: the thread forces flushes and waits for its own slots to resolve
// before it returns, so no evaluator thread ever writes into a released arena.
#pragma once

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <deque>
#include <memory>
#include <thread>
#include <vector>

namespace bida {

namespace fast_cbdfs {

inline int idle_sleep_us() {
    static const int us = [] {
        const char *v = std::getenv("BIDA_SEARCH_IDLE_SLEEP_US");
        return v ? std::atoi(v) : 0;
    }();
    return us;
}

template <class D>
struct FastFrame {
    typename D::State state;
    int g = 0;
    int h = -1;                  // -1 while the slot is unresolved
    TicketSlot *slot = nullptr;  // pending evaluation (h < 0), else nullptr
    typename D::Action last = D::kNoAction;
};

template <class D>
struct FastWork {
    const WorkSeed<D> *seed = nullptr;
    std::vector<FastFrame<D>> stack;
    // slot of the frame at stack position i: an expansion's children sit at
    // consecutive positions, so their slots share cache lines -- the agent
    // resolves them with one or two line transfers, and the searcher's poll of
    // the first brings its siblings' values along.  A position is reused only
    // after its frame was popped, i.e. after its value was read.
    std::deque<TicketSlot> slot_arena;
    TicketSlot *slot_at(std::size_t i) {
        while (slot_arena.size() <= i)
            slot_arena.emplace_back();
        TicketSlot *t = &slot_arena[i];
        t->value.store(-1, std::memory_order_relaxed);
        return t;
    }
    std::vector<typename D::Action> path;  // path[i]: action at depth i+1 below the work root
    int root_g = 0;
    bool done() const { return stack.empty(); }
};

template <class D>
class Searcher {
public:
    Searcher(int tid, std::int64_t bound, EvaluatorGroup<D> &group, BoundCollector &collector,
             IterationShared<D> &shared, SearchStats &stats, const ExpandHook<D> *on_expand)
        : tid_(tid), bound_(bound), group_(group), collector_(collector), shared_(shared), stats_(stats),
          on_expand_(on_expand) {}

    // detail::push_root_frame (cbdfs.hpp:232-247)
    void push_root(FastWork<D> &w, const WorkSeed<D> *seed) {
        w.seed = seed;
        w.stack.clear();
        w.path.clear();
        FastFrame<D> f;
        f.state = seed->root;
        f.g = static_cast<int>(seed->init_history.size());
        w.root_g = f.g;
        f.h = seed->root_h;
        if (f.h < 0) {
            f.slot = w.slot_at(0);
            group_.submit_state_slot(tid_, f.state, f.slot);
        }
        f.last = seed->init_history.empty() ? D::kNoAction : seed->init_history.back();
        w.stack.push_back(f);
        ++live_;
        if (live_ > stats_.peak_live_frames)
            stats_.peak_live_frames = live_;
    }

    // do_iteration (cbdfs.hpp:254-330)
    StepStatus step(FastWork<D> &w) {
        for (;;) {
            if (w.stack.empty())
                return StepStatus::Done;
            FastFrame<D> &top = w.stack.back();
            if (top.h < 0) {
                const int v = top.slot->value.load(std::memory_order_acquire);
                if (v < 0)
                    return StepStatus::Blocked;
                top.h = v;
                top.slot = nullptr;
            }
            const std::int64_t f = top.g + top.h;
            if (f > bound_) {
                collector_.record(tid_, f);
                w.stack.pop_back();
                --live_;
                continue;
            }
            const FastFrame<D> parent = top;
            w.stack.pop_back();
            --live_;
            ++stats_.expanded;
            ++unflushed_expanded_;
            if (on_expand_ && *on_expand_)
                (*on_expand_)(parent.state, parent.g);
            // the parent's own action joins the path at its depth
            const int d = parent.g - w.root_g;
            if (d > 0) {
                w.path.resize(static_cast<std::size_t>(d));
                w.path[static_cast<std::size_t>(d - 1)] = parent.last;
            } else {
                w.path.clear();
            }
            std::array<typename D::Action, D::kMaxBranching> acts{};
            const int n = D::actions(parent.state, parent.last, /*prune=*/true, acts);
            // children are submitted together after the loop (one ring reservation)
            std::size_t nk = 0;
            for (int i = 0; i < n; ++i) {
                const typename D::Action a = acts[static_cast<std::size_t>(i)];
                FastFrame<D> fr;
                fr.state = D::apply(parent.state, a);
                ++stats_.generated;
                if (fr.state == *shared_.goal) {
                    const std::int64_t cost = parent.g + 1;
                    if (cost <= bound_) {
                        std::vector<typename D::Action> full = w.seed->init_history;
                        full.insert(full.end(), w.path.begin(), w.path.end());
                        full.push_back(a);
                        shared_.offer_solution(cost, full);
                    } else {
                        collector_.record(tid_, cost);
                    }
                    continue;
                }
                fr.g = parent.g + 1;
                fr.last = a;
                fr.slot = w.slot_at(w.stack.size());
                kids_[nk] = fr.state;
                kid_slots_[nk++] = fr.slot;
                w.stack.push_back(fr);
                ++live_;
            }
            group_.submit_states_slots(tid_, kids_.data(), kid_slots_.data(), nk);
            if (live_ > stats_.peak_live_frames)
                stats_.peak_live_frames = live_;
            return StepStatus::Progress;
        }
    }

    void flush_expanded() {
        if (unflushed_expanded_) {
            shared_.expanded.fetch_add(unflushed_expanded_, std::memory_order_relaxed);
            unflushed_expanded_ = 0;
        }
    }

    // Frames still waiting on the evaluator when the round stops: wait for
    // their slots (the arenas must outlive every write into them).
    void drain(std::vector<FastWork<D>> &slots) {
        for (;;) {
            bool pending = false;
            for (auto &w : slots)
                for (auto &fr : w.stack)
                    if (fr.slot && fr.slot->value.load(std::memory_order_acquire) < 0)
                        pending = true;
            if (!pending)
                return;
            group_.kick_all();
            std::this_thread::yield();
        }
    }

private:

    int tid_;
    std::int64_t bound_;
    EvaluatorGroup<D> &group_;
    BoundCollector &collector_;
    IterationShared<D> &shared_;
    SearchStats &stats_;
    const ExpandHook<D> *on_expand_;
    std::array<typename D::State, D::kMaxBranching> kids_;  // one expansion's children (submit_states_slots)
    std::array<TicketSlot *, D::kMaxBranching> kid_slots_{};
    std::uint64_t live_ = 0;
    std::uint64_t unflushed_expanded_ = 0;
};

} // namespace fast_cbdfs

// cb_dfs (cbdfs.hpp:337-415): round-robin over work_num subtrees, refill from
// the queue, all-blocked kick, budget and deadline checks once per cycle.
template <class D>
void cb_dfs(int tid, int work_num, std::int64_t bound, WorkQueue<D> &queue, EvaluatorGroup<D> &group,
            BoundCollector &collector, IterationShared<D> &shared, SearchStats &stats,
            const ExpandHook<D> *on_expand = nullptr) {
    fast_cbdfs::Searcher<D> srch(tid, bound, group, collector, shared, stats, on_expand);
    std::vector<fast_cbdfs::FastWork<D>> slots(static_cast<std::size_t>(work_num));
    std::vector<char> terminated(static_cast<std::size_t>(work_num), 0);
    int miss = 0;

    shared.running.fetch_add(1, std::memory_order_acq_rel);

    for (int i = 0; i < work_num; ++i) {
        const WorkSeed<D> *seed = queue.pop();
        if (seed) {
            srch.push_root(slots[static_cast<std::size_t>(i)], seed);
        } else {
            terminated[static_cast<std::size_t>(i)] = 1;
            ++miss;
        }
    }

    int counter = 0;
    int blocked_in_cycle = 0;
    int idle_cycles = 0;
    while (miss < work_num && !shared.stop.load(std::memory_order_acquire)) {
        if (!terminated[static_cast<std::size_t>(counter)]) {
            fast_cbdfs::FastWork<D> &w = slots[static_cast<std::size_t>(counter)];
            if (w.done()) {
                const WorkSeed<D> *seed = queue.pop();
                if (seed) {
                    srch.push_root(w, seed);
                } else {
                    terminated[static_cast<std::size_t>(counter)] = 1;
                    ++miss;
                }
            }
            if (!terminated[static_cast<std::size_t>(counter)]) {
                if (srch.step(w) == StepStatus::Blocked)
                    ++blocked_in_cycle;
            }
        }
        ++counter;
        if (counter == work_num) {
            counter = 0;
            srch.flush_expanded();
            const int active = work_num - miss;
            if (active > 0 && blocked_in_cycle >= active) {
                const int b = shared.blocked.fetch_add(1, std::memory_order_acq_rel) + 1;
                if (b >= shared.running.load(std::memory_order_acquire))
                    group.kick_all();
                // the reference sleeps 50 us after 64 idle cycles (cbdfs.hpp:392-395);
                // on a device round trip of ~20 us that sleep is the latency, so
                // the overlay only yields unless BIDA_SEARCH_IDLE_SLEEP_US says so
                if (++idle_cycles > 64 && fast_cbdfs::idle_sleep_us() > 0)
                    std::this_thread::sleep_for(std::chrono::microseconds(fast_cbdfs::idle_sleep_us()));
                else
                    std::this_thread::yield();
                shared.blocked.fetch_sub(1, std::memory_order_acq_rel);
            } else {
                idle_cycles = 0;
            }
            blocked_in_cycle = 0;

            if (shared.expansion_budget > 0 &&
                shared.expanded_base + shared.expanded.load(std::memory_order_relaxed) > shared.expansion_budget) {
                shared.budget_exhausted.store(true, std::memory_order_release);
                shared.stop.store(true, std::memory_order_release);
            }
            if (shared.has_deadline && std::chrono::steady_clock::now() >= shared.deadline) {
                shared.timed_out.store(true, std::memory_order_release);
                shared.stop.store(true, std::memory_order_release);
            }
        }
    }
    srch.flush_expanded();
    srch.drain(slots);

    shared.running.fetch_sub(1, std::memory_order_acq_rel);
}

} // namespace bida
