// TEST INFRASTRUCTURE ONLY — extern "C" access to the UNMODIFIED reference Scheduler
// (/root/reference/proj/src/scheduler.cpp) for the differential tests of the product's
// step planner (tests/test_scheduler.py).  Built into oracle/_ref/libkvsim_ref.so.
#include "kvsim/errors.hpp"
#include "kvsim/scheduler.hpp"

#include <cstdint>
#include <memory>
#include <vector>

using namespace kvsim;

namespace {

struct RefSched {
    std::unique_ptr<PagedKvCache> cache;
    CostProfile profile;
    ConversationRegistry registry;
    std::unique_ptr<Scheduler> sched;
    std::vector<BatchPlan> plans;
};

template <class F> int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const DimensionMismatch&) {
        return 1;
    } catch (const NumericError&) {
        return 2;
    } catch (const InsufficientDeviceMemory&) {
        return 4;
    } catch (const InsufficientHostMemory&) {
        return 5;
    } catch (const InvalidChunkState&) {
        return 6;
    } catch (const UnknownConversation&) {
        return 7;
    } catch (const ConfigError&) {
        return 8;
    } catch (const NotEnoughEvictable&) {
        return 9;
    } catch (const TraceMissing&) {
        return 10;
    } catch (const CannotSuspendAll&) {
        return 11;
    } catch (const Error&) {
        return 3;
    }
}

} // namespace

extern "C" {

void* ref_sched_create(int chunk, int dev_slots, int host_slots, double k_attn, double c_other, double per_token,
                       int split, int lru, int stateful, long long token_budget, double swap_threshold,
                       double reserve) {
    auto* r = new RefSched;
    r->cache = std::make_unique<PagedKvCache>(chunk, dev_slots, host_slots);
    r->profile = synthetic_profile(k_attn, c_other, per_token);
    SchedulerParams p;
    p.mode = split ? BatchMode::Split : BatchMode::Unified;
    p.policy = lru ? PolicyKind::Lru : PolicyKind::Pensieve;
    p.stateful = stateful != 0;
    p.token_budget = token_budget;
    p.swap_threshold = swap_threshold;
    p.reserve_fraction = reserve;
    r->sched = std::make_unique<Scheduler>(*r->cache, r->profile, r->registry, p);
    return r;
}

void ref_sched_destroy(void* h) { delete static_cast<RefSched*>(h); }

int ref_sched_enqueue(void* h, long long req, long long conv, int turn, double arrival, long long prompt,
                      long long output) {
    auto* r = static_cast<RefSched*>(h);
    return guarded([&] {
        Request q;
        q.req_id = req;
        q.conv_id = conv;
        q.turn_index = turn;
        q.arrival_time = arrival;
        q.prompt_tokens = prompt;
        q.output_tokens = output;
        r->sched->enqueue(q);
    });
}

int ref_sched_step(void* h, double now, int* n_plans) {
    auto* r = static_cast<RefSched*>(h);
    return guarded([&] {
        r->sched->begin_step();
        r->sched->maybe_swap_out(now);
        r->sched->admit(now);
        r->sched->ensure_generation_capacity(now);
        r->plans = r->sched->build_batch(now);
        *n_plans = static_cast<int>(r->plans.size());
    });
}

// info[6]: n_spans, total tokens, block-table entries, swap_in, swap_out, recompute tokens
int ref_sched_plan_info(void* h, int plan, long long* info) {
    auto* r = static_cast<RefSched*>(h);
    const BatchPlan& p = r->plans.at(static_cast<size_t>(plan));
    long long bt = 0;
    for (const auto& s : p.sub_requests) bt += static_cast<long long>(s.block_table.size());
    info[0] = static_cast<long long>(p.sub_requests.size());
    info[1] = p.total_input_tokens;
    info[2] = bt;
    info[3] = static_cast<long long>(p.swap_in.size());
    info[4] = static_cast<long long>(p.swap_out.size());
    info[5] = p.recompute_token_count;
    return 0;
}

int ref_sched_plan_spans(void* h, int plan, long long* req, long long* qs, long long* ql, long long* cl,
                         long long* co, int* bt, long long* bt_off, long long* swap_in_chunk, int* swap_in_slot,
                         long long* swap_out) {
    auto* r = static_cast<RefSched*>(h);
    const BatchPlan& p = r->plans.at(static_cast<size_t>(plan));
    long long off = 0;
    for (size_t i = 0; i < p.sub_requests.size(); ++i) {
        const auto& s = p.sub_requests[i];
        req[i] = s.req_id;
        qs[i] = s.query_start;
        ql[i] = s.query_len;
        cl[i] = s.context_len;
        co[i] = s.causal_offset;
        bt_off[i] = off;
        for (int x : s.block_table) bt[off++] = x;
    }
    bt_off[p.sub_requests.size()] = off;
    for (size_t i = 0; i < p.swap_in.size(); ++i) {
        swap_in_chunk[i] = p.swap_in[i].first;
        swap_in_slot[i] = p.swap_in[i].second;
    }
    for (size_t i = 0; i < p.swap_out.size(); ++i) swap_out[i] = p.swap_out[i];
    return 0;
}

int ref_sched_complete(void* h, int plan, double end_time, long long* finished, long long cap, long long* n) {
    auto* r = static_cast<RefSched*>(h);
    return guarded([&] {
        std::vector<Request> done;
        r->sched->complete_plan(r->plans.at(static_cast<size_t>(plan)), end_time, done);
        *n = static_cast<long long>(done.size());
        for (size_t i = 0; i < done.size() && static_cast<long long>(i) < cap; ++i) finished[i] = done[i].req_id;
    });
}

long long ref_sched_queue_size(void* h) { return static_cast<long long>(static_cast<RefSched*>(h)->sched->queue_size()); }
long long ref_sched_running_size(void* h) {
    return static_cast<long long>(static_cast<RefSched*>(h)->sched->running_size());
}

int ref_sched_dump(void* h, char* buf, long long cap) {
    auto* r = static_cast<RefSched*>(h);
    std::string s = r->cache->dump();
    size_t n = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
    std::copy(s.data(), s.data() + n, buf);
    buf[n] = '\0';
    return static_cast<int>(s.size());
}

} // extern "C"
