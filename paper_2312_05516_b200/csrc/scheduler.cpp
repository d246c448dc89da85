// Step planner (see scheduler.hpp).  Each function names the reference function whose
// behaviour it restates (/root/reference/proj/src/...).
#include "scheduler.hpp"

#include "pb_common.hpp"

#include <algorithm>
#include <cmath>
#include <memory>
#include <set>
#include <unordered_set>

namespace pb {

// ------------------------------------------------------------------ cost model
// cost_model.cpp:77-85
CostProfile synthetic_profile(double k_attn, double c_other, double per_token_other) {
    CostProfile p;
    p.c_other = c_other;
    p.per_token_other = per_token_other;
    for (int64_t len = 32; len <= 65536; len *= 2) p.anchors.emplace_back(len, k_attn * static_cast<double>(len));
    return p;
}

// cost_model.cpp:33-62: piecewise linear, origin ray below the first anchor, last slope above
double attention_cost(const CostProfile& p, int64_t l) {
    if (p.anchors.empty()) fail(PB_ERR_CONFIG, "cost profile has no anchors");
    if (l <= 0) return 0.0;
    const auto& a = p.anchors;
    if (l <= a.front().first)
        return a.front().second * static_cast<double>(l) / static_cast<double>(a.front().first);
    for (size_t i = 1; i < a.size(); ++i)
        if (l <= a[i].first) {
            const double frac = static_cast<double>(l - a[i - 1].first) / static_cast<double>(a[i].first - a[i - 1].first);
            return a[i - 1].second + frac * (a[i].second - a[i - 1].second);
        }
    const double slope = a.size() == 1 ? a.back().second / static_cast<double>(a.back().first)
                                       : (a.back().second - a[a.size() - 2].second) /
                                             static_cast<double>(a.back().first - a[a.size() - 2].first);
    return a.back().second + slope * static_cast<double>(l - a.back().first);
}

double chunk_cost(const CostProfile& p, int64_t l) { return attention_cost(p, l) + p.c_other; }

// ------------------------------------------------------------------ victim ranking
// eviction_policy.cpp:12-74.  Both orders are total (ties end on (conv, offset), unique per
// chunk), so a full sort picks exactly the reference's nth_element + sort prefix.
std::vector<int64_t> select_victims(Policy policy, const PagedKvCache& cache, const std::vector<int64_t>& cand,
                                    const CostProfile& profile, double now, int needed) {
    if (needed <= 0) return {};
    if (static_cast<int>(cand.size()) < needed)
        fail(PB_ERR_NOT_ENOUGH_EVICTABLE,
             "need " + std::to_string(needed) + " victims, only " + std::to_string(cand.size()) + " evictable");
    struct Key {
        double value, last;
        int64_t conv, start, id;
    };
    std::vector<Key> keys;
    keys.reserve(cand.size());
    for (int64_t id : cand) {
        const ChunkRec& r = cache.chunk(id);
        double v = 0.0;
        if (policy == Policy::Pensieve) {
            const double inactive = std::max(now - r.last_active, 1e-3); // kInactiveTimeFloor
            v = chunk_cost(profile, r.end()) / inactive;
        }
        keys.push_back({v, r.last_active, r.conv, r.start, id});
    }
    auto less = [policy](const Key& a, const Key& b) {
        if (policy == Policy::Pensieve && a.value != b.value) return a.value < b.value;
        if (a.last != b.last) return a.last < b.last;
        if (a.conv != b.conv) return a.conv < b.conv;
        return a.start < b.start;
    };
    std::partial_sort(keys.begin(), keys.begin() + needed, keys.end(), less);
    std::vector<int64_t> out;
    out.reserve(static_cast<size_t>(needed));
    for (int i = 0; i < needed; ++i) out.push_back(keys[static_cast<size_t>(i)].id);
    return out;
}

// ------------------------------------------------------------------ scheduler
Scheduler::Scheduler(PagedKvCache& cache, CostProfile profile, SchedParams params)
    : cache_(cache), profile_(std::move(profile)), params_(params) {
    if (params_.token_budget < 1) fail(PB_ERR_CONFIG, "token_budget must be positive");
    if (params_.swap_threshold < 0.0 || params_.swap_threshold > 1.0) fail(PB_ERR_CONFIG, "swap_threshold must lie in [0, 1]");
    if (params_.reserve_fraction < 0.0 || params_.reserve_fraction >= 1.0)
        fail(PB_ERR_CONFIG, "reserve_fraction must lie in [0, 1)");
}

void Scheduler::enqueue(Request r) { // scheduler.cpp:229-235
    if (r.prompt < 1 || r.output < 1) fail(PB_ERR_CONFIG, "requests need positive prompt and output lengths");
    history_.try_emplace(r.conv_id, 0);
    if (r.state != ReqState::Suspended) r.state = ReqState::Waiting;
    queue_.push_back(r);
}

void Scheduler::begin_step() {
    step_out_.clear();
    step_in_.clear();
    step_out_moves_.clear();
    step_in_moves_.clear();
    step_recompute_ = 0;
}

std::vector<int64_t> Scheduler::pinned(bool include_queue, int64_t also) const {
    std::set<int64_t> s;
    for (const auto& e : running_) s.insert(e.req.conv_id);
    if (include_queue)
        for (const auto& r : queue_) s.insert(r.conv_id);
    if (also >= 0) s.insert(also);
    return {s.begin(), s.end()};
}

// scheduler.cpp:71-104: host overflow drops the cheapest host incumbents first, then the
// leading victims themselves; the rest move to the host (their bytes must be copied)
void Scheduler::evict_device_chunks(std::vector<int64_t> victims, double now) {
    if (victims.empty()) return;
    if (cache_.host().capacity() == 0) {
        cache_.apply_evictions(victims, false);
        return;
    }
    const int deficit = static_cast<int>(victims.size()) - cache_.host().n_free();
    std::vector<int64_t> to_host = victims;
    if (deficit > 0) {
        const std::vector<int64_t> incumbents = cache_.collect(Loc::Host, pinned(true, -1));
        const int from_host = std::min<int>(deficit, static_cast<int>(incumbents.size()));
        if (from_host > 0)
            cache_.apply_evictions(select_victims(params_.policy, cache_, incumbents, profile_, now, from_host), false);
        const int shortfall = deficit - from_host;
        if (shortfall > 0) {
            std::vector<int64_t> dropping(to_host.begin(), to_host.begin() + shortfall);
            to_host.erase(to_host.begin(), to_host.begin() + shortfall);
            cache_.apply_evictions(dropping, false);
        }
    }
    if (!to_host.empty()) {
        const std::vector<SlotMove> mv = cache_.apply_evictions(to_host, true);
        step_out_.insert(step_out_.end(), to_host.begin(), to_host.end());
        step_out_moves_.insert(step_out_moves_.end(), mv.begin(), mv.end());
    }
}

// scheduler.cpp:106-123
std::vector<int64_t> Scheduler::maybe_swap_out(double now) {
    if (params_.swap_threshold <= 0.0) return {};
    const int target = static_cast<int>(std::ceil(params_.swap_threshold * static_cast<double>(cache_.device().capacity())));
    if (available() >= target) return {};
    int needed = target - available();
    const std::vector<int64_t> cand = cache_.collect(Loc::Device, pinned(true, -1));
    if (cand.empty()) return {};
    needed = std::min<int>(needed, static_cast<int>(cand.size()));
    std::vector<int64_t> victims = select_victims(params_.policy, cache_, cand, profile_, now, needed);
    evict_device_chunks(victims, now);
    return victims;
}

// scheduler.cpp:125-160: two passes (outside running+queued, then outside running+self)
bool Scheduler::make_room(int32_t min_available, double now, int64_t for_conv) {
    if (available() >= min_available) return true;
    for (int pass = 0; pass < 2; ++pass) {
        const std::vector<int64_t> cand =
            cache_.collect(Loc::Device, pass == 0 ? pinned(true, -1) : pinned(false, for_conv));
        const int take = std::min<int>(min_available - available(), static_cast<int>(cand.size()));
        if (take > 0) evict_device_chunks(select_victims(params_.policy, cache_, cand, profile_, now, take), now);
        if (pass == 0 && available() >= min_available) return true;
    }
    return available() >= min_available;
}

// scheduler.cpp:162-230: dropped segments, missing suffix and pending input become spans;
// touching spans merge
RequestPlan Scheduler::plan_request(const Request& r) const {
    RequestPlan plan;
    const int64_t conv = r.conv_id;
    std::vector<Segment> segs;
    int64_t cached = 0;
    if (cache_.has_conversation(conv)) segs = cache_.layout(conv, &cached);
    auto hit = history_.find(conv);
    const int64_t history = hit == history_.end() ? 0 : hit->second;
    const int64_t missing = std::max<int64_t>(0, history - cached);
    if (missing > 0 && hit == history_.end())
        fail(PB_ERR_TRACE_MISSING, "conversation " + std::to_string(conv) + " has no refetchable history");
    plan.pending_tokens = r.state == ReqState::Suspended ? 1 : r.prompt;
    plan.finish_bonus = (r.generated + 1 == r.output) ? 1 : 0;
    const int64_t ctx_before = cached + missing;
    std::vector<std::pair<int64_t, int64_t>> spans;
    for (const Segment& s : segs) {
        if (s.kind == Loc::Dropped) {
            spans.emplace_back(s.begin, s.end);
            plan.recompute_tokens += s.end - s.begin;
            plan.rematerialize.insert(plan.rematerialize.end(), s.chunks.begin(), s.chunks.end());
        } else if (s.kind == Loc::Host) {
            plan.host_hit += s.end - s.begin;
            plan.swap_in.insert(plan.swap_in.end(), s.chunks.begin(), s.chunks.end());
        } else {
            plan.device_hit += s.end - s.begin;
        }
    }
    if (missing > 0) {
        spans.emplace_back(cached, history);
        plan.recompute_tokens += missing;
    }
    spans.emplace_back(ctx_before, ctx_before + plan.pending_tokens);
    std::vector<std::pair<int64_t, int64_t>> merged;
    for (const auto& s : spans) {
        if (!merged.empty() && merged.back().second == s.first) merged.back().second = s.second;
        else merged.push_back(s);
    }
    for (const auto& [b, e] : merged) {
        Span sp;
        sp.req_id = r.req_id;
        sp.query_len = e - b;
        sp.context_len = e;
        sp.causal_offset = b;
        plan.spans.push_back(std::move(sp));
    }
    plan.input_tokens = plan.recompute_tokens + plan.pending_tokens;
    const int64_t add = missing + plan.pending_tokens + plan.finish_bonus;
    plan.append_slots = cache_.has_conversation(conv)
                            ? cache_.append_chunks_needed(conv, add)
                            : static_cast<int32_t>((add + cache_.page_tokens() - 1) / cache_.page_tokens());
    return plan;
}

// scheduler.cpp:232-258: rematerialize, restore (swap-in slots recorded), then allocate
void Scheduler::commit(Request r, RequestPlan plan, double now) {
    const int64_t conv = r.conv_id;
    if (!plan.rematerialize.empty()) cache_.rematerialize(plan.rematerialize);
    if (!plan.swap_in.empty()) {
        const std::vector<SlotMove> mv = cache_.restore(plan.swap_in);
        for (const auto& m : mv) step_in_.emplace_back(m.chunk, m.dst_slot);
        step_in_moves_.insert(step_in_moves_.end(), mv.begin(), mv.end());
    }
    const int64_t cached = cache_.has_conversation(conv) ? cache_.total_tokens(conv) : 0;
    auto hit = history_.find(conv);
    const int64_t missing = std::max<int64_t>(0, (hit == history_.end() ? 0 : hit->second) - cached);
    cache_.allocate(conv, missing + plan.pending_tokens + plan.finish_bonus, now);
    cache_.touch(conv, now);
    step_recompute_ += plan.recompute_tokens;
    recompute_total_ += static_cast<uint64_t>(plan.recompute_tokens);
    Running e;
    e.req = r;
    e.req.state = r.state == ReqState::Suspended ? ReqState::Generating : ReqState::Prefill;
    e.pending = true;
    e.plan = std::move(plan);
    running_.push_back(std::move(e));
}

// scheduler.cpp:260-290: FCFS, no skipping, token budget, strict reserve
std::vector<int64_t> Scheduler::admit(double now) {
    std::vector<int64_t> admitted;
    int64_t batch_tokens = 0;
    for (const auto& e : running_)
        if (!e.pending) batch_tokens += 1;
    while (!queue_.empty()) {
        const Request& head = queue_.front();
        RequestPlan plan = plan_request(head);
        if (batch_tokens + plan.input_tokens > params_.token_budget) break;
        const double reserve = params_.reserve_fraction * static_cast<double>(cache_.device().capacity());
        const int slots = plan.total_slots();
        auto fits = [&] { return static_cast<double>(available() - slots) > reserve; };
        if (!fits()) {
            const int min_avail = static_cast<int>(std::floor(reserve + static_cast<double>(slots))) + 1;
            if (!make_room(min_avail, now, head.conv_id)) break;
            if (!fits()) break;
        }
        Request r = queue_.front();
        queue_.pop_front();
        batch_tokens += plan.input_tokens;
        admitted.push_back(r.req_id);
        commit(std::move(r), std::move(plan), now);
    }
    return admitted;
}

// scheduler.cpp:292-334: youngest generating requests first, their device chunks swapped out
std::vector<int64_t> Scheduler::suspend_for_memory(int32_t deficit, double now) {
    std::vector<Request> suspended;
    while (available() < deficit) {
        int pick = -1;
        for (int i = 0; i < static_cast<int>(running_.size()); ++i) {
            const auto& e = running_[static_cast<size_t>(i)];
            if (e.pending || e.req.state != ReqState::Generating) continue;
            if (pick < 0) {
                pick = i;
                continue;
            }
            const auto& best = running_[static_cast<size_t>(pick)].req;
            if (e.req.arrival > best.arrival || (e.req.arrival == best.arrival && e.req.req_id > best.req_id)) pick = i;
        }
        if (pick < 0)
            fail(PB_ERR_CANNOT_SUSPEND_ALL,
                 "cannot free " + std::to_string(deficit) + " device slots: no suspendable requests remain");
        Running e = std::move(running_[static_cast<size_t>(pick)]);
        running_.erase(running_.begin() + pick);
        std::vector<int64_t> dev;
        for (int64_t id : cache_.conversation_chunks(e.req.conv_id))
            if (cache_.chunk(id).loc == Loc::Device) dev.push_back(id);
        evict_device_chunks(std::move(dev), now);
        e.req.state = ReqState::Suspended;
        suspended.push_back(e.req);
    }
    std::sort(suspended.begin(), suspended.end(), [](const Request& a, const Request& b) {
        if (a.arrival != b.arrival) return a.arrival < b.arrival;
        return a.req_id < b.req_id;
    });
    std::vector<int64_t> ids;
    for (const auto& r : suspended) ids.push_back(r.req_id);
    for (auto it = suspended.rbegin(); it != suspended.rend(); ++it) queue_.push_front(*it);
    return ids;
}

// scheduler.cpp:336-350
std::vector<int64_t> Scheduler::ensure_generation_capacity(double now) {
    std::vector<int64_t> all;
    for (;;) {
        int needed = 0;
        for (const auto& e : running_) {
            if (e.pending || e.req.state != ReqState::Generating) continue;
            const int64_t bonus = (e.req.generated + 1 == e.req.output) ? 1 : 0;
            needed += cache_.append_chunks_needed(e.req.conv_id, 1 + bonus);
        }
        if (available() >= needed) return all;
        std::vector<int64_t> b = suspend_for_memory(available() + 1, now);
        all.insert(all.end(), b.begin(), b.end());
    }
}

// scheduler.cpp:352-420: prefill spans (admitted this step) then decode spans; query_start
// prefix sums; unified = one plan, split = prefill plan + generation plan
std::vector<StepPlan> Scheduler::build_batch(double now) {
    std::vector<Span> prefill, gen;
    for (auto& e : running_) {
        if (!e.pending) continue;
        for (Span sp : e.plan.spans) {
            sp.table = cache_.block_table(e.req.conv_id, sp.context_len);
            prefill.push_back(std::move(sp));
        }
    }
    for (auto& e : running_) {
        if (e.pending || e.req.state != ReqState::Generating) continue;
        const int64_t bonus = (e.req.generated + 1 == e.req.output) ? 1 : 0;
        const int64_t before = cache_.total_tokens(e.req.conv_id);
        cache_.allocate(e.req.conv_id, 1 + bonus, now);
        Span sp;
        sp.req_id = e.req.req_id;
        sp.query_len = 1;
        sp.causal_offset = before;
        sp.context_len = before + 1;
        sp.table = cache_.block_table(e.req.conv_id, sp.context_len);
        gen.push_back(std::move(sp));
    }
    auto finalize = [](StepPlan& p) {
        int64_t cursor = 0;
        for (auto& sp : p.spans) {
            sp.query_start = cursor;
            cursor += sp.query_len;
        }
        p.total_input_tokens = cursor;
    };
    auto attach_swaps = [&](StepPlan& p) {
        p.swap_in = step_in_;
        p.swap_out = step_out_;
        p.in_moves = step_in_moves_;
        p.out_moves = step_out_moves_;
    };
    std::vector<StepPlan> plans;
    if (!params_.split_mode) {
        if (prefill.empty() && gen.empty()) return plans;
        StepPlan p;
        p.spans = std::move(prefill);
        p.spans.insert(p.spans.end(), std::make_move_iterator(gen.begin()), std::make_move_iterator(gen.end()));
        finalize(p);
        p.recompute_tokens = step_recompute_;
        attach_swaps(p);
        plans.push_back(std::move(p));
        return plans;
    }
    if (!prefill.empty()) {
        StepPlan p;
        p.spans = std::move(prefill);
        finalize(p);
        p.recompute_tokens = step_recompute_;
        plans.push_back(std::move(p));
    }
    if (!gen.empty()) {
        StepPlan p;
        p.spans = std::move(gen);
        finalize(p);
        plans.push_back(std::move(p));
    }
    if (!plans.empty()) attach_swaps(plans.front());
    return plans;
}

void Scheduler::retire(Running& e, double end_time) { // scheduler.cpp:603-612
    e.req.completion = end_time;
    e.req.state = ReqState::Finished;
    if (params_.stateful) cache_.touch(e.req.conv_id, end_time);
    else cache_.release_conversation(e.req.conv_id);
    history_[e.req.conv_id] += e.req.prompt + e.req.output;
}

// scheduler.cpp:614-638
void Scheduler::complete_plan(const StepPlan& plan, double end_time, std::vector<Request>& finished) {
    std::vector<int64_t> order;
    std::unordered_set<int64_t> seen;
    for (const auto& sp : plan.spans)
        if (seen.insert(sp.req_id).second) order.push_back(sp.req_id);
    for (int64_t id : order) {
        auto it = std::find_if(running_.begin(), running_.end(), [&](const Running& e) { return e.req.req_id == id; });
        if (it == running_.end()) fail(PB_ERR_ERROR, "completed plan references unknown request " + std::to_string(id));
        it->pending = false;
        it->req.generated += 1;
        if (it->req.first_token < 0.0) it->req.first_token = end_time;
        if (it->req.state == ReqState::Prefill) it->req.state = ReqState::Generating;
        if (it->req.generated >= it->req.output) {
            retire(*it, end_time);
            finished.push_back(it->req);
            running_.erase(it);
        }
    }
}

} // namespace pb

// ====================================================================== C-ABI
using namespace pb;

struct pb_scheduler {
    std::unique_ptr<Scheduler> s;
    std::vector<StepPlan> plans;
};

namespace {
SchedParams to_params(const pb_sched_params* p) {
    SchedParams q;
    if (p) {
        q.split_mode = p->split_mode != 0;
        q.policy = p->policy == 1 ? Policy::Lru : Policy::Pensieve;
        q.stateful = p->stateful != 0;
        q.token_budget = p->token_budget;
        q.swap_threshold = p->swap_threshold;
        q.reserve_fraction = p->reserve_fraction;
    }
    return q;
}
const StepPlan& plan_at(const pb_scheduler* S, int32_t i) {
    if (!S || i < 0 || i >= static_cast<int32_t>(S->plans.size())) fail(PB_ERR_DIMENSION_MISMATCH, "no such plan");
    return S->plans[static_cast<size_t>(i)];
}
} // namespace

extern "C" {

void pb_sched_default_params(pb_sched_params* p) {
    SchedParams d;
    p->split_mode = 0;
    p->policy = 0;
    p->stateful = 1;
    p->token_budget = d.token_budget;
    p->swap_threshold = d.swap_threshold;
    p->reserve_fraction = d.reserve_fraction;
}

pb_status pb_sched_create(pb_kv_cache* cache, const int64_t* anchor_len, const double* anchor_sec, int32_t n_anchors,
                          double c_other, double per_token_other, const pb_sched_params* params, pb_scheduler** out) {
    return guarded([&] {
        if (!cache || !out) fail(PB_ERR_ERROR, "null argument");
        CostProfile prof;
        for (int32_t i = 0; i < n_anchors; ++i) prof.anchors.emplace_back(anchor_len[i], anchor_sec[i]);
        prof.c_other = c_other;
        prof.per_token_other = per_token_other;
        if (prof.anchors.empty()) fail(PB_ERR_CONFIG, "cost profile has no anchors");
        auto S = std::make_unique<pb_scheduler>();
        S->s = std::make_unique<Scheduler>(pb_cache_impl(cache), std::move(prof), to_params(params));
        *out = S.release();
    });
}

pb_status pb_sched_create_synthetic(pb_kv_cache* cache, double k_attn, double c_other, double per_token_other,
                                    const pb_sched_params* params, pb_scheduler** out) {
    const CostProfile p = synthetic_profile(k_attn, c_other, per_token_other);
    std::vector<int64_t> len;
    std::vector<double> sec;
    for (const auto& a : p.anchors) {
        len.push_back(a.first);
        sec.push_back(a.second);
    }
    return pb_sched_create(cache, len.data(), sec.data(), static_cast<int32_t>(len.size()), c_other,
                           per_token_other, params, out);
}

void pb_sched_destroy(pb_scheduler* S) { delete S; }

pb_status pb_sched_enqueue(pb_scheduler* S, int64_t req_id, int64_t conv_id, int32_t turn, double arrival,
                           int64_t prompt, int64_t output) {
    return guarded([&] {
        Request r;
        r.req_id = req_id;
        r.conv_id = conv_id;
        r.turn = turn;
        r.arrival = arrival;
        r.prompt = prompt;
        r.output = output;
        S->s->enqueue(r);
    });
}

pb_status pb_sched_append_history(pb_scheduler* S, int64_t conv, int64_t tokens) {
    return guarded([&] { S->s->append_history(conv, tokens); });
}

pb_status pb_sched_step(pb_scheduler* S, double now, int32_t* n_plans) {
    return guarded([&] {
        S->s->begin_step();
        S->s->maybe_swap_out(now);
        S->s->admit(now);
        S->s->ensure_generation_capacity(now);
        S->plans = S->s->build_batch(now);
        if (n_plans) *n_plans = static_cast<int32_t>(S->plans.size());
    });
}

pb_status pb_sched_plan_info(const pb_scheduler* S, int32_t plan, int64_t* info8) {
    return guarded([&] {
        const StepPlan& p = plan_at(S, plan);
        int64_t n_bt = 0;
        for (const auto& sp : p.spans) n_bt += static_cast<int64_t>(sp.table.size());
        info8[0] = static_cast<int64_t>(p.spans.size());
        info8[1] = p.total_input_tokens;
        info8[2] = n_bt;
        info8[3] = static_cast<int64_t>(p.swap_in.size());
        info8[4] = static_cast<int64_t>(p.swap_out.size());
        info8[5] = p.recompute_tokens;
        info8[6] = static_cast<int64_t>(p.in_moves.size());
        info8[7] = static_cast<int64_t>(p.out_moves.size());
    });
}

pb_status pb_sched_plan_spans(const pb_scheduler* S, int32_t plan, int64_t* req_id, int64_t* query_start,
                              int64_t* query_len, int64_t* context_len, int64_t* causal_offset, int32_t* block_tables,
                              int64_t* bt_offsets) {
    return guarded([&] {
        const StepPlan& p = plan_at(S, plan);
        int64_t off = 0;
        for (size_t i = 0; i < p.spans.size(); ++i) {
            const Span& sp = p.spans[i];
            req_id[i] = sp.req_id;
            query_start[i] = sp.query_start;
            query_len[i] = sp.query_len;
            context_len[i] = sp.context_len;
            causal_offset[i] = sp.causal_offset;
            bt_offsets[i] = off;
            for (int32_t s : sp.table) block_tables[off++] = s;
        }
        bt_offsets[p.spans.size()] = off;
    });
}

pb_status pb_sched_plan_moves(const pb_scheduler* S, int32_t plan, pb_slot_move* in_moves, pb_slot_move* out_moves) {
    return guarded([&] {
        const StepPlan& p = plan_at(S, plan);
        for (size_t i = 0; i < p.in_moves.size(); ++i)
            in_moves[i] = {p.in_moves[i].chunk, p.in_moves[i].src_slot, p.in_moves[i].dst_slot};
        for (size_t i = 0; i < p.out_moves.size(); ++i)
            out_moves[i] = {p.out_moves[i].chunk, p.out_moves[i].src_slot, p.out_moves[i].dst_slot};
    });
}

pb_status pb_sched_complete(pb_scheduler* S, int32_t plan, double end_time, int64_t* finished, int64_t cap,
                            int64_t* n_finished) {
    return guarded([&] {
        std::vector<Request> done;
        S->s->complete_plan(plan_at(S, plan), end_time, done);
        if (n_finished) *n_finished = static_cast<int64_t>(done.size());
        for (size_t i = 0; finished && i < done.size() && static_cast<int64_t>(i) < cap; ++i) finished[i] = done[i].req_id;
    });
}

pb_status pb_sched_plan_request(const pb_scheduler* S, int64_t req_id, int64_t conv_id, int64_t prompt, int64_t output,
                                int64_t generated, int32_t suspended, int64_t* info8, int64_t* span3, int64_t cap) {
    return guarded([&] {
        Request r;
        r.req_id = req_id;
        r.conv_id = conv_id;
        r.prompt = prompt;
        r.output = output;
        r.generated = generated;
        r.state = suspended ? ReqState::Suspended : ReqState::Waiting;
        const RequestPlan p = S->s->plan_request(r);
        info8[0] = p.input_tokens;
        info8[1] = p.recompute_tokens;
        info8[2] = p.pending_tokens;
        info8[3] = static_cast<int64_t>(p.rematerialize.size());
        info8[4] = static_cast<int64_t>(p.swap_in.size());
        info8[5] = p.append_slots;
        info8[6] = p.device_hit;
        info8[7] = p.host_hit;
        for (size_t i = 0; i < p.spans.size() && static_cast<int64_t>(i) < cap; ++i) {
            span3[3 * i + 0] = p.spans[i].query_len;
            span3[3 * i + 1] = p.spans[i].context_len;
            span3[3 * i + 2] = p.spans[i].causal_offset;
        }
        info8[8] = static_cast<int64_t>(p.spans.size());
    });
}

int64_t pb_sched_queue_size(const pb_scheduler* S) { return static_cast<int64_t>(S->s->queue_size()); }
int64_t pb_sched_running_size(const pb_scheduler* S) { return static_cast<int64_t>(S->s->running_size()); }

} // extern "C"
