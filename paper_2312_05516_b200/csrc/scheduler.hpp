// Host-side step planner: turns queued conversation turns into the ragged batch the attention
// kernels consume (spans + block tables) and the slot moves the swap engine executes.
//
// Restates the observable behaviour of the reference Scheduler
// (/root/reference/proj/include/kvsim/scheduler.hpp:88-179, src/scheduler.cpp) — FCFS
// admission with reserve, prefix-drop span construction (plan_request :162-230), the
// rematerialize -> restore -> allocate order (commit_admission :232-258), ahead-of-time
// eviction with host-overflow drops (:71-123), make_room (:125-160), suspension (:292-350)
// and batch assembly (build_batch :352-420) — so spans and block tables are bit-identical,
// and adds what a device needs: the (chunk, src slot, dst slot) triples of every swap.
// Victim ranking (EvictionPolicy, src/eviction_policy.cpp) and the piecewise-linear cost
// model behind it (src/cost_model.cpp:33-66) are restated because they decide which slots
// move; neither is on the device path.
#pragma once

#include "kv_cache.hpp"

#include <cstdint>
#include <deque>
#include <utility>
#include <vector>

namespace pb {

struct CostProfile {
    std::vector<std::pair<int64_t, double>> anchors; // (context_len, seconds per 32-token chunk)
    double c_other = 0.0;
    double per_token_other = 0.0;
};
CostProfile synthetic_profile(double k_attn, double c_other, double per_token_other);
double attention_cost(const CostProfile& p, int64_t context_len);
double chunk_cost(const CostProfile& p, int64_t context_len);

enum class Policy : int { Pensieve = 0, Lru = 1 };
// `needed` victims in eviction order (ascending retention value / oldest first); throws
// PB_ERR_NOT_ENOUGH_EVICTABLE when fewer candidates exist.
std::vector<int64_t> select_victims(Policy policy, const PagedKvCache& cache, const std::vector<int64_t>& candidates,
                                    const CostProfile& profile, double now, int needed);

enum class ReqState : int { Waiting = 0, Prefill = 1, Generating = 2, Suspended = 3, Finished = 4 };

struct Request {
    int64_t req_id = -1, conv_id = -1;
    int32_t turn = 0;
    double arrival = 0.0;
    int64_t prompt = 0, output = 0;
    ReqState state = ReqState::Waiting;
    int64_t generated = 0;
    double first_token = -1.0, completion = -1.0;
};

struct Span { // SubRequest, include/kvsim/batch.hpp:17-24
    int64_t req_id = -1, query_start = 0, query_len = 0, context_len = 0, causal_offset = 0;
    std::vector<int32_t> table;
};

struct RequestPlan {
    int64_t input_tokens = 0, recompute_tokens = 0, pending_tokens = 0, finish_bonus = 0;
    std::vector<int64_t> rematerialize, swap_in;
    int32_t append_slots = 0;
    int64_t device_hit = 0, host_hit = 0;
    std::vector<Span> spans; // tables filled at build time
    int32_t total_slots() const {
        return static_cast<int32_t>(rematerialize.size() + swap_in.size()) + append_slots;
    }
};

struct StepPlan { // BatchPlan, include/kvsim/batch.hpp:28-34, plus slot pairs
    std::vector<Span> spans;
    std::vector<std::pair<int64_t, int32_t>> swap_in; // chunk -> device slot
    std::vector<int64_t> swap_out;                     // chunks headed to the host
    std::vector<SlotMove> in_moves;                    // host src -> device dst
    std::vector<SlotMove> out_moves;                   // device src -> host dst
    int64_t recompute_tokens = 0, total_input_tokens = 0;
};

struct SchedParams {
    bool split_mode = false; // false: unified prefill+decode batch
    Policy policy = Policy::Pensieve;
    bool stateful = true;
    int64_t token_budget = 4096;
    double swap_threshold = 0.25;
    double reserve_fraction = 0.10;
};

class Scheduler {
public:
    Scheduler(PagedKvCache& cache, CostProfile profile, SchedParams params);

    void enqueue(Request r);
    void begin_step();
    std::vector<int64_t> maybe_swap_out(double now);
    std::vector<int64_t> admit(double now);
    RequestPlan plan_request(const Request& r) const;
    std::vector<int64_t> suspend_for_memory(int32_t deficit_slots, double now);
    std::vector<int64_t> ensure_generation_capacity(double now);
    std::vector<StepPlan> build_batch(double now);
    void complete_plan(const StepPlan& plan, double end_time, std::vector<Request>& finished);

    size_t queue_size() const { return queue_.size(); }
    size_t running_size() const { return running_.size(); }
    void append_history(int64_t conv, int64_t tokens) { history_[conv] += tokens; }
    void ensure_conv(int64_t conv) { history_.try_emplace(conv, 0); }
    uint64_t recompute_total() const { return recompute_total_; }

private:
    struct Running {
        Request req;
        bool pending = false;
        RequestPlan plan;
    };
    std::vector<int64_t> pinned(bool include_queue, int64_t also) const;
    bool make_room(int32_t min_available, double now, int64_t for_conv);
    void evict_device_chunks(std::vector<int64_t> victims, double now);
    void commit(Request r, RequestPlan plan, double now);
    void retire(Running& e, double end_time);
    int32_t available() const { return cache_.device().available(); }

    PagedKvCache& cache_;
    CostProfile profile_;
    SchedParams params_;
    std::map<int64_t, int64_t> history_; // completed-turn text length per conversation
    std::deque<Request> queue_;
    std::vector<Running> running_;
    std::vector<int64_t> step_out_;
    std::vector<std::pair<int64_t, int32_t>> step_in_;
    std::vector<SlotMove> step_out_moves_, step_in_moves_;
    int64_t step_recompute_ = 0;
    uint64_t recompute_total_ = 0;
};

} // namespace pb
