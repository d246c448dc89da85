// Device-timestamped event log of the swap / attention pipeline, and the reference's
// LayerDependencyAuditor restated over it (/root/reference/proj/src/event_log.cpp:90-118;
// EventKind order of include/kvsim/event_log.hpp:14).  The reference logs simulated times;
// here every event is a %globaltimer stamp written by a one-thread kernel enqueued on the
// stream whose progress it marks, so "attention of layer l started" can only be stamped
// after everything that stream waited on, and the audit checks real GPU ordering.
#include "pb_common.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <numeric>
#include <vector>

namespace pb {
namespace {

__global__ void stamp_kernel(pb_event_record* recs, unsigned long long* count, int64_t cap, int32_t kind,
                             int32_t layer, int64_t req) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned long long i = atomicAdd(count, 1ull);
    if (static_cast<int64_t>(i) < cap) {
        pb_event_record r;
        r.t_ns = static_cast<int64_t>(t);
        r.kind = kind;
        r.layer = layer;
        r.req = req;
        recs[i] = r;
    }
}

} // namespace
} // namespace pb

using namespace pb;

struct pb_event_log {
    pb_event_record* recs = nullptr;
    unsigned long long* count = nullptr;
    int64_t cap = 0;
};

extern "C" {

pb_status pb_evlog_create(int64_t capacity, pb_event_log** out) {
    return guarded([&] {
        if (!out) fail(PB_ERR_ERROR, "null out");
        *out = nullptr;
        if (capacity < 1) fail(PB_ERR_CONFIG, "event log capacity must be >= 1");
        auto L = std::make_unique<pb_event_log>();
        L->cap = capacity;
        cuda_check(cudaMalloc(&L->recs, sizeof(pb_event_record) * static_cast<size_t>(capacity)), "cudaMalloc(log)");
        cuda_check(cudaMalloc(&L->count, sizeof(unsigned long long)), "cudaMalloc(log count)");
        cuda_check(cudaMemset(L->count, 0, sizeof(unsigned long long)), "log reset");
        *out = L.release();
    });
}

void pb_evlog_destroy(pb_event_log* L) {
    if (!L) return;
    cudaFree(L->recs);
    cudaFree(L->count);
    delete L;
}

pb_status pb_evlog_mark(pb_event_log* L, int32_t kind, int32_t layer, int64_t req, void* stream) {
    return guarded([&] {
        if (!L) fail(PB_ERR_ERROR, "null log");
        if (kind < PB_EV_SWAP_IN_LAYER || kind > PB_EV_STEP_END) fail(PB_ERR_ERROR, "unknown event kind");
        stamp_kernel<<<1, 1, 0, as_stream(stream)>>>(L->recs, L->count, L->cap, kind, layer, req);
        cuda_check(cudaGetLastError(), "event stamp");
        count_launch();
    });
}

pb_status pb_evlog_read(pb_event_log* L, pb_event_record* out, int64_t cap, int64_t* n) {
    return guarded([&] {
        if (!L || !n) fail(PB_ERR_ERROR, "null argument");
        cuda_check(cudaDeviceSynchronize(), "log sync");
        unsigned long long c = 0;
        cuda_check(cudaMemcpy(&c, L->count, sizeof(c), cudaMemcpyDeviceToHost), "log count");
        const int64_t have = std::min<int64_t>(static_cast<int64_t>(c), L->cap);
        if (have > L->cap || static_cast<int64_t>(c) > L->cap) fail(PB_ERR_ERROR, "event log overflowed its capacity");
        *n = have;
        if (out && cap > 0)
            cuda_check(cudaMemcpy(out, L->recs, sizeof(pb_event_record) * static_cast<size_t>(std::min(cap, have)),
                                  cudaMemcpyDeviceToHost),
                       "log copy");
    });
}

pb_status pb_evlog_reset(pb_event_log* L) {
    return guarded([&] {
        if (!L) fail(PB_ERR_ERROR, "null log");
        cuda_check(cudaMemset(L->count, 0, sizeof(unsigned long long)), "log reset");
    });
}

// LayerDependencyAuditor::on_event (src/event_log.cpp:90-118) over the events in log order
// (a device log is in stamp order): within a step, an attention start of layer l more than
// 1 ns (the reference's 1e-9 s) before the latest swap-in completion of layer l is a
// violation; a swap-in with layer < 0 is one too.
pb_status pb_evlog_audit(const pb_event_record* ev, int64_t n, uint64_t* violations, uint64_t* steps) {
    return guarded([&] {
        if ((!ev && n > 0) || !violations || !steps) fail(PB_ERR_ERROR, "null argument");
        std::vector<int64_t> ready;
        uint64_t v = 0, st = 0;
        for (int64_t i = 0; i < n; ++i) { // log order, as the reference's streaming sink
            const pb_event_record& e = ev[i];
            switch (e.kind) {
                case PB_EV_SWAP_IN_LAYER:
                    if (e.layer < 0) {
                        ++v;
                        break;
                    }
                    if (static_cast<size_t>(e.layer) >= ready.size()) ready.resize(static_cast<size_t>(e.layer) + 1, -1);
                    ready[static_cast<size_t>(e.layer)] = std::max(ready[static_cast<size_t>(e.layer)], e.t_ns);
                    break;
                case PB_EV_ATTN_START:
                    if (e.layer >= 0 && static_cast<size_t>(e.layer) < ready.size()) {
                        const int64_t r = ready[static_cast<size_t>(e.layer)];
                        if (r >= 0 && e.t_ns < r - 1) ++v;
                    }
                    break;
                case PB_EV_STEP_END:
                    ready.clear();
                    ++st;
                    break;
                default:
                    break;
            }
        }
        *violations = v;
        *steps = st;
    });
}

// The same rule per step instead of streaming: the events between two STEP_ENDs (in log
// order) form a step; a layer's readiness is the latest SWAP_IN_LAYER of that layer anywhere
// in the step, and every ATTN_START of the layer in the step must be at or after it (1 ns
// tolerance).  On a device-stamped log (stamp order = time order) the streaming auditor can
// only see an attention that was stamped before its swap-in as "not yet ready"; this form
// flags it.
pb_status pb_evlog_audit_steps(const pb_event_record* ev, int64_t n, uint64_t* violations, uint64_t* steps) {
    return guarded([&] {
        if ((!ev && n > 0) || !violations || !steps) fail(PB_ERR_ERROR, "null argument");
        uint64_t v = 0, st = 0;
        int64_t begin = 0;
        std::vector<int64_t> ready;
        for (int64_t end = 0; end <= n; ++end) {
            if (end < n && ev[end].kind != PB_EV_STEP_END) continue;
            ready.clear();
            for (int64_t i = begin; i < end; ++i) {
                const pb_event_record& e = ev[i];
                if (e.kind != PB_EV_SWAP_IN_LAYER) continue;
                if (e.layer < 0) {
                    ++v;
                    continue;
                }
                if (static_cast<size_t>(e.layer) >= ready.size()) ready.resize(static_cast<size_t>(e.layer) + 1, -1);
                ready[static_cast<size_t>(e.layer)] = std::max(ready[static_cast<size_t>(e.layer)], e.t_ns);
            }
            for (int64_t i = begin; i < end; ++i) {
                const pb_event_record& e = ev[i];
                if (e.kind != PB_EV_ATTN_START || e.layer < 0 || static_cast<size_t>(e.layer) >= ready.size()) continue;
                const int64_t r = ready[static_cast<size_t>(e.layer)];
                if (r >= 0 && e.t_ns < r - 1) ++v;
            }
            if (end < n) ++st;
            begin = end + 1;
        }
        *violations = v;
        *steps = st;
    });
}

} // extern "C"
