// TEST INFRASTRUCTURE ONLY — extern "C" shim over the UNMODIFIED reference library.
//
// oracle/Makefile compiles this file together with the reference sources where they lie
// (/root/reference/proj/src/*.cpp, read-only) into oracle/_ref/libkvsim_ref.so.  Tests use
// it to pin the oracle restatement (oracle/attn_oracle.c) and the product's host
// bookkeeping against the real reference; bench.py's cpu_baseline / --impl reference leg
// times the reference's own paged_multi_token_attention through it.  No reference code is
// copied: this file only marshals plain arrays into the reference's own types and maps its
// exception classes (proj/include/kvsim/errors.hpp) onto PB_* status codes.
#include "kvsim/attention.hpp"
#include "kvsim/event_log.hpp"
#include "kvsim/errors.hpp"
#include "kvsim/model_config.hpp"
#include "kvsim/paged_kv_cache.hpp"
#include "kvsim/swap_engine.hpp"
#include "kvsim/workload.hpp"

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

using namespace kvsim;

namespace {

// Mirrors include/pensieve_b200.h PB_* codes.
enum : int {
    kOk = 0,
    kDimensionMismatch = 1,
    kNumeric = 2,
    kError = 3,
    kInsufficientDevice = 4,
    kInsufficientHost = 5,
    kInvalidChunkState = 6,
    kUnknownConversation = 7,
    kConfig = 8,
    kNotEnoughEvictable = 9,
};

template <class F> int guarded(F&& f) {
    try {
        f();
        return kOk;
    } catch (const DimensionMismatch&) {
        return kDimensionMismatch;
    } catch (const NumericError&) {
        return kNumeric;
    } catch (const InsufficientDeviceMemory&) {
        return kInsufficientDevice;
    } catch (const InsufficientHostMemory&) {
        return kInsufficientHost;
    } catch (const InvalidChunkState&) {
        return kInvalidChunkState;
    } catch (const UnknownConversation&) {
        return kUnknownConversation;
    } catch (const ConfigError&) {
        return kConfig;
    } catch (const NotEnoughEvictable&) {
        return kNotEnoughEvictable;
    } catch (const Error&) {
        return kError;
    }
}

RaggedQueryBatch make_batch(int n_head, int head_size, double scale, const float* q,
                            int64_t q_elems, int n_spans, const int64_t* qs, const int64_t* ql,
                            const int64_t* cl, const int64_t* co, const int32_t* bt,
                            const int64_t* bt_off) {
    RaggedQueryBatch b;
    b.n_head = n_head;
    b.head_size = head_size;
    b.scale = scale;
    b.q.assign(q, q + q_elems);
    for (int s = 0; s < n_spans; ++s) {
        SubRequest sub;
        sub.req_id = s;
        sub.query_start = qs[s];
        sub.query_len = ql[s];
        sub.context_len = cl[s];
        sub.causal_offset = co[s];
        sub.block_table.assign(bt + bt_off[s], bt + bt_off[s + 1]);
        b.sub_requests.push_back(std::move(sub));
    }
    return b;
}

} // namespace

extern "C" {

// ------------------------------------------------------------------------ attention
void* ref_store_create(int chunk, int n_kv_head, int head_size, int n_slots,
                       const float* keys, const float* values) {
    auto* st = new PagedKvStore(chunk, n_kv_head, head_size, n_slots);
    if (keys) std::memcpy(st->keys.data(), keys, st->keys.size() * sizeof(float));
    if (values) std::memcpy(st->values.data(), values, st->values.size() * sizeof(float));
    return st;
}

void ref_store_destroy(void* h) { delete static_cast<PagedKvStore*>(h); }

// mode 0: paged_multi_token_attention, 1: single_token_attention, 2: copyout_then_dense
int ref_attention(void* store, int mode, int n_head, int head_size, double scale,
                  const float* q, int64_t q_elems, int n_spans, const int64_t* qs,
                  const int64_t* ql, const int64_t* cl, const int64_t* co, const int32_t* bt,
                  const int64_t* bt_off, float* out, uint64_t* gathered_values) {
    const auto& st = *static_cast<PagedKvStore*>(store);
    return guarded([&] {
        RaggedQueryBatch b = make_batch(n_head, head_size, scale, q, q_elems, n_spans, qs, ql,
                                        cl, co, bt, bt_off);
        std::vector<float> o;
        if (mode == 0) {
            o = paged_multi_token_attention(b, st);
        } else if (mode == 1) {
            o = single_token_attention(b, st);
        } else {
            CopyOutResult r = copyout_then_dense(b, st);
            o = std::move(r.out);
            if (gathered_values) *gathered_values = r.gathered_values;
        }
        std::memcpy(out, o.data(), o.size() * sizeof(float));
    });
}

// The reference's paged_multi_token_attention run per sub-request on n_threads host
// threads (batch items may be evaluated independently).  Each thread hands
// the reference a one-span RaggedQueryBatch; outputs are bit-identical to a single call.
int ref_attention_mt(void* store, int n_threads, int n_head, int head_size, double scale,
                     const float* q, int n_spans, const int64_t* qs, const int64_t* ql,
                     const int64_t* cl, const int64_t* co, const int32_t* bt,
                     const int64_t* bt_off, float* out) {
    const auto& st = *static_cast<PagedKvStore*>(store);
    const int64_t row = static_cast<int64_t>(n_head) * head_size;
    std::atomic<int> next{0};
    std::atomic<int> status{kOk};
    auto worker = [&] {
        for (;;) {
            int s = next.fetch_add(1);
            if (s >= n_spans) return;
            int rc = guarded([&] {
                int64_t zero = 0;
                int64_t off[2] = {0, bt_off[s + 1] - bt_off[s]};
                RaggedQueryBatch b =
                    make_batch(n_head, head_size, scale, q + qs[s] * row, ql[s] * row, 1, &zero,
                               &ql[s], &cl[s], &co[s], bt + bt_off[s], off);
                std::vector<float> o = paged_multi_token_attention(b, st);
                std::memcpy(out + qs[s] * row, o.data(), o.size() * sizeof(float));
            });
            if (rc != kOk) status.store(rc);
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, n_threads); ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    return status.load();
}

int ref_dense_attention(const float* q, const float* k, const float* v, int64_t q_len,
                        int64_t kv_len, int64_t causal_offset, int n_head, int n_kv_head,
                        int head_size, double scale, float* out) {
    return guarded([&] {
        std::vector<float> qv(q, q + q_len * n_head * head_size);
        std::vector<float> kv(k, k + kv_len * n_kv_head * head_size);
        std::vector<float> vv(v, v + kv_len * n_kv_head * head_size);
        auto o = dense_attention(qv, kv, vv, q_len, kv_len, causal_offset, n_head, n_kv_head,
                                 head_size, scale);
        std::memcpy(out, o.data(), o.size() * sizeof(float));
    });
}

// qkv_project's paged K/V write (proj/src/attention.cpp:287-329) with identity-free
// weights supplied by the caller; returns q/k/v projections and updates the store.
int ref_qkv_project(void* store, const float* x, int rows, int hidden, const float* wq,
                    int q_cols, const float* wk, const float* wv, int kv_cols,
                    const int32_t* bt, int64_t bt_len, int64_t start_pos, float* q_out,
                    float* k_out, float* v_out) {
    auto& st = *static_cast<PagedKvStore*>(store);
    return guarded([&] {
        Mat mx(rows, hidden), mq(hidden, q_cols), mk(hidden, kv_cols), mv(hidden, kv_cols);
        std::memcpy(mx.data.data(), x, sizeof(float) * mx.data.size());
        std::memcpy(mq.data.data(), wq, sizeof(float) * mq.data.size());
        std::memcpy(mk.data.data(), wk, sizeof(float) * mk.data.size());
        std::memcpy(mv.data.data(), wv, sizeof(float) * mv.data.size());
        std::vector<SlotId> table(bt, bt + bt_len);
        QkvResult r = qkv_project(mx, mq, mk, mv, st, table, start_pos);
        std::memcpy(q_out, r.q.data.data(), sizeof(float) * r.q.data.size());
        std::memcpy(k_out, r.k.data.data(), sizeof(float) * r.k.data.size());
        std::memcpy(v_out, r.v.data.data(), sizeof(float) * r.v.data.size());
    });
}

void ref_store_read(void* store, float* keys, float* values) {
    const auto& st = *static_cast<PagedKvStore*>(store);
    std::memcpy(keys, st.keys.data(), st.keys.size() * sizeof(float));
    std::memcpy(values, st.values.data(), st.values.size() * sizeof(float));
}

// ------------------------------------------------------------------------ SplitMix64
uint64_t ref_splitmix_next(uint64_t* state) {
    SplitMix64 r{*state};
    uint64_t v = r.next();
    *state = r.state;
    return v;
}

// ------------------------------------------------------------------------ model config
int ref_model_bytes(const char* preset, int n_kv_override, int chunk, uint64_t* kv_token_bytes,
                    uint64_t* chunk_bytes) {
    return guarded([&] {
        ModelConfig m = ModelConfig::preset(preset);
        if (n_kv_override > 0) m.n_kv_head = n_kv_override;
        *kv_token_bytes = m.kv_token_bytes();
        *chunk_bytes = m.chunk_bytes(chunk);
    });
}

// ------------------------------------------------------------------------ swap engine
int ref_schedule_swap_in(double issued_at, uint64_t bytes, int n_layer, double bandwidth,
                         double first_compute_start, const double* per_layer_compute,
                         double* layer_ready, double* attn_start, double* summary3) {
    return guarded([&] {
        std::vector<double> c(per_layer_compute, per_layer_compute + n_layer);
        SwapInSchedule s = schedule_swap_in(issued_at, bytes, n_layer, bandwidth,
                                            first_compute_start, c);
        std::copy(s.layer_ready.begin(), s.layer_ready.end(), layer_ready);
        std::copy(s.attn_start.begin(), s.attn_start.end(), attn_start);
        summary3[0] = s.transfer_done;
        summary3[1] = s.finish;
        summary3[2] = s.stall;
    });
}

int ref_transfer_time(uint64_t bytes, double bandwidth, int contended, double penalty,
                      double* out) {
    return guarded([&] { *out = transfer_time(bytes, bandwidth, contended != 0, penalty); });
}

double ref_swap_out_start(double now, double inflight, int allow_duplex) {
    return schedule_swap_out_start(now, inflight, allow_duplex != 0);
}

// ------------------------------------------------------------------------ PagedKvCache
void* ref_cache_create(int chunk, int device_slots, int host_slots) {
    try {
        return new PagedKvCache(chunk, device_slots, host_slots);
    } catch (const Error&) {
        return nullptr;
    }
}
void ref_cache_destroy(void* h) { delete static_cast<PagedKvCache*>(h); }

// Writes created chunk ids to out (capacity cap); *n_out = count.
int ref_cache_allocate(void* h, int64_t conv, int64_t n_tokens, double now, int64_t* out,
                       int64_t cap, int64_t* n_out) {
    auto& c = *static_cast<PagedKvCache*>(h);
    return guarded([&] {
        auto ids = c.allocate(conv, n_tokens, now);
        *n_out = static_cast<int64_t>(ids.size());
        for (size_t i = 0; i < ids.size() && static_cast<int64_t>(i) < cap; ++i) out[i] = ids[i];
    });
}

int ref_cache_evict(void* h, const int64_t* ids, int64_t n, int to_host) {
    auto& c = *static_cast<PagedKvCache*>(h);
    return guarded([&] {
        std::vector<ChunkId> v(ids, ids + n);
        c.apply_evictions(v, to_host ? EvictTarget::Host : EvictTarget::Dropped);
    });
}

// kind 0 restore, 1 rematerialize; out_slots[i] = device slot for ids[i]
int ref_cache_bring_back(void* h, int kind, const int64_t* ids, int64_t n, int32_t* out_slots) {
    auto& c = *static_cast<PagedKvCache*>(h);
    return guarded([&] {
        std::vector<ChunkId> v(ids, ids + n);
        auto a = kind == 0 ? c.restore(v) : c.rematerialize(v);
        for (size_t i = 0; i < a.size(); ++i) out_slots[i] = a[i].slot;
    });
}

int ref_cache_release(void* h, int64_t conv) {
    auto& c = *static_cast<PagedKvCache*>(h);
    return guarded([&] { c.release_conversation(conv); });
}

int ref_cache_retain(void* h, int64_t conv, double now) {
    auto& c = *static_cast<PagedKvCache*>(h);
    return guarded([&] { c.retain_on_finish(conv, now); });
}

int ref_cache_block_table(void* h, int64_t conv, int64_t ctx, int32_t* out, int64_t cap,
                          int64_t* n_out) {
    auto& c = *static_cast<PagedKvCache*>(h);
    return guarded([&] {
        auto t = c.block_table(conv, ctx);
        *n_out = static_cast<int64_t>(t.size());
        for (size_t i = 0; i < t.size() && static_cast<int64_t>(i) < cap; ++i) out[i] = t[i];
    });
}

// counts[8] = device cap, free, reclaimable, allocated, host cap, free, allocated, verify-rc
void ref_cache_counts(void* h, int64_t* counts) {
    auto& c = *static_cast<PagedKvCache*>(h);
    counts[0] = c.device_capacity();
    counts[1] = c.device_free();
    counts[2] = c.device_reclaimable();
    counts[3] = c.device_allocated();
    counts[4] = c.host_capacity();
    counts[5] = c.host_free();
    counts[6] = c.host_allocated();
    counts[7] = guarded([&] { c.verify(); });
}

int ref_cache_has(void* h, int64_t conv) {
    return static_cast<PagedKvCache*>(h)->has_conversation(conv) ? 1 : 0;
}

int64_t ref_cache_total_tokens(void* h, int64_t conv) {
    return static_cast<PagedKvCache*>(h)->total_tokens(conv);
}

int ref_cache_append_needed(void* h, int64_t conv, int64_t add) {
    return static_cast<PagedKvCache*>(h)->append_chunks_needed(conv, add);
}

// Chunk ids of the conversation (offset order) with location kind (0 device,1 host,
// 2 dropped) and slot.
int ref_cache_conv_chunks(void* h, int64_t conv, int64_t* ids, int32_t* kinds, int32_t* slots,
                          int64_t cap, int64_t* n_out) {
    auto& c = *static_cast<PagedKvCache*>(h);
    return guarded([&] {
        const auto& v = c.conversation_chunks(conv);
        *n_out = static_cast<int64_t>(v.size());
        for (size_t i = 0; i < v.size() && static_cast<int64_t>(i) < cap; ++i) {
            const ChunkRecord& r = c.chunk(v[i]);
            ids[i] = v[i];
            kinds[i] = r.location.kind == ChunkLocationKind::DeviceSlot ? 0
                       : r.location.kind == ChunkLocationKind::HostSlot ? 1
                                                                         : 2;
            slots[i] = r.location.slot;
        }
    });
}

// dump() text; returns required length (excluding NUL), writes up to cap-1 chars.
int64_t ref_cache_dump(void* h, char* buf, int64_t cap) {
    std::string s = static_cast<PagedKvCache*>(h)->dump();
    if (buf && cap > 0) {
        size_t n = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
        std::memcpy(buf, s.data(), n);
        buf[n] = '\0';
    }
    return static_cast<int64_t>(s.size());
}

// ------------------------------------------------------------------------ event log
// The reference's LayerDependencyAuditor over n events (times in seconds, kinds in
// kvsim::EventKind order), fed in the given order.
void ref_audit_layer_deps(int n, const int* kinds, const int* layers, const double* times,
                          unsigned long long* violations, unsigned long long* steps) {
    LayerDependencyAuditor a;
    for (int i = 0; i < n; ++i) {
        LogEvent ev;
        ev.t = times[i];
        ev.kind = static_cast<EventKind>(kinds[i]);
        ev.layer = layers[i];
        a.on_event(ev);
    }
    *violations = a.violations();
    *steps = a.steps_checked();
}

} // extern "C"
