// Library-level C-ABI glue: error strings, launch accounting, and the synchronous
// host-buffer mirrors of the reference's value-semantics attention API
// (/root/reference/proj/include/kvsim/attention.hpp:71-77).
#include "pb_common.hpp"

#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

namespace pb {

namespace {
thread_local std::string t_last_error;
std::atomic<uint64_t> g_launches{0};
thread_local uint64_t* t_capture_count = nullptr; // set while this thread captures a graph
} // namespace

void set_last_error(const std::string& msg) { t_last_error = msg; }
void count_launch(uint64_t n) {
    if (t_capture_count)
        *t_capture_count += n; // captured into a graph: counted when the graph is launched
    else
        g_launches.fetch_add(n, std::memory_order_relaxed);
}
LaunchCapture::LaunchCapture() : prev_(t_capture_count) { t_capture_count = &n; }
LaunchCapture::~LaunchCapture() { t_capture_count = prev_; }

int device_sms() {
    static std::once_flag once[kMaxDevices];
    static int sms[kMaxDevices];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
        cudaGetLastError();
        return 148;
    }
    std::call_once(once[dev], [&] {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = 148;
        }
        sms[dev] = n;
    });
    return sms[dev];
}

void plan_validate_with_q(const pb_attn_shape& s, int32_t n_spans, const int64_t* qs,
                          const int64_t* ql, const int64_t* cl, const int64_t* co,
                          const int32_t* bt, const int64_t* bt_off, int64_t total_tokens,
                          const float* q_host);

namespace {

uint16_t f32_to_bf16_rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) return static_cast<uint16_t>((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

float bf16_to_f32(uint16_t h) {
    uint32_t u = static_cast<uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void alloc(size_t n) { cuda_check(cudaMalloc(&p, n ? n : 16), "cudaMalloc"); }
};

void upload(DevBuf& d, const float* src, int64_t n, int dtype) {
    const size_t eb = dtype == PB_F32 ? 4 : 2;
    d.alloc(static_cast<size_t>(n) * eb);
    if (n == 0) return;
    if (dtype == PB_F32) {
        cuda_check(cudaMemcpy(d.p, src, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice), "H2D");
    } else {
        std::vector<uint16_t> tmp(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) tmp[static_cast<size_t>(i)] = f32_to_bf16_rne(src[i]);
        cuda_check(cudaMemcpy(d.p, tmp.data(), tmp.size() * 2, cudaMemcpyHostToDevice), "H2D");
    }
}

pb_status one_shot(bool single, const pb_attn_shape* shape, int32_t n_spans, const int64_t* qs,
                   const int64_t* ql, const int64_t* cl, const int64_t* co, const int32_t* bt,
                   const int64_t* bt_off, const float* q, int64_t total_tokens,
                   const float* keys, const float* values, float* out) {
    return guarded([&] {
        if (!shape) fail(PB_ERR_ERROR, "null shape");
        const pb_attn_shape& s = *shape;
        plan_validate_with_q(s, n_spans, qs, ql, cl, co, bt, bt_off, total_tokens, q);
        if (single)
            for (int32_t i = 0; i < n_spans; ++i)
                require(ql[i] == 1, "single-token path requires query_len == 1 spans");
        // lazy k_row[0] check of the reference (attention.cpp:100-101): every position a
        // span's last token attends to, every kv head
        const int64_t row = static_cast<int64_t>(s.n_kv_head) * s.head_size;
        for (int32_t i = 0; i < n_spans; ++i) {
            if (ql[i] == 0) continue;
            for (int64_t p = 0; p < cl[i]; ++p) {
                const int64_t slot = bt[bt_off[i] + p / s.chunk_size];
                const float* r = keys + (slot * s.chunk_size + p % s.chunk_size) * row;
                for (int kvh = 0; kvh < s.n_kv_head; ++kvh)
                    if (!std::isfinite(r[static_cast<int64_t>(kvh) * s.head_size]))
                        fail(PB_ERR_NUMERIC, "key cache contains non-finite values");
            }
        }
        const int64_t q_elems = total_tokens * s.n_head * s.head_size;
        const int64_t pool_elems = static_cast<int64_t>(s.n_slots) * s.chunk_size * row;
        pb_attn_plan* plan = nullptr;
        pb_status st = pb_attn_plan_create(shape, n_spans, qs, ql, cl, co, bt, bt_off, total_tokens,
                                           single ? PB_PLAN_SINGLE_TOKEN : 0, &plan);
        if (st != PB_OK) fail(st, pb_last_error());
        struct PlanGuard {
            pb_attn_plan* p;
            ~PlanGuard() { pb_attn_plan_destroy(p); }
        } guard{plan};
        st = pb_attn_plan_upload(plan, nullptr);
        if (st != PB_OK) fail(st, pb_last_error());
        DevBuf dq, dk, dv, dout, dws;
        upload(dq, q, q_elems, s.dtype);
        upload(dk, keys, pool_elems, s.dtype);
        upload(dv, values, pool_elems, s.dtype);
        const size_t eb = s.dtype == PB_F32 ? 4 : 2;
        dout.alloc(static_cast<size_t>(q_elems) * eb);
        dws.alloc(pb_attn_plan_workspace_bytes(plan));
        cuda_check(cudaMemset(dws.p, 0, pb_attn_plan_workspace_bytes(plan)), "workspace memset");
        st = pb_attn_run(plan, dq.p, dk.p, dv.p, dout.p, dws.p, nullptr);
        if (st != PB_OK) fail(st, pb_last_error());
        cuda_check(cudaDeviceSynchronize(), "attention");
        if (q_elems == 0) return;
        if (s.dtype == PB_F32) {
            cuda_check(cudaMemcpy(out, dout.p, static_cast<size_t>(q_elems) * 4, cudaMemcpyDeviceToHost), "D2H");
        } else {
            std::vector<uint16_t> tmp(static_cast<size_t>(q_elems));
            cuda_check(cudaMemcpy(tmp.data(), dout.p, tmp.size() * 2, cudaMemcpyDeviceToHost), "D2H");
            for (int64_t i = 0; i < q_elems; ++i) out[i] = bf16_to_f32(tmp[static_cast<size_t>(i)]);
        }
    });
}

} // namespace
} // namespace pb

using namespace pb;

extern "C" {

const char* pb_last_error(void) { return t_last_error.c_str(); }
const char* pb_version(void) { return "pensieve_b200 0.1 (sm_100a)"; }
uint64_t pb_launch_count(void) { return g_launches.load(); }

pb_status pb_paged_multi_token_attention(const pb_attn_shape* shape, int32_t n_spans,
                                         const int64_t* query_start, const int64_t* query_len,
                                         const int64_t* context_len, const int64_t* causal_offset,
                                         const int32_t* block_tables,
                                         const int64_t* block_table_offsets, const float* q,
                                         int64_t total_tokens, const float* keys,
                                         const float* values, float* out) {
    return one_shot(false, shape, n_spans, query_start, query_len, context_len, causal_offset,
                    block_tables, block_table_offsets, q, total_tokens, keys, values, out);
}

pb_status pb_single_token_attention(const pb_attn_shape* shape, int32_t n_spans,
                                    const int64_t* query_start, const int64_t* query_len,
                                    const int64_t* context_len, const int64_t* causal_offset,
                                    const int32_t* block_tables,
                                    const int64_t* block_table_offsets, const float* q,
                                    int64_t total_tokens, const float* keys, const float* values,
                                    float* out) {
    return one_shot(true, shape, n_spans, query_start, query_len, context_len, causal_offset,
                    block_tables, block_table_offsets, q, total_tokens, keys, values, out);
}

} // extern "C"
