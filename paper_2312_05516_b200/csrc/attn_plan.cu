// Host side of the attention C-ABI: batch validation (the reference's check_batch), the
// work-list builder, descriptor upload and the per-layer launch.
//
// The plan is the B200 analogue of the "auxiliary data computed on the CPU and reused
// across layers" of PAPER.md:967-970: spans, the block-table CSR and the work list are
// built once per batch, uploaded once, and every layer's pb_attn_run reuses them.
#include "attn_internal.hpp"
#include "pb_common.hpp"
#include "sm100_attn.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#ifndef PB_DEC_CTA_SCALE_SMALL
#define PB_DEC_CTA_SCALE_SMALL 2.0 // decode CTA share multiplier below a 25% decode share
#endif
#ifndef PB_DEC_CTA_SCALE_LARGE
#define PB_DEC_CTA_SCALE_LARGE 0.6 // ... and at or above it (config 2: 5014 -> 5104 GB/s, config 5:
                                   // 3939 -> 4053 over 1.0; 0.4-1.2 swept, profiles/r2_experiments.md)
#endif

namespace pb {
void launch_attn_simt(const AttnParams& p, int dtype, int n_items, cudaStream_t stream);
void launch_check_numerics(const AttnParams& p, int dtype, int64_t q_elems, int32_t* d_flag,
                           cudaStream_t stream);
} // namespace pb

using namespace pb;

struct pb_attn_plan {
    pb_attn_shape shape{};
    int32_t flags = 0;
    int32_t group = 1;
    int64_t total_tokens = 0;
    std::vector<SpanDev> spans;
    std::vector<int32_t> bt;
    std::vector<WorkItem> simt_items;
    std::vector<WorkItem> tc_items;     // prefill tiles for the sm_100a tcgen05 kernel
    std::vector<WorkItem> decode_items; // single-token split-KV units
    bool decode_kernel = false;         // decode units built (else decode spans go SIMT)
    bool fused = false;                 // decode units ride in the tile kernel's launch
    double dec_share = 0;               // fused: est. share of SM time spent on decode units
    void* trace = nullptr;              // diagnostics: per-CTA pass timeline (pb_attn_set_trace)
    void* h_buf = nullptr;              // pinned upload staging
    size_t h_bytes = 0;
    cudaEvent_t up_done = nullptr;
    cudaStream_t side = nullptr;        // decode units overlap the tile kernel tail
    cudaEvent_t fork = nullptr, join = nullptr;
    cudaStream_t io[2] = {nullptr, nullptr}; // pb_attn_run_layers_host: H2D and D2H streams
    cudaEvent_t io_ev[10] = {};
    int32_t n_groups = 0;
    int32_t n_parts = 0;
    int32_t n_prefill = 0, n_decode = 0, n_split_spans = 0;
    double flops = 0, bytes = 0;
    // device copies: [spans | block tables | simt items | tc items]
    void* d_buf = nullptr;
    size_t d_bytes = 0;
    size_t off_bt = 0, off_simt = 0, off_tc = 0, off_dec = 0;
    size_t off_ctr = 0; // split-group arrival counters: plan-private (zeroed by the upload,
                        // self-resetting), so plans sharing one workspace cannot clobber them
    bool uploaded = false;
    void* last_workspace = nullptr;
    Sm100Cache sm100;
    // pb_attn_run_layers: the layer loop captured once as a CUDA graph, replayed while the
    // pointers (and trace buffer) it was captured with stay the same
    cudaStream_t cap = nullptr;
    cudaGraphExec_t gexec = nullptr;
    std::vector<const void*> gkey;
    uint64_t g_launches = 0; // kernels per replay
};

namespace {

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int sm_count() { return device_sms(); }

int dtype_bytes(int dtype) { return dtype == PB_F32 ? 4 : 2; }

// check_batch, /root/reference/proj/src/attention.cpp:23-48, in the reference's order.
// q (host) may be null: the finiteness scan then moves to pb_attn_check_numerics.
void validate(const pb_attn_shape& s, int32_t n_spans, const int64_t* qs, const int64_t* ql,
              const int64_t* cl, const int64_t* co, const int32_t* bt, const int64_t* bt_off,
              int64_t total_tokens, const float* q_host) {
    require(s.n_head > 0 && s.head_size > 0, "batch head shape must be positive");
    require(s.n_kv_head > 0, "store/batch head_size mismatch");
    require(s.n_head % s.n_kv_head == 0, "n_head must be a multiple of the store's n_kv_head");
    require(s.scale > 0, "scale must be positive");
    if (s.chunk_size < 1) fail(PB_ERR_CONFIG, "chunk_size must be >= 1");
    if (s.n_slots < 0) fail(PB_ERR_CONFIG, "n_slots must be >= 0");
    if (s.dtype != PB_F32 && s.dtype != PB_BF16) fail(PB_ERR_UNSUPPORTED, "dtype must be f32 or bf16");
    if (q_host) {
        const int64_t n = total_tokens * s.n_head * s.head_size;
        for (int64_t i = 0; i < n; ++i)
            if (!std::isfinite(q_host[i])) fail(PB_ERR_NUMERIC, "query contains non-finite values");
    }
    require(n_spans >= 0, "negative span count");
    int64_t expect = 0;
    for (int32_t i = 0; i < n_spans; ++i) {
        require(ql[i] >= 0, "negative query span");
        require(qs[i] == expect, "sub-request spans must tile the batch");
        require(cl[i] == co[i] + ql[i], "context_len must equal causal_offset + query_len");
        require(co[i] >= 0, "negative causal offset");
        const int64_t need = (cl[i] + s.chunk_size - 1) / s.chunk_size;
        require(bt_off[i + 1] - bt_off[i] == need,
                "block table must cover exactly ceil(context/chunk_size) slots");
        for (int64_t j = bt_off[i]; j < bt_off[i + 1]; ++j)
            if (bt[j] < 0 || bt[j] >= s.n_slots)
                fail(PB_ERR_ERROR, "block table references out-of-range slot " + std::to_string(bt[j]));
        expect += ql[i];
    }
    require(expect == total_tokens, "sub-request spans must tile the batch");
    if (total_tokens > INT32_MAX / 2) fail(PB_ERR_UNSUPPORTED, "too many query tokens");
    for (int32_t i = 0; i < n_spans; ++i)
        if (cl[i] > INT32_MAX / 2) fail(PB_ERR_UNSUPPORTED, "context too long");
}

// Decode spans are cut into units of at most split_pages pages (split-KV); partial results
// are merged by the last-arriving unit inside the same launch.  The unit size adapts to the
// batch: ~kDecodeUnitsTarget units in total (several per decode warp on 148 SMs, for load
// balance), never more than 64 pages (the decode kernel caches a unit's block-table slice in
// two registers per lane) and never fewer than 8.
constexpr int kDecodeUnitsTarget = 4096;

void build_work(pb_attn_plan& P) {
    const pb_attn_shape& s = P.shape;
    const int g = P.group;
    const bool tc = (P.flags & PB_PLAN_FORCE_SIMT) == 0 && s.dtype == PB_BF16 &&
                    sm100_supports(s.head_size, s.chunk_size, g);
    // SIMT tiles: blocks of tokens, ~16 rows per warp-pass
    const int simt_tokens = std::max(1, 32 / g);
    const int tc_tokens = tc ? sm100_tile_tokens(g) : 0;
    P.decode_kernel = tc && (decode_supports(s.head_size, s.chunk_size, g) ||
                             decode_tc_supports(s.head_size, s.chunk_size, g));
    std::vector<std::pair<double, WorkItem>> tc_list, dec_list;
    int64_t decode_pages = 0;
    for (const SpanDev& sp : P.spans)
        if (sp.query_len == 1) decode_pages += static_cast<int64_t>(sp.n_pages) * s.n_kv_head;
    // the tcgen05 decode kernel streams one unit per CTA (148 in flight): ~10 units per CTA,
    // 16..128 pages each; the SIMT kernel streams one unit per warp: ~kDecodeUnitsTarget units
    const bool dec_tc = P.decode_kernel && decode_tc_supports(s.head_size, s.chunk_size, g);
    int64_t decode_pairs = 0;
    for (const SpanDev& sp : P.spans)
        if (sp.query_len == 1) decode_pairs += s.n_kv_head;
    // tcgen05 decode: a split span costs a partial write, an atomic ticket and a merge, which
    // measured slower than whole spans as soon as there is at least one (span, kv head) pair
    // per CTA (cfg3: 95% -> 99% of HBM; the config-5 steps: 52 -> 40 us); with fewer pairs,
    // split to ~1.5 units per CTA (>= 16 pages each).
    const int64_t sms = sm_count();
    bool multi_token = false;
    for (const SpanDev& sp : P.spans) multi_token = multi_token || sp.query_len >= 2;
    // In the fused launch the tile items fill the SMs, so decode spans stay whole: splitting
    // them to fill the GPU (the decode-only rule below) only adds partial writes and merges
    // to the few decode CTAs (config 4 at an 8-way shard: 86.0 -> 75.8 us per layer, 4-way
    // 136.7 -> 126.5; unchanged at 1- and 2-way, where nothing is split).
    const bool fused_launch = dec_tc && tc && multi_token && !(P.flags & PB_PLAN_SEPARATE_DECODE);
    int split_pages;
    if (dec_tc && fused_launch)
        split_pages = 1 << 24; // no split
    else if (dec_tc)
        split_pages = decode_pairs >= sms
                          ? (1 << 24) // no split
                          : static_cast<int>(std::max<int64_t>(16, (2 * decode_pages + 3 * sms - 1) / (3 * sms)));
    else
        split_pages = static_cast<int>(std::max<int64_t>(8, std::min<int64_t>(64, decode_pages / kDecodeUnitsTarget)));
    for (int32_t si = 0; si < static_cast<int32_t>(P.spans.size()); ++si) {
        const SpanDev& sp = P.spans[si];
        if (sp.query_len == 0) continue;
        for (int kvh = 0; kvh < s.n_kv_head; ++kvh) {
            if (!tc) {
                for (int t0 = 0; t0 < sp.query_len; t0 += simt_tokens) {
                    WorkItem w{};
                    w.span = si;
                    w.kvh = kvh;
                    w.type = kWorkSimt;
                    w.t0 = t0;
                    w.nt = std::min(simt_tokens, sp.query_len - t0);
                    w.group = -1;
                    P.simt_items.push_back(w);
                }
            } else if (sp.query_len >= 2) {
                for (int t0 = 0; t0 < sp.query_len; t0 += tc_tokens) {
                    WorkItem w{};
                    w.span = si;
                    w.kvh = kvh;
                    w.type = kWorkPrefill;
                    w.t0 = t0;
                    w.nt = std::min(tc_tokens, sp.query_len - t0);
                    w.group = -1;
                    const double kv = sp.causal_offset + w.t0 + w.nt;
                    // est. SM cycles per kv position: a 128-position kv tile takes ~3400
                    // cycles for two query tiles and ~3000 for one (tile trace: one softmax
                    // group alone is latency-bound, not half the work)
                    tc_list.push_back({kv * (w.nt > sm100_tile_tokens(g) / 2 ? 26.5 : 23.5), w});
                    ++P.n_prefill;
                }
            } else if (!P.decode_kernel) {
                WorkItem w{};
                w.span = si;
                w.kvh = kvh;
                w.type = kWorkSimt;
                w.t0 = 0;
                w.nt = 1;
                w.group = -1;
                P.simt_items.push_back(w);
            } else {
                const int pages = sp.n_pages;
                const int n_parts = (P.flags & PB_PLAN_NO_SPLIT)
                                        ? 1
                                        : std::max(1, (pages + split_pages - 1) / split_pages);
                const int per = (pages + n_parts - 1) / n_parts;
                int group_id = -1, part_base = 0;
                if (n_parts > 1) {
                    group_id = P.n_groups++;
                    part_base = P.n_parts;
                    P.n_parts += n_parts;
                    if (kvh == 0) ++P.n_split_spans;
                }
                for (int part = 0; part < n_parts; ++part) {
                    WorkItem w{};
                    w.span = si;
                    w.kvh = kvh;
                    w.type = kWorkDecode;
                    w.t0 = 0;
                    w.nt = 1;
                    w.n_parts = static_cast<int16_t>(n_parts);
                    w.part_idx = static_cast<int16_t>(part);
                    w.kv_begin = part * per * s.chunk_size;
                    w.kv_end = std::min(sp.context_len, (part + 1) * per * s.chunk_size);
                    w.group = group_id;
                    w.part_base = part_base;
                    // est. SM cycles: 8 KB (K+V, d = 128) per 16 positions at 1/148 of HBM
                    dec_list.push_back({22.5 * static_cast<double>(w.kv_end - w.kv_begin), w});
                    ++P.n_decode;
                }
            }
        }
    }
    // One launch for the whole batch: when both kinds exist and the decode units fit the
    // tensor-core decode path, they join the tile kernel's work list (the fused kernel serves
    // both; HBM-bound units fill SMs next to tensor-bound tiles).
    P.fused = dec_tc && !tc_list.empty() && !dec_list.empty() &&
              !(P.flags & PB_PLAN_SEPARATE_DECODE);
    // Heavy items first so the persistent CTAs finish together (LPT order).
    auto lpt = [](auto& v) {
        std::stable_sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
    };
    lpt(dec_list);
    // Few items per CTA (small shards, e.g. config 4 at a 2..8-way kv-head shard): strict LPT,
    // so no heavy item is taken late by a CTA that already ran one (per-CTA end times: N = 8
    // max 57.4 vs 59.3 us grouped, N = 2 195.3 vs 198.9).  Many items per CTA: grouped by
    // (span, kv head) for L2 reuse of the shared K/V pages (N = 1: 372.4 vs 377.3 us).
    if (!tc_list.empty() && ((P.flags & PB_PLAN_LPT_ORDER) || static_cast<int64_t>(tc_list.size()) < 8 * sms)) {
        lpt(tc_list);
    } else if (!tc_list.empty()) {
        // The query blocks of one (span, kv head) stream the same K/V pages: keeping them
        // adjacent in the queue lets concurrently running CTAs share those pages through L2.
        // Groups go heaviest first (by their heaviest item), items heaviest first inside.
        std::map<std::pair<int32_t, int32_t>, double> gmax;
        for (auto& e : tc_list) {
            auto& m = gmax[{e.second.span, e.second.kvh}];
            m = std::max(m, e.first);
        }
        std::stable_sort(tc_list.begin(), tc_list.end(), [&](const auto& a, const auto& b) {
            const double ga = gmax[{a.second.span, a.second.kvh}], gb = gmax[{b.second.span, b.second.kvh}];
            if (ga != gb) return ga > gb;
            if (a.second.span != b.second.span) return a.second.span < b.second.span;
            if (a.second.kvh != b.second.kvh) return a.second.kvh < b.second.kvh;
            return a.first > b.first;
        });
    } else {
        lpt(tc_list);
    }
    if (P.fused) {
        // share of the launch's SM time the decode queue needs (est. cycles); the fused kernel
        // starts that share of its CTAs on decode units, the rest steal once their queue is dry
        double tot_tile = 0, tot_dec = 0;
        for (auto& e : tc_list) tot_tile += e.first;
        for (auto& e : dec_list) tot_dec += e.first;
        P.dec_share = tot_dec / std::max(1.0, tot_tile + tot_dec);
    }
    P.tc_items.reserve(tc_list.size());
    for (auto& e : tc_list) P.tc_items.push_back(e.second);
    for (auto& e : dec_list) P.decode_items.push_back(e.second);
}

} // namespace

extern "C" {

pb_status pb_attn_plan_create(const pb_attn_shape* shape, int32_t n_spans,
                              const int64_t* query_start, const int64_t* query_len,
                              const int64_t* context_len, const int64_t* causal_offset,
                              const int32_t* block_tables, const int64_t* block_table_offsets,
                              int64_t total_tokens, int32_t flags, pb_attn_plan** out) {
    return guarded([&] {
        if (!shape || !out) fail(PB_ERR_ERROR, "null argument");
        *out = nullptr;
        validate(*shape, n_spans, query_start, query_len, context_len, causal_offset,
                 block_tables, block_table_offsets, total_tokens, nullptr);
        if (flags & PB_PLAN_SINGLE_TOKEN)
            for (int32_t i = 0; i < n_spans; ++i)
                require(query_len[i] == 1, "single-token path requires query_len == 1 spans");
        if (shape->head_size > 256) fail(PB_ERR_UNSUPPORTED, "head_size > 256");
        auto P = std::make_unique<pb_attn_plan>();
        P->shape = *shape;
        P->flags = flags;
        P->group = shape->n_head / shape->n_kv_head;
        P->total_tokens = total_tokens;
        const int64_t n_bt = n_spans > 0 ? block_table_offsets[n_spans] - block_table_offsets[0] : 0;
        P->bt.assign(block_tables + (n_spans > 0 ? block_table_offsets[0] : 0),
                     block_tables + (n_spans > 0 ? block_table_offsets[0] : 0) + n_bt);
        const int eb = dtype_bytes(shape->dtype);
        const double d = shape->head_size;
        for (int32_t i = 0; i < n_spans; ++i) {
            SpanDev sp{};
            sp.query_start = static_cast<int32_t>(query_start[i]);
            sp.query_len = static_cast<int32_t>(query_len[i]);
            sp.causal_offset = static_cast<int32_t>(causal_offset[i]);
            sp.context_len = static_cast<int32_t>(context_len[i]);
            sp.bt_off = block_table_offsets[i] - block_table_offsets[0];
            sp.n_pages = static_cast<int32_t>(block_table_offsets[i + 1] - block_table_offsets[i]);
            P->spans.push_back(sp);
            // unmasked score pairs only; K+V once per kv head; Q, O, table.
            const double q = static_cast<double>(query_len[i]);
            const double allowed_sum = q * static_cast<double>(causal_offset[i]) + q * (q + 1) / 2;
            P->flops += 4.0 * shape->n_head * d * allowed_sum;
            if (query_len[i] > 0)
                P->bytes += 2.0 * context_len[i] * shape->n_kv_head * d * eb +
                            2.0 * q * shape->n_head * d * eb + 4.0 * sp.n_pages;
        }
        build_work(*P);
        *out = P.release();
    });
}

pb_status pb_attn_plan_upload(pb_attn_plan* P, void* stream) {
    return guarded([&] {
        if (!P) fail(PB_ERR_ERROR, "null plan");
        const size_t b_spans = sizeof(SpanDev) * P->spans.size();
        P->off_bt = align_up(b_spans, 256);
        P->off_simt = align_up(P->off_bt + sizeof(int32_t) * P->bt.size(), 256);
        P->off_tc = align_up(P->off_simt + sizeof(WorkItem) * P->simt_items.size(), 256);
        P->off_dec = align_up(P->off_tc + sizeof(WorkItem) * P->tc_items.size(), 256);
        P->off_ctr = align_up(P->off_dec + sizeof(WorkItem) * P->decode_items.size(), 256);
        const size_t total = std::max<size_t>(256, P->off_ctr + sizeof(int32_t) * static_cast<size_t>(P->n_groups));
        if (P->d_bytes < total) {
            if (P->d_buf) cudaFree(P->d_buf);
            P->d_buf = nullptr;
            cuda_check(cudaMalloc(&P->d_buf, total), "cudaMalloc(plan descriptors)");
            P->d_bytes = total;
        }
        // One pinned staging copy so the H2D is a single transfer that does not block the
        // host; the staging buffer is reused only after its previous upload completed.
        if (P->h_bytes < total) {
            if (P->h_buf) {
                cudaEventSynchronize(P->up_done);
                cudaFreeHost(P->h_buf);
            }
            P->h_buf = nullptr;
            cuda_check(cudaMallocHost(&P->h_buf, total), "cudaMallocHost(plan staging)");
            P->h_bytes = total;
        }
        if (!P->up_done) cuda_check(cudaEventCreateWithFlags(&P->up_done, cudaEventDisableTiming), "event");
        else cuda_check(cudaEventSynchronize(P->up_done), "plan staging reuse");
        auto* host = static_cast<uint8_t*>(P->h_buf);
        std::memset(host, 0, total);
        if (b_spans) std::memcpy(host, P->spans.data(), b_spans);
        if (!P->bt.empty()) std::memcpy(host + P->off_bt, P->bt.data(), sizeof(int32_t) * P->bt.size());
        if (!P->simt_items.empty())
            std::memcpy(host + P->off_simt, P->simt_items.data(), sizeof(WorkItem) * P->simt_items.size());
        if (!P->tc_items.empty())
            std::memcpy(host + P->off_tc, P->tc_items.data(), sizeof(WorkItem) * P->tc_items.size());
        if (!P->decode_items.empty())
            std::memcpy(host + P->off_dec, P->decode_items.data(), sizeof(WorkItem) * P->decode_items.size());
        cuda_check(cudaMemcpyAsync(P->d_buf, host, total, cudaMemcpyHostToDevice, as_stream(stream)), "plan upload");
        cuda_check(cudaEventRecord(P->up_done, as_stream(stream)), "plan upload event");
        P->uploaded = true;
    });
}

size_t pb_attn_plan_workspace_bytes(const pb_attn_plan* P) {
    if (!P) return 0;
    const size_t g = static_cast<size_t>(P->group);
    size_t b = 256; // work-queue tickets (self-resetting) + padding
    b += align_up(sizeof(float) * 2 * g * static_cast<size_t>(P->n_parts), 256);
    b += align_up(sizeof(float) * g * P->shape.head_size * static_cast<size_t>(P->n_parts), 256);
    return b;
}

void pb_attn_plan_stats(const pb_attn_plan* P, double* o) {
    if (!P || !o) return;
    o[0] = P->n_prefill;
    o[1] = P->n_decode;
    o[2] = P->n_split_spans;
    o[3] = P->flops;
    o[4] = P->bytes;
    o[5] = static_cast<double>(P->total_tokens);
    o[6] = static_cast<double>(P->simt_items.size());
    double rows = 0;
    for (const auto& w : P->simt_items) rows += static_cast<double>(w.nt) * P->group;
    for (const auto& w : P->tc_items)
        if (w.type != kWorkDecode || w.part_idx == 0) rows += static_cast<double>(w.nt) * P->group;
    for (const auto& w : P->decode_items)
        if (w.part_idx == 0) rows += static_cast<double>(w.nt) * P->group;
    o[7] = rows;
}

static AttnParams make_params(pb_attn_plan* P, const void* q, const void* k, const void* v,
                              void* out, void* ws) {
    AttnParams p{};
    p.n_head = P->shape.n_head;
    p.n_kv_head = P->shape.n_kv_head;
    p.head_size = P->shape.head_size;
    p.chunk = P->shape.chunk_size;
    p.n_slots = P->shape.n_slots;
    p.group = P->group;
    p.scale = static_cast<float>(P->shape.scale);
    p.scale_log2 = static_cast<float>(1.4426950408889634 / P->shape.scale);
    p.n_groups = P->n_groups;
    p.total_tokens = static_cast<int32_t>(P->total_tokens);
    p.n_spans = static_cast<int32_t>(P->spans.size());
    p.row_bytes = P->shape.n_kv_head * P->shape.head_size * dtype_bytes(P->shape.dtype);
    auto* base = static_cast<uint8_t*>(P->d_buf);
    p.spans = reinterpret_cast<const SpanDev*>(base);
    p.block_tables = reinterpret_cast<const int32_t*>(base + P->off_bt);
    p.counters = reinterpret_cast<int32_t*>(base + P->off_ctr);
    p.q = q;
    p.k_pages = k;
    p.v_pages = v;
    p.out = out;
    auto* w = static_cast<uint8_t*>(ws);
    if (w) {
        const size_t g = static_cast<size_t>(P->group);
        p.work_counter = reinterpret_cast<int32_t*>(w);
        size_t off = 256;
        p.part_ml = reinterpret_cast<float*>(w + off);
        off += align_up(sizeof(float) * 2 * g * static_cast<size_t>(P->n_parts), 256);
        p.part_o = reinterpret_cast<float*>(w + off);
    }
    return p;
}

// One attention launch sequence for a layer; with k_new / v_new the batch's new K/V rows are
// first written into the pages (fused into the launch where possible).
static void run_impl(pb_attn_plan* P, const void* q, const void* k_pages, const void* v_pages, void* out,
                     void* workspace, void* stream, const void* k_new, const void* v_new) {

        if (!P) fail(PB_ERR_ERROR, "null plan");
        if (!P->uploaded) fail(PB_ERR_ERROR, "plan not uploaded (call pb_attn_plan_upload)");
        if (P->total_tokens == 0) return;
        if (!q || !k_pages || !v_pages || !out) fail(PB_ERR_ERROR, "null device pointer");
        if ((!P->tc_items.empty() || !P->decode_items.empty()) && !workspace)
            fail(PB_ERR_ERROR, "workspace required");
        cudaStream_t st = as_stream(stream);
        AttnParams p = make_params(P, q, k_pages, v_pages, out, workspace);
        p.trace = static_cast<unsigned long long*>(P->trace);
        if (workspace && workspace != P->last_workspace) {
            // the queue tickets are self-resetting; zero them once per workspace buffer
            cuda_check(cudaMemsetAsync(workspace, 0, 256, st), "workspace init");
            P->last_workspace = workspace;
        }
        if (k_new) {
            // fused append: inside the (single) attention launch when there is one, else a
            // stand-alone row-write launch first (the same rows, the same addressing)
            const bool single = P->simt_items.empty() && P->shape.dtype == PB_BF16 &&
                                (P->fused || P->decode_items.empty() ||
                                 (P->tc_items.empty() && decode_tc_supports(P->shape.head_size, P->shape.chunk_size,
                                                                            P->group)));
            if (single) {
                p.k_new = k_new;
                p.v_new = v_new;
            } else {
                AttnParams pa = p;
                pa.k_new = k_new;
                pa.v_new = v_new;
                launch_append_spans(pa, st);
            }
        }
        if (!P->simt_items.empty()) {
            AttnParams ps = p;
            ps.items = reinterpret_cast<const WorkItem*>(static_cast<uint8_t*>(P->d_buf) + P->off_simt);
            ps.n_items = static_cast<int32_t>(P->simt_items.size());
            launch_attn_simt(ps, P->shape.dtype, ps.n_items, st);
        }
        // Tensor-bound tiles and HBM-bound decode units of the same batch: the decode kernel
        // is forked onto a side stream so its persistent CTAs take SMs as soon as tile CTAs
        // retire (the tile kernel's tail) and the two bottlenecks overlap; joined back before
        // pb_attn_run's stream continues.
        if (P->fused) {
            // one launch: tile items and decode units from two queues (sm100_attn.cu)
            // A decode CTA next to tensor-bound tiles streams slower than 1/148 of HBM, so a
            // small decode share is under-estimated: double it below 25% (measured: cfg4 at an
            // 8-way kv-head shard 92 -> 83 us per layer, unchanged at N = 1; cfg2, where decode
            // is most of the launch, is best unscaled, profiles/r1_variants.md).
            const double cta_scale = P->dec_share < 0.25 ? PB_DEC_CTA_SCALE_SMALL : PB_DEC_CTA_SCALE_LARGE;
            AttnParams pf = p;
            pf.items = reinterpret_cast<const WorkItem*>(static_cast<uint8_t*>(P->d_buf) + P->off_tc);
            pf.n_items = static_cast<int32_t>(P->tc_items.size());
            pf.dec_items = reinterpret_cast<const WorkItem*>(static_cast<uint8_t*>(P->d_buf) + P->off_dec);
            pf.n_dec_items = static_cast<int32_t>(P->decode_items.size());
            const int sms = sm_count();
            const int grid = std::min(sms, pf.n_items + pf.n_dec_items);
            pf.n_dec_ctas = std::max(1, std::min({grid - 1, pf.n_dec_items,
                                                  static_cast<int>(std::lround(grid * P->dec_share * cta_scale))}));
            launch_attn_sm100(pf, P->shape, P->sm100, P->total_tokens, st);
            return;
        }
        const bool run_tc = !P->tc_items.empty();
        const bool run_dec = !P->decode_items.empty();
        const bool both = run_tc && run_dec;
        cudaStream_t dst = st;
        if (both) {
            if (!P->side) {
                cuda_check(cudaStreamCreateWithFlags(&P->side, cudaStreamNonBlocking), "side stream");
                cuda_check(cudaEventCreateWithFlags(&P->fork, cudaEventDisableTiming), "event");
                cuda_check(cudaEventCreateWithFlags(&P->join, cudaEventDisableTiming), "event");
            }
            cuda_check(cudaEventRecord(P->fork, st), "fork");
            cuda_check(cudaStreamWaitEvent(P->side, P->fork, 0), "fork wait");
            dst = P->side;
        }
        if (run_tc) {
            AttnParams pt = p;
            pt.items = reinterpret_cast<const WorkItem*>(static_cast<uint8_t*>(P->d_buf) + P->off_tc);
            pt.n_items = static_cast<int32_t>(P->tc_items.size());
            launch_attn_sm100(pt, P->shape, P->sm100, P->total_tokens, st);
        }
        if (run_dec) {
            AttnParams pd = p;
            pd.items = reinterpret_cast<const WorkItem*>(static_cast<uint8_t*>(P->d_buf) + P->off_dec);
            pd.n_items = static_cast<int32_t>(P->decode_items.size());
            launch_attn_decode(pd, P->shape, P->sm100, P->total_tokens, dst);
        }
        if (both) {
            cuda_check(cudaEventRecord(P->join, P->side), "join");
            cuda_check(cudaStreamWaitEvent(st, P->join, 0), "join wait");
        }
    }

pb_status pb_attn_run(pb_attn_plan* P, const void* q, const void* k_pages, const void* v_pages,
                      void* out, void* workspace, void* stream) {
    return guarded([&] { run_impl(P, q, k_pages, v_pages, out, workspace, stream, nullptr, nullptr); });
}

pb_status pb_attn_run_append(pb_attn_plan* P, const void* q, const void* k_new, const void* v_new,
                             void* k_pages, void* v_pages, void* out, void* workspace, void* stream) {
    return guarded([&] {
        if (!k_new || !v_new) fail(PB_ERR_ERROR, "null new-row pointer");
        run_impl(P, q, k_pages, v_pages, out, workspace, stream, k_new, v_new);
    });
}

pb_status pb_attn_run_layers(pb_attn_plan* P, int32_t n_layer, const void* const* q,
                             const void* const* k_pages, const void* const* v_pages, void* const* out,
                             void* workspace, void* stream) {
    return guarded([&] {
        if (!P) fail(PB_ERR_ERROR, "null plan");
        if (n_layer < 0) fail(PB_ERR_DIMENSION_MISMATCH, "n_layer < 0");
        if (!P->uploaded) fail(PB_ERR_ERROR, "plan not uploaded (call pb_attn_plan_upload)");
        if (n_layer == 0 || P->total_tokens == 0) return;
        if (!q || !k_pages || !v_pages || !out) fail(PB_ERR_ERROR, "null argument");
        for (int l = 0; l < n_layer; ++l)
            if (!q[l] || !k_pages[l] || !v_pages[l] || !out[l]) fail(PB_ERR_ERROR, "null device pointer");
        if ((!P->tc_items.empty() || !P->decode_items.empty()) && !workspace)
            fail(PB_ERR_ERROR, "workspace required");
        cudaStream_t st = as_stream(stream);
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cuda_check(cudaStreamIsCapturing(st, &cs), "capture status");
        if (cs != cudaStreamCaptureStatusNone) {
            // inside the caller's own capture: the launches become part of the caller's graph
            for (int l = 0; l < n_layer; ++l) run_impl(P, q[l], k_pages[l], v_pages[l], out[l], workspace, st, nullptr, nullptr);
            return;
        }
        std::vector<const void*> key;
        key.reserve(4 * static_cast<size_t>(n_layer) + 3);
        key.push_back(workspace);
        key.push_back(P->trace);
        key.push_back(reinterpret_cast<const void*>(static_cast<intptr_t>(n_layer)));
        for (int l = 0; l < n_layer; ++l) {
            key.push_back(q[l]);
            key.push_back(k_pages[l]);
            key.push_back(v_pages[l]);
            key.push_back(out[l]);
        }
        if (!P->gexec || key != P->gkey) {
            // the tickets of a new workspace are zeroed here, on the caller's stream, so the
            // graph itself holds only the attention launches
            if (workspace && workspace != P->last_workspace) {
                cuda_check(cudaMemsetAsync(workspace, 0, 256, st), "workspace init");
                P->last_workspace = workspace;
            }
            if (!P->cap) cuda_check(cudaStreamCreateWithFlags(&P->cap, cudaStreamNonBlocking), "capture stream");
            if (P->gexec) {
                cuda_check(cudaGraphExecDestroy(P->gexec), "graph destroy");
                P->gexec = nullptr;
                P->gkey.clear();
            }
            cudaGraph_t g = nullptr;
            uint64_t n_launch = 0;
            cuda_check(cudaStreamBeginCapture(P->cap, cudaStreamCaptureModeRelaxed), "begin capture");
            try {
                LaunchCapture counted;
                for (int l = 0; l < n_layer; ++l)
                    run_impl(P, q[l], k_pages[l], v_pages[l], out[l], workspace, P->cap, nullptr, nullptr);
                n_launch = counted.n;
            } catch (...) {
                cudaStreamEndCapture(P->cap, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            cuda_check(cudaStreamEndCapture(P->cap, &g), "end capture");
            cudaGraphExec_t ge = nullptr;
            const cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
            cudaGraphDestroy(g);
            cuda_check(e, "graph instantiate");
            P->gexec = ge;
            P->gkey = std::move(key);
            P->g_launches = n_launch;
        }
        cuda_check(cudaGraphLaunch(P->gexec, st), "graph launch");
        count_launch(P->g_launches);
    });
}

void pb_attn_set_trace(pb_attn_plan* P, void* d_trace) {
    if (P) P->trace = d_trace;
}

size_t pb_attn_stage_bytes(const pb_attn_plan* P) {
    if (!P) return 0;
    const size_t io = align_up(static_cast<size_t>(P->total_tokens) * P->shape.n_head * P->shape.head_size *
                                   dtype_bytes(P->shape.dtype),
                               256);
    return 4 * std::max<size_t>(io, 256); // q[2], out[2]
}

pb_status pb_attn_run_layers_host(pb_attn_plan* P, int32_t n_layer, const void* const* q_host,
                                  void* const* out_host, const void* const* k_pages,
                                  const void* const* v_pages, void* staging, void* workspace,
                                  void* stream) {
    return guarded([&] {
        if (!P) fail(PB_ERR_ERROR, "null plan");
        if (n_layer < 0) fail(PB_ERR_DIMENSION_MISMATCH, "n_layer < 0");
        if (n_layer == 0 || P->total_tokens == 0) return;
        if (!q_host || !out_host || !k_pages || !v_pages || !staging) fail(PB_ERR_ERROR, "null argument");
        cudaStream_t st = as_stream(stream);
        if (!P->io[0]) {
            for (auto& x : P->io) cuda_check(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking), "io stream");
            for (auto& e : P->io_ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "io event");
        }
        cudaStream_t h2d = P->io[0], d2h = P->io[1];
        // events: [0..1] q ready, [2..3] q free, [4..5] out ready, [6..7] out free
        cudaEvent_t* ev = P->io_ev;
        const size_t bytes = static_cast<size_t>(P->total_tokens) * P->shape.n_head * P->shape.head_size *
                             dtype_bytes(P->shape.dtype);
        const size_t slot = pb_attn_stage_bytes(P) / 4;
        auto* base = static_cast<uint8_t*>(staging);
        // the layer loop starts after whatever is already queued on the caller's stream
        cuda_check(cudaEventRecord(ev[8], st), "io event");
        cuda_check(cudaStreamWaitEvent(h2d, ev[8], 0), "io wait");
        for (int32_t l = 0; l < n_layer; ++l) {
            const int b = l & 1;
            void* qd = base + b * slot;
            void* od = base + (2 + b) * slot;
            if (l >= 2) cuda_check(cudaStreamWaitEvent(h2d, ev[2 + b], 0), "q free wait");
            cuda_check(cudaMemcpyAsync(qd, q_host[l], bytes, cudaMemcpyHostToDevice, h2d), "q H2D");
            cuda_check(cudaEventRecord(ev[b], h2d), "q ready");
            cuda_check(cudaStreamWaitEvent(st, ev[b], 0), "q ready wait");
            if (l >= 2) cuda_check(cudaStreamWaitEvent(st, ev[6 + b], 0), "out free wait");
            const pb_status r = pb_attn_run(P, qd, k_pages[l], v_pages[l], od, workspace, st);
            if (r != PB_OK) fail(r, "pb_attn_run");
            cuda_check(cudaEventRecord(ev[2 + b], st), "q free");
            cuda_check(cudaEventRecord(ev[4 + b], st), "out ready");
            cuda_check(cudaStreamWaitEvent(d2h, ev[4 + b], 0), "out ready wait");
            cuda_check(cudaMemcpyAsync(out_host[l], od, bytes, cudaMemcpyDeviceToHost, d2h), "out D2H");
            cuda_check(cudaEventRecord(ev[6 + b], d2h), "out free");
        }
        cuda_check(cudaEventRecord(ev[9], d2h), "io done");
        cuda_check(cudaStreamWaitEvent(st, ev[9], 0), "io done wait");
    });
}

pb_status pb_attn_check_numerics(pb_attn_plan* P, const void* q, const void* k_pages,
                                 int32_t* d_flag, void* stream) {
    return guarded([&] {
        if (!P || !P->uploaded) fail(PB_ERR_ERROR, "plan not uploaded");
        AttnParams p = make_params(P, q, k_pages, nullptr, nullptr, nullptr);
        p.n_items = static_cast<int32_t>(P->spans.size());
        launch_check_numerics(p, P->shape.dtype, P->total_tokens * P->shape.n_head * P->shape.head_size,
                              d_flag, as_stream(stream));
    });
}

void pb_attn_plan_destroy(pb_attn_plan* P) {
    if (!P) return;
    if (P->up_done) {
        cudaEventSynchronize(P->up_done);
        cudaEventDestroy(P->up_done);
    }
    if (P->h_buf) cudaFreeHost(P->h_buf);
    if (P->d_buf) cudaFree(P->d_buf);
    sm100_cache_release(P->sm100);
    if (P->io[0]) {
        for (auto& x : P->io) {
            cudaStreamSynchronize(x);
            cudaStreamDestroy(x);
        }
        for (auto& e : P->io_ev) cudaEventDestroy(e);
    }
    if (P->side) {
        cudaStreamSynchronize(P->side);
        cudaStreamDestroy(P->side);
        cudaEventDestroy(P->fork);
        cudaEventDestroy(P->join);
    }
    if (P->gexec) cudaGraphExecDestroy(P->gexec);
    if (P->cap) cudaStreamDestroy(P->cap);
    delete P;
}

} // extern "C"

// Host-side helpers for the one-shot API (api_host.cu).
namespace pb {
void plan_validate_with_q(const pb_attn_shape& s, int32_t n_spans, const int64_t* qs,
                          const int64_t* ql, const int64_t* cl, const int64_t* co,
                          const int32_t* bt, const int64_t* bt_off, int64_t total_tokens,
                          const float* q_host) {
    validate(s, n_spans, qs, ql, cl, co, bt, bt_off, total_tokens, q_host);
}
} // namespace pb
