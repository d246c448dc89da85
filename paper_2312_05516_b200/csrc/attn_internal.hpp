// Internal descriptors shared by the attention plan builder (host) and kernels (device).
#pragma once

#include <cstdint>

namespace pb {

// One sub-request span as the kernels see it (include/kvsim/batch.hpp:17-24).
struct SpanDev {
    int32_t query_start;   // token offset into q / out
    int32_t query_len;
    int32_t causal_offset; // token i attends to [0, causal_offset + i]
    int32_t context_len;   // causal_offset + query_len
    int64_t bt_off;        // first block-table entry of this span
    int32_t n_pages;       // ceil(context_len / chunk)
    int32_t pad;
};

enum WorkType : int16_t {
    kWorkSimt = 0,    // generic SIMT tile (fp32 validation mode / unsupported shapes)
    kWorkPrefill = 1, // tcgen05 tile: up to 128 rows = tokens x GQA group, one kv head
    kWorkDecode = 2   // single-token span, one kv head, kv range [kv_begin, kv_end)
};

struct WorkItem {
    int32_t span;
    int32_t kvh;
    int16_t type;
    int16_t n_parts;   // decode: number of kv splits of this (span, kvh); 1 = unsplit
    int16_t part_idx;  // decode: which split
    int16_t pad;
    int32_t t0;        // tiles: first span-relative query token
    int32_t nt;        // tiles: number of query tokens
    int32_t kv_begin;  // decode: first context position (multiple of the page size)
    int32_t kv_end;    // decode: one past the last position
    int32_t group;     // decode split group (counter index), -1 if unsplit
    int32_t part_base; // decode: first partial-result index of the group
};
static_assert(sizeof(WorkItem) == 40, "WorkItem layout");

// Kernel-wide constants for one attention launch.
struct AttnParams {
    int32_t n_head, n_kv_head, head_size, chunk, n_slots, group;
    float scale;             // scores are dot / scale
    float scale_log2;        // log2(e) / scale: exp(dot/scale - m) == exp2(dot*scale_log2 - m')
    int32_t n_items;
    int32_t n_groups;        // decode split groups
    const SpanDev* spans;
    const int32_t* block_tables;
    const WorkItem* items;
    const void* q;
    const void* k_pages;
    const void* v_pages;
    void* out;
    int32_t* counters;       // [n_groups] split arrival counters (self-resetting)
    float* part_ml;          // [n_parts][group][2] running max (log2 domain) and sum
    float* part_o;           // [n_parts][group][head_size] unnormalised outputs
    // workspace counters, all self-resetting (zeroed once per workspace buffer):
    // [0] SIMT decode next unit, [1] SIMT decode retired warps, [2] fused: next tile item,
    // [3] fused: retired CTAs, [4] next tcgen05 decode unit, [5] stand-alone decode: retired
    // CTAs, [6] fused-append grid barrier arrivals, [7] its generation
    int32_t* work_counter;
    // fused launch: decode units next to the tile items (items / n_items)
    const WorkItem* dec_items;
    int32_t n_dec_items;
    int32_t n_dec_ctas;      // CTAs that start on the decode queue
    // diagnostics only (pb_attn_set_trace): per CTA and pass, {mode, items, t_begin, t_end}
    // in %globaltimer ns, 4 x uint64 per (CTA, pass); null in production
    unsigned long long* trace;
    // fused K/V append (pb_attn_run_append): new rows [total_tokens][n_kv][d], null = none
    const void* k_new;
    const void* v_new;
    int32_t total_tokens;
    int32_t n_spans;
    int32_t row_bytes;       // n_kv_head * head_size * element bytes
};

} // namespace pb
