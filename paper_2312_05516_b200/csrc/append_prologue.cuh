// Paged K/V append fused into the attention launch.  Semantics: the
// row-write loop of qkv_project, /root/reference/proj/src/attention.cpp:315-327 — token i of
// span s (row query_start + i of the new K/V rows) goes to position causal_offset + i, i.e.
// page block_table[pos / chunk], row pos % chunk, every kv head.  In the fused launch every
// CTA writes a share of the rows, then a grid-wide barrier orders those writes before any
// CTA's TMA reads the pages.  The barrier needs every CTA co-resident, so launches carrying
// new rows are cooperative (launch_fused / launch_dt fall back to a separate row-write launch
// when the runtime refuses a cooperative launch).
#pragma once

#include "attn_internal.hpp"

#include <cstdint>

namespace pb {

// One token row = n_kv_head * head_size elements (p.row_bytes, a multiple of 16).
__device__ __forceinline__ void append_rows(const AttnParams& p, int first_warp, int n_warps) {
    const int row_vecs = p.row_bytes / 16; // 16-B vectors per token row
    const int lane = threadIdx.x & 31;
    auto* kp = reinterpret_cast<uint4*>(const_cast<void*>(p.k_pages));
    auto* vp = reinterpret_cast<uint4*>(const_cast<void*>(p.v_pages));
    const auto* kn = reinterpret_cast<const uint4*>(p.k_new);
    const auto* vn = reinterpret_cast<const uint4*>(p.v_new);
    for (int t = first_warp; t < p.total_tokens; t += n_warps) {
        // span of token t: the last span whose query_start <= t (query_start is the running
        // total of query_len, so a zero-length span is followed by one with the same start)
        int lo = 0, hi = p.n_spans - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (p.spans[mid].query_start <= t) lo = mid;
            else hi = mid - 1;
        }
        const SpanDev sp = p.spans[lo];
        const int i = t - sp.query_start;
        if (i < 0 || i >= sp.query_len) continue;
        const int pos = sp.causal_offset + i;
        const int slot = p.block_tables[sp.bt_off + pos / p.chunk];
        const size_t dst = (static_cast<size_t>(slot) * p.chunk + pos % p.chunk) * row_vecs;
        const size_t src = static_cast<size_t>(t) * row_vecs;
        for (int v = lane; v < row_vecs; v += 32) {
            kp[dst + v] = kn[src + v];
            vp[dst + v] = vn[src + v];
        }
    }
}

// Whole CTA.  ctr[6] counts arrivals, ctr[7] is the barrier generation (workspace counters).
__device__ __forceinline__ void append_prologue(const AttnParams& p, int* ctr) {
    if (!p.k_new) return;
    append_rows(p, static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5),
                static_cast<int>((gridDim.x * blockDim.x) >> 5));
    // generic-proxy writes -> other CTAs' TMA (async proxy) reads
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile int* gen = ctr + 7;
        const int g0 = *gen;
        if (atomicAdd(ctr + 6, 1) == static_cast<int>(gridDim.x) - 1) {
            ctr[6] = 0;
            __threadfence();
            atomicAdd(ctr + 7, 1);
        } else {
            while (*gen == g0) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

} // namespace pb
