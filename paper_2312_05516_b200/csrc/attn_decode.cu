// Single-token (decode) spans: memory-bound split-KV SIMT path.
//
// Semantics: single_token_attention, /root/reference/proj/src/attention.cpp:134-188 (one
// query row per head against the whole context; identical to the multi-token path with
// q_len = 1).  B200 design:
//   * one work unit = (span, kv head, page range of <= 64 pages); long contexts are split and
//     the partial (max, sum, unnormalised O) of each split is merged in the same launch by
//     the last-arriving split (atomic ticket, self-resetting);
//   * all `group` query heads of the kv head are served by the same K/V bytes;
//   * persistent CTAs; every WARP is an independent streaming engine: it pulls units from a
//     global atomic queue (work stealing, units sorted longest-first) and keeps a private
//     3-stage ring of 16-token pages filled by TMA ({64 dims, 1 kv head, 16 rows} boxes,
//     SWIZZLE_128B, so row reads are bank-conflict free) that runs ahead ACROSS unit
//     boundaries — no per-unit pipeline start-up, no cross-warp merge;
//   * the unit's q rows (bf16, contiguous) arrive by cp.async.bulk on their own barrier,
//     issued together with the unit's first page;
//   * scores: lane = (page row, half of the dims), halves combined with one shuffle, page max
//     with 4 xor-shuffles per head; P broadcast through shared memory; lanes own D/32 output
//     dims for the PV update.
#include "attn_internal.hpp"
#include "pb_common.hpp"
#include "sm100_attn.hpp"
#include "sm100_ptx.cuh"

#include <cuda.h>
#include <cuda_bf16.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdlib>
#include <string>

namespace pb {

namespace {

using namespace pb::sm100;

constexpr int kDecStages = 2; // page ring depth per warp (1 page in flight while one is consumed)
constexpr int kMaxGroup = 16;

// warps per CTA (one CTA per SM): as many independent page streams as shared memory allows
// (defined after DecWarp: the count is bounded by shared memory and by registers)

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { // FFMA2 (sm_100)
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(d)
        : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
          "l"(*reinterpret_cast<uint64_t*>(&c)));
    return *reinterpret_cast<float2*>(&d);
}

template <int D, int G>
struct __align__(1024) DecWarp {
    static constexpr int KH = D / 64;
    static constexpr int kPageBytes = 16 * D * 2;        // one kv head, 16 rows
    uint8_t page[kDecStages][2][kPageBytes];             // [stage][K|V][half][row][128 B]
    // q rows of a unit, slot = unit seq % stages: bf16 by cp.async.bulk, widened to fp32 in
    // place when the unit starts
    uint8_t qraw[kDecStages][G * D * 4];
    float pbuf[G][16];                                   // page probabilities
    uint64_t full[kDecStages];
    uint64_t qfull[kDecStages];
};

// warps per CTA (one CTA per SM): as many independent page streams as shared memory (227 KB)
// and the register file allow (the G=8 and G=16 variants need ~250 registers per thread)
template <int D, int G>
constexpr int dec_warps() {
    constexpr int by_smem = static_cast<int>((232448 - 1024) / sizeof(DecWarp<D, G>));
    constexpr int by_regs = G >= 16 ? 6 : (G >= 8 ? 8 : 12);
    return by_smem < by_regs ? by_smem : by_regs;
}

__device__ __forceinline__ float bf_lo(uint32_t x) { return __uint_as_float(x << 16); }
__device__ __forceinline__ float bf_hi(uint32_t x) { return __uint_as_float(x & 0xffff0000u); }

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <int D, int G>
__global__ void __launch_bounds__(dec_warps<D, G>() * 32, 1)
    attn_decode_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                       const AttnParams p) {
    constexpr int KH = D / 64;
    constexpr int kChunks = D / 16;       // 16 B chunks per lane and row (D/2 dims)
    constexpr int kDimsPerLane = D / 32;
    constexpr int kWarps = dec_warps<D, G>();
    constexpr int kFifo = kDecStages + 1;
    using W = DecWarp<D, G>;
    extern __shared__ uint8_t smem_raw[];
    // align with pointer arithmetic on the __shared__ array so accesses stay LDS/STS
    uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    W& s = *reinterpret_cast<W*>(base + warp * sizeof(W));
    const int g = p.group;
    const float sl2 = p.scale_log2;
    const uint32_t q_bytes = static_cast<uint32_t>(g * D * 2);
    const uint32_t page_tx = 2u * KH * 16u * 128u;
    int* queue = p.work_counter; // [0] next unit, [1] retired warps

    if (lane == 0) {
        for (int st = 0; st < kDecStages; ++st) {
            mbar_init(&s.full[st], 1);
            mbar_init(&s.qfull[st], 1);
        }
        mbar_fence_init();
    }
    __syncwarp();

    // ---- unit FIFO: fetched in order; the issue and consume cursors walk the same sequence ----
    int fifo[kFifo];
    int n_fetched = 0;
    bool exhausted = false;
    auto fetch = [&]() {
        int u = 0;
        if (lane == 0) u = atomicAdd(&queue[0], 1);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= p.n_items) {
            exhausted = true;
            return;
        }
        fifo[n_fetched % kFifo] = u;
        ++n_fetched;
    };

    int iss_unit = 0, iss_page = 0; // issue cursor
    int issued = 0, consumed = 0;   // pages
    // issue-side cache of the unit being issued: no global loads per page (the block-table
    // slice of the unit, <= 64 pages, lives in two registers per lane)
    int iss_np = -1, iss_kvh = 0, tbl_lo = 0, tbl_hi = 0;
    const __nv_bfloat16* iss_q = nullptr;
    fetch();
    auto issue_one = [&]() -> bool {
        while (true) {
            if (iss_unit >= n_fetched) {
                if (exhausted) return false;
                fetch();
                if (iss_unit >= n_fetched) return false;
            }
            if (iss_np < 0) { // first page of a new unit: load its descriptor once
                const WorkItem wi = p.items[fifo[iss_unit % kFifo]];
                const SpanDev sp = p.spans[wi.span];
                iss_np = (wi.kv_end - wi.kv_begin + 15) >> 4;
                iss_kvh = wi.kvh;
                const int32_t* t = p.block_tables + sp.bt_off + (wi.kv_begin >> 4);
                tbl_lo = lane < iss_np ? t[lane] : 0;
                tbl_hi = lane + 32 < iss_np ? t[lane + 32] : 0;
                iss_q = static_cast<const __nv_bfloat16*>(p.q) +
                        (static_cast<size_t>(sp.query_start) * p.n_head + static_cast<size_t>(wi.kvh) * g) * D;
            }
            if (iss_page < iss_np) break;
            ++iss_unit;
            iss_page = 0;
            iss_np = -1;
        }
        const int stage = issued % kDecStages;
        int slot = __shfl_sync(0xffffffffu, iss_page < 32 ? tbl_lo : tbl_hi, iss_page & 31);
        if (iss_page >= 64) { // unsplit long unit (PB_PLAN_NO_SPLIT): past the cached slice
            const WorkItem wi = p.items[fifo[iss_unit % kFifo]];
            slot = p.block_tables[p.spans[wi.span].bt_off + (wi.kv_begin >> 4) + iss_page];
        }
        if (lane == 0) {
            fence_proxy_async_smem();
            if (iss_page == 0) {
                uint64_t* qb = &s.qfull[iss_unit % kDecStages];
                mbar_arrive_expect_tx(qb, q_bytes);
                bulk_g2s(s.qraw[iss_unit % kDecStages], iss_q, q_bytes, qb);
            }
            const int row = slot * 16;
            uint8_t* dst = s.page[stage][0];
            mbar_arrive_expect_tx(&s.full[stage], page_tx);
            for (int h = 0; h < KH; ++h) {
                tma_load_3d(dst + h * 2048, &tm_k, &s.full[stage], h * 64, iss_kvh, row);
                tma_load_3d(dst + W::kPageBytes + h * 2048, &tm_v, &s.full[stage], h * 64, iss_kvh, row);
            }
        }
        ++iss_page;
        ++issued;
        return true;
    };
    for (int i = 0; i < kDecStages; ++i)
        if (!issue_one()) break;

    const int r = lane & 15;   // page row scored by this lane
    const int hh = lane >> 4;  // half of the dims
    int con_unit = 0;
    while (consumed < issued) {
        // ---------------- start of a unit ----------------
        const WorkItem w = p.items[fifo[con_unit % kFifo]];
        const SpanDev sp = p.spans[w.span];
        const int np = (w.kv_end - w.kv_begin + 15) >> 4;
        mbar_wait(&s.qfull[con_unit % kDecStages], (con_unit / kDecStages) & 1);
        float* qf = reinterpret_cast<float*>(s.qraw[con_unit % kDecStages]); // [g][D] fp32 after widening
        {
            constexpr int kWords = G * D / 2 / 32; // bf16 pairs per lane (upper bound)
            uint32_t wv[kWords];
            const uint32_t* qr = reinterpret_cast<const uint32_t*>(qf);
#pragma unroll
            for (int k = 0; k < kWords; ++k) wv[k] = (lane + 32 * k < g * D / 2) ? qr[lane + 32 * k] : 0u;
            __syncwarp();
#pragma unroll
            for (int k = 0; k < kWords; ++k)
                if (lane + 32 * k < g * D / 2)
                    reinterpret_cast<float2*>(qf)[lane + 32 * k] = make_float2(bf_lo(wv[k]), bf_hi(wv[k]));
        }
        __syncwarp();
        float m_run[G], l_lane[G];
        float2 acc[G][kDimsPerLane / 2]; // FFMA2 pairs of this lane's output dims
#pragma unroll
        for (int j = 0; j < G; ++j) {
            m_run[j] = -CUDART_INF_F;
            l_lane[j] = 0.f;
#pragma unroll
            for (int e = 0; e < kDimsPerLane / 2; ++e) acc[j][e] = make_float2(0.f, 0.f);
        }
        for (int pg = 0; pg < np; ++pg) {
            const int stage = consumed % kDecStages;
            mbar_wait(&s.full[stage], (consumed / kDecStages) & 1);
            const uint8_t* kpg = s.page[stage][0];
            const uint8_t* vpg = s.page[stage][1];
            const int valid_rows = min(16, w.kv_end - (w.kv_begin + pg * 16));
            // ---- scores: lane (r, hh) dots its row's half with every query head ----
            float2 sc[G]; // two partial sums per head (FFMA2 lanes)
#pragma unroll
            for (int j = 0; j < G; ++j) sc[j] = make_float2(0.f, 0.f);
#pragma unroll
            for (int c = 0; c < kChunks; ++c) {
                const int half = (D == 128) ? hh : 0;
                const int cin = (D == 128) ? c : hh * kChunks + c;
                const uint4 kv4 = *reinterpret_cast<const uint4*>(kpg + half * 2048 + r * 128 + ((cin ^ (r & 7)) << 4));
                const float2 k2[4] = {make_float2(bf_lo(kv4.x), bf_hi(kv4.x)), make_float2(bf_lo(kv4.y), bf_hi(kv4.y)),
                                      make_float2(bf_lo(kv4.z), bf_hi(kv4.z)), make_float2(bf_lo(kv4.w), bf_hi(kv4.w))};
                const int d0 = hh * (D / 2) + c * 8;
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    if (j < g) {
                        const float4 qa = *reinterpret_cast<const float4*>(qf + j * D + d0);
                        const float4 qb = *reinterpret_cast<const float4*>(qf + j * D + d0 + 4);
                        float2 t = sc[j];
                        t = ffma2(make_float2(qa.x, qa.y), k2[0], t);
                        t = ffma2(make_float2(qa.z, qa.w), k2[1], t);
                        t = ffma2(make_float2(qb.x, qb.y), k2[2], t);
                        t = ffma2(make_float2(qb.z, qb.w), k2[3], t);
                        sc[j] = t;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < G; ++j) {
                if (j < g) {
                    float x = sc[j].x + sc[j].y;
                    x += __shfl_xor_sync(0xffffffffu, x, 16);
                    x = r < valid_rows ? x * sl2 : -CUDART_INF_F;
                    float mx = x;
                    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
                    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
                    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
                    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
                    const float m_new = fmaxf(m_run[j], mx);
                    const float corr = ex2(m_run[j] - m_new);
                    const float pr = ex2(x - m_new);
                    m_run[j] = m_new;
                    l_lane[j] = l_lane[j] * corr + (hh == 0 ? pr : 0.f);
#pragma unroll
                    for (int e = 0; e < kDimsPerLane / 2; ++e) acc[j][e] = make_float2(acc[j][e].x * corr, acc[j][e].y * corr);
                    if (hh == 0) s.pbuf[j][r] = pr;
                }
            }
            __syncwarp();
            // ---- PV: lane owns dims [lane*kDimsPerLane, +kDimsPerLane) ----
            const int vh = (D == 128) ? (lane >> 4) : 0;
            const int vbyte = (D == 128) ? ((lane & 15) * 8) : (lane * 4);
#pragma unroll
            for (int r4 = 0; r4 < 4; ++r4) {
                float4 p4[G]; // probabilities of rows 4*r4 .. 4*r4+3, one broadcast LDS.128 per head
#pragma unroll
                for (int j = 0; j < G; ++j)
                    if (j < g) p4[j] = *reinterpret_cast<const float4*>(&s.pbuf[j][r4 * 4]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int rr = r4 * 4 + q;
                    if (rr < valid_rows) {
                        const uint8_t* src = vpg + vh * 2048 + rr * 128 + ((((vbyte >> 4) ^ (rr & 7)) << 4) | (vbyte & 15));
                        float2 vv[kDimsPerLane / 2];
                        if constexpr (kDimsPerLane == 4) {
                            const uint2 uv = *reinterpret_cast<const uint2*>(src);
                            vv[0] = make_float2(bf_lo(uv.x), bf_hi(uv.x));
                            vv[1] = make_float2(bf_lo(uv.y), bf_hi(uv.y));
                        } else {
                            const uint32_t uv = *reinterpret_cast<const uint32_t*>(src);
                            vv[0] = make_float2(bf_lo(uv), bf_hi(uv));
                        }
#pragma unroll
                        for (int j = 0; j < G; ++j) {
                            if (j < g) {
                                const float pj = q == 0 ? p4[j].x : q == 1 ? p4[j].y : q == 2 ? p4[j].z : p4[j].w;
#pragma unroll
                                for (int e = 0; e < kDimsPerLane / 2; ++e)
                                    acc[j][e] = ffma2(make_float2(pj, pj), vv[e], acc[j][e]);
                            }
                        }
                    }
                }
            }
            __syncwarp(); // stage and pbuf reads done before they are overwritten
            ++consumed;
            issue_one();
        }
        // ---------------- end of a unit: normalise or publish a split partial ----------------
        float l_tot[G];
#pragma unroll
        for (int j = 0; j < G; ++j) {
            float lsum = l_lane[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
            l_tot[j] = lsum;
        }
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out) +
                             (static_cast<size_t>(sp.query_start) * p.n_head + static_cast<size_t>(w.kvh) * g) * D;
        const int d0 = lane * kDimsPerLane;
        if (w.n_parts <= 1) {
#pragma unroll
            for (int j = 0; j < G; ++j)
                if (j < g) {
                    const float inv = 1.f / l_tot[j];
#pragma unroll
                    for (int e = 0; e < kDimsPerLane / 2; ++e) {
                        out[static_cast<size_t>(j) * D + d0 + 2 * e] = __float2bfloat16_rn(acc[j][e].x * inv);
                        out[static_cast<size_t>(j) * D + d0 + 2 * e + 1] = __float2bfloat16_rn(acc[j][e].y * inv);
                    }
                }
        } else {
            const int part = w.part_base + w.part_idx;
#pragma unroll
            for (int j = 0; j < G; ++j)
                if (j < g) {
#pragma unroll
                    for (int e = 0; e < kDimsPerLane / 2; ++e) {
                        p.part_o[(static_cast<size_t>(part) * g + j) * D + d0 + 2 * e] = acc[j][e].x;
                        p.part_o[(static_cast<size_t>(part) * g + j) * D + d0 + 2 * e + 1] = acc[j][e].y;
                    }
                    if (lane == 0) {
                        p.part_ml[(static_cast<size_t>(part) * g + j) * 2 + 0] = m_run[j];
                        p.part_ml[(static_cast<size_t>(part) * g + j) * 2 + 1] = l_tot[j];
                    }
                }
            __threadfence();
            __syncwarp();
            int last = 0;
            if (lane == 0) last = atomicAdd(&p.counters[w.group], 1) == w.n_parts - 1;
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last) {
                __threadfence();
#pragma unroll
                for (int j = 0; j < G; ++j)
                    if (j < g) {
                        float M = -CUDART_INF_F;
                        for (int q = 0; q < w.n_parts; ++q)
                            M = fmaxf(M, __ldcg(&p.part_ml[(static_cast<size_t>(w.part_base + q) * g + j) * 2]));
                        float L = 0.f, O[kDimsPerLane];
#pragma unroll
                        for (int e = 0; e < kDimsPerLane; ++e) O[e] = 0.f;
                        for (int q = 0; q < w.n_parts; ++q) {
                            const size_t b = static_cast<size_t>(w.part_base + q) * g + j;
                            const float f = ex2(__ldcg(&p.part_ml[b * 2]) - M);
                            L += f * __ldcg(&p.part_ml[b * 2 + 1]);
#pragma unroll
                            for (int e = 0; e < kDimsPerLane; ++e) O[e] += f * __ldcg(&p.part_o[b * D + d0 + e]);
                        }
                        const float inv = 1.f / L;
#pragma unroll
                        for (int e = 0; e < kDimsPerLane; ++e)
                            out[static_cast<size_t>(j) * D + d0 + e] = __float2bfloat16_rn(O[e] * inv);
                    }
                if (lane == 0) p.counters[w.group] = 0; // self-reset for the next launch
            }
        }
        ++con_unit;
    }
    // retire: the last warp of the launch resets the queue for the next launch
    if (lane == 0) {
        const int total = static_cast<int>(gridDim.x) * kWarps;
        if (atomicAdd(&queue[1], 1) == total - 1) {
            queue[0] = 0;
            queue[1] = 0;
            __threadfence();
        }
    }
}

template <int D, int G>
void launch_decode_t(const AttnParams& p, const CUtensorMap* maps, cudaStream_t st) {
    const size_t smem = sizeof(DecWarp<D, G>) * dec_warps<D, G>() + 1024;
    static std::once_flag attr[kMaxDevices];
    set_smem_once(attr, attn_decode_kernel<D, G>, smem, "cudaFuncSetAttribute(decode smem)");
    const int grid = std::max(1, std::min(device_sms(), (p.n_items + dec_warps<D, G>() - 1) / dec_warps<D, G>()));
    attn_decode_kernel<D, G><<<grid, dec_warps<D, G>() * 32, smem, st>>>(maps[1], maps[2], p);
    cuda_check(cudaGetLastError(), "attn_decode launch");
    count_launch();
}

template <int D>
void launch_decode_d(const AttnParams& p, const CUtensorMap* maps, cudaStream_t st) {
    const int g = p.group;
    if (g <= 1) launch_decode_t<D, 1>(p, maps, st);
    else if (g <= 2) launch_decode_t<D, 2>(p, maps, st);
    else if (g <= 4) launch_decode_t<D, 4>(p, maps, st);
    else if (g <= 8) launch_decode_t<D, 8>(p, maps, st);
    else launch_decode_t<D, 16>(p, maps, st);
}

} // namespace

bool decode_supports(int head_size, int chunk, int group) {
    return (head_size == 64 || head_size == 128) && chunk == 16 && group >= 1 && group <= kMaxGroup;
}

void launch_attn_decode(const AttnParams& p, const pb_attn_shape& shape, Sm100Cache& cache, int64_t total_tokens,
                        cudaStream_t stream) {
    if (p.n_items <= 0) return;
    // GQA groups of 3..16 heads at d = 128 go to the tcgen05 decode kernel (attn_decode_tc.cu)
    if (decode_tc_supports(shape.head_size, shape.chunk_size, p.group)) {
        launch_attn_decode_tc(p, shape, cache, total_tokens, stream);
        return;
    }
    sm100_prepare_maps(p, shape, cache, total_tokens);
    const auto* maps = reinterpret_cast<const CUtensorMap*>(cache.maps);
    if (shape.head_size == 128) launch_decode_d<128>(p, maps, stream);
    else launch_decode_d<64>(p, maps, stream);
}

} // namespace pb
