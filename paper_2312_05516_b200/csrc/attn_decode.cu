// Single-token (decode) spans: memory-bound split-KV SIMT path.
//
// Semantics: single_token_attention, /root/reference/proj/src/attention.cpp:134-188 (one
// query row per head against the whole context; the same as the multi-token path with
// q_len = 1).  B200 design:
//   * one work item = (span, kv head, page range); long contexts are split across CTAs and
//     the partial (max, sum, unnormalised O) of each split is merged inside the same launch by
//     the last-arriving split (atomic ticket, self-resetting);
//   * all `group` query heads of the kv head are served by the same K/V bytes (each KV byte is
//     read from HBM once);
//   * each of the 4 warps owns a private 3-stage ring of pages in shared memory, filled by TMA
//     ({64 dims, 1 kv head, 16 rows} boxes, SWIZZLE_128B => conflict-free row reads), and
//     walks pages w, w+4, ...; the 4 warps' partials are merged through shared memory;
//   * scores: lane = (row, 64-dim half), halves combined with one shuffle, page max with
//     4 xor-shuffles per head; P broadcast through shared memory; lanes own 4 (or 2) output
//     dims for the PV update.
#include "attn_internal.hpp"
#include "pb_common.hpp"
#include "sm100_attn.hpp"
#include "sm100_ptx.cuh"

#include <cuda.h>
#include <cuda_bf16.h>
#include <math_constants.h>

#include <algorithm>

namespace pb {

namespace {

using namespace pb::sm100;

constexpr int kDecWarps = 4;
constexpr int kDecStages = 3;
constexpr int kMaxGroup = 16;

template <int D, int G>
struct __align__(1024) DecSmem {
    static constexpr int KH = D / 64 > 0 ? D / 64 : 1;
    static constexpr int kPageBytes = 16 * D * 2;             // one kv head, 16 rows
    static_assert(G * D * 4 <= kDecStages * 2 * kPageBytes, "merge buffer aliases the warp's ring");
    // [warp][stage][K|V][half][row][128B]; after the page loop each warp's ring is reused
    // as its fp32 O partial [G][D] for the cross-warp merge
    uint8_t kv[kDecWarps][kDecStages][2][kPageBytes];
    float q[G][D];                                            // query rows (fp32)
    float pbuf[kDecWarps][G][16];                             // per-warp page probabilities
    float m[kDecWarps][G];
    float l[kDecWarps][G];
    uint64_t full[kDecWarps][kDecStages];
    int last;
    __device__ float* o(int warp) { return reinterpret_cast<float*>(kv[warp][0][0]); }
};

__device__ __forceinline__ float bf_lo(uint32_t x) { return __uint_as_float(x << 16); }
__device__ __forceinline__ float bf_hi(uint32_t x) { return __uint_as_float(x & 0xffff0000u); }

template <int D, int kMaxGroup>
__global__ void __launch_bounds__(kDecWarps * 32, 2)
    attn_decode_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                       const AttnParams p) {
    constexpr int KH = DecSmem<D, kMaxGroup>::KH;
    constexpr int kChunks = D / 16;  // 16B chunks per half-row handled by one lane (D/2 dims)
    constexpr int kDimsPerLane = D / 32;
    extern __shared__ uint8_t smem_raw[];
    // align with pointer arithmetic on the __shared__ array so loads stay LDS (not generic LD)
    DecSmem<D, kMaxGroup>& s = *reinterpret_cast<DecSmem<D, kMaxGroup>*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const WorkItem w = p.items[blockIdx.x];
    const SpanDev sp = p.spans[w.span];
    const int g = p.group;
    const int32_t* table = p.block_tables + sp.bt_off;
    const int page0 = w.kv_begin >> 4;
    const int n_pages = (w.kv_end - w.kv_begin + 15) >> 4;
    const float sl2 = p.scale_log2;

    if (lane == 0) {
        for (int st = 0; st < kDecStages; ++st) mbar_init(&s.full[warp][st], 1);
        mbar_fence_init();
    }
    // query rows of the group, fp32
    {
        const __nv_bfloat16* q = static_cast<const __nv_bfloat16*>(p.q) +
                                 (static_cast<size_t>(sp.query_start) * p.n_head + static_cast<size_t>(w.kvh) * g) * D;
        for (int e = threadIdx.x; e < g * D; e += blockDim.x) s.q[e / D][e % D] = __bfloat162float(q[e]);
    }
    __syncthreads();

    // ---- per-warp page ring ----
    const uint32_t page_tx = 2u * KH * 16u * 128u;
    auto issue = [&](int local_page, int stage) {
        const int row = table[page0 + local_page] * 16;
        uint8_t* dst = s.kv[warp][stage][0];
        mbar_arrive_expect_tx(&s.full[warp][stage], page_tx);
        for (int h = 0; h < KH; ++h) {
            tma_load_3d(dst + h * 2048, &tm_k, &s.full[warp][stage], h * 64, w.kvh, row);
            tma_load_3d(dst + DecSmem<D, kMaxGroup>::kPageBytes + h * 2048, &tm_v, &s.full[warp][stage], h * 64, w.kvh, row);
        }
    };
    int my_pages = 0;
    for (int lp = warp; lp < n_pages; lp += kDecWarps) ++my_pages;
    if (lane == 0)
        for (int i = 0; i < kDecStages - 1 && i < my_pages; ++i) issue(warp + i * kDecWarps, i);

    float m_run[kMaxGroup], l_lane[kMaxGroup], acc[kMaxGroup][kDimsPerLane];
#pragma unroll
    for (int j = 0; j < kMaxGroup; ++j) {
        m_run[j] = -CUDART_INF_F;
        l_lane[j] = 0.f;
#pragma unroll
        for (int e = 0; e < kDimsPerLane; ++e) acc[j][e] = 0.f;
    }
    const int r = lane & 15;        // page row scored by this lane
    const int hh = lane >> 4;       // which half of the dims
    for (int i = 0; i < my_pages; ++i) {
        const int stage = i % kDecStages;
        if (lane == 0 && i + kDecStages - 1 < my_pages) {
            fence_proxy_async_smem();
            issue(warp + (i + kDecStages - 1) * kDecWarps, (i + kDecStages - 1) % kDecStages);
        }
        mbar_wait(&s.full[warp][stage], (i / kDecStages) & 1);
        const uint8_t* kpg = s.kv[warp][stage][0];
        const uint8_t* vpg = s.kv[warp][stage][1];
        const int pos0 = w.kv_begin + (warp + i * kDecWarps) * 16;
        const int valid_rows = min(16, w.kv_end - pos0);
        // ---- scores: lane (r, hh) dots its row's half with every query head ----
        float sc[kMaxGroup], sc2[kMaxGroup]; // two chains per head (latency, small groups)
#pragma unroll
        for (int j = 0; j < kMaxGroup; ++j) sc[j] = sc2[j] = 0.f;
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
            // dims hh*(D/2) + c*8 .. +8 ; for D=128 that is half hh, 16B chunk c of the row
            int half, cin;
            if (D == 128) { half = hh; cin = c; }
            else { half = 0; cin = hh * (kChunks) + c; }
            const uint4 kv4 = *reinterpret_cast<const uint4*>(kpg + half * 2048 + r * 128 + ((cin ^ (r & 7)) << 4));
            const float k8[8] = {bf_lo(kv4.x), bf_hi(kv4.x), bf_lo(kv4.y), bf_hi(kv4.y),
                                 bf_lo(kv4.z), bf_hi(kv4.z), bf_lo(kv4.w), bf_hi(kv4.w)};
            const int d0 = hh * (D / 2) + c * 8;
#pragma unroll
            for (int j = 0; j < kMaxGroup; ++j) {
                if (j < g) {
                    const float4 qa = *reinterpret_cast<const float4*>(&s.q[j][d0]);
                    const float4 qb = *reinterpret_cast<const float4*>(&s.q[j][d0 + 4]);
                    float t = sc[j], u = sc2[j];
                    t = fmaf(qa.x, k8[0], t);
                    u = fmaf(qa.y, k8[1], u);
                    t = fmaf(qa.z, k8[2], t);
                    u = fmaf(qa.w, k8[3], u);
                    t = fmaf(qb.x, k8[4], t);
                    u = fmaf(qb.y, k8[5], u);
                    t = fmaf(qb.z, k8[6], t);
                    u = fmaf(qb.w, k8[7], u);
                    sc[j] = t;
                    sc2[j] = u;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kMaxGroup; ++j) {
            if (j < g) {
                float x = sc[j] + sc2[j];
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
                for (int e = 0; e < kDimsPerLane; ++e) acc[j][e] *= corr;
                if (hh == 0) s.pbuf[warp][j][r] = pr;
            }
        }
        __syncwarp();
        // ---- PV: lane owns dims [lane*kDimsPerLane, +kDimsPerLane) ----
        const int vh = (D == 128) ? (lane >> 4) : 0;
        const int vbyte = (D == 128) ? ((lane & 15) * 8) : (lane * 4); // byte offset inside the 128 B row
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) {
            if (rr < valid_rows) {
                const uint8_t* vrow = vpg + vh * 2048 + rr * 128;
                const int chunk16 = vbyte >> 4;
                const uint8_t* src = vrow + (((chunk16 ^ (rr & 7)) << 4) | (vbyte & 15));
                float vv[kDimsPerLane];
                if (kDimsPerLane == 4) {
                    const uint2 u = *reinterpret_cast<const uint2*>(src);
                    vv[0] = bf_lo(u.x);
                    vv[1] = bf_hi(u.x);
                    vv[2] = bf_lo(u.y);
                    vv[3] = bf_hi(u.y);
                } else {
                    const uint32_t u = *reinterpret_cast<const uint32_t*>(src);
                    vv[0] = bf_lo(u);
                    vv[1] = bf_hi(u);
                }
#pragma unroll
                for (int j = 0; j < kMaxGroup; ++j) {
                    if (j < g) {
                        const float pj = s.pbuf[warp][j][rr];
#pragma unroll
                        for (int e = 0; e < kDimsPerLane; ++e) acc[j][e] = fmaf(pj, vv[e], acc[j][e]);
                    }
                }
            }
        }
        __syncwarp();
    }
    // ---- merge the 4 warps (shared memory) ----
    __syncwarp();
    float* o_mine = s.o(warp);
#pragma unroll
    for (int j = 0; j < kMaxGroup; ++j) {
        if (j < g) {
            float lsum = l_lane[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
            if (lane == 0) {
                s.m[warp][j] = m_run[j];
                s.l[warp][j] = lsum;
            }
#pragma unroll
            for (int e = 0; e < kDimsPerLane; ++e) o_mine[j * D + lane * kDimsPerLane + e] = acc[j][e];
        }
    }
    __syncthreads();
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out) +
                         (static_cast<size_t>(sp.query_start) * p.n_head + static_cast<size_t>(w.kvh) * g) * D;
    const bool split = w.n_parts > 1;
    for (int e = threadIdx.x; e < g * D; e += blockDim.x) {
        const int j = e / D, d = e % D;
        float M = -CUDART_INF_F;
#pragma unroll
        for (int q = 0; q < kDecWarps; ++q) M = fmaxf(M, s.m[q][j]);
        float L = 0.f, O = 0.f;
#pragma unroll
        for (int q = 0; q < kDecWarps; ++q) {
            const float f = ex2(s.m[q][j] - M);
            L += f * s.l[q][j];
            O += f * s.o(q)[j * D + d];
        }
        if (!split) {
            out[static_cast<size_t>(j) * D + d] = __float2bfloat16_rn(O / L);
        } else {
            const int part = w.part_base + w.part_idx;
            p.part_o[(static_cast<size_t>(part) * g + j) * D + d] = O;
            if (d == 0) {
                p.part_ml[(static_cast<size_t>(part) * g + j) * 2 + 0] = M;
                p.part_ml[(static_cast<size_t>(part) * g + j) * 2 + 1] = L;
            }
        }
    }
    if (!split) return;
    // ---- split-KV merge by the last-arriving part (same launch) ----
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int prev = atomicAdd(&p.counters[w.group], 1);
        s.last = (prev == w.n_parts - 1);
    }
    __syncthreads();
    if (!s.last) return;
    __threadfence();
    for (int e = threadIdx.x; e < g * D; e += blockDim.x) {
        const int j = e / D, d = e % D;
        float M = -CUDART_INF_F;
        for (int q = 0; q < w.n_parts; ++q)
            M = fmaxf(M, __ldcg(&p.part_ml[(static_cast<size_t>(w.part_base + q) * g + j) * 2]));
        float L = 0.f, O = 0.f;
        for (int q = 0; q < w.n_parts; ++q) {
            const size_t b = static_cast<size_t>(w.part_base + q) * g + j;
            const float f = ex2(__ldcg(&p.part_ml[b * 2]) - M);
            L += f * __ldcg(&p.part_ml[b * 2 + 1]);
            O += f * __ldcg(&p.part_o[b * D + d]);
        }
        out[static_cast<size_t>(j) * D + d] = __float2bfloat16_rn(O / L);
    }
    if (threadIdx.x == 0) p.counters[w.group] = 0; // self-reset for the next launch
}

template <int D, int G>
void launch_decode_t(const AttnParams& p, const CUtensorMap* maps, cudaStream_t st) {
    const size_t smem = sizeof(DecSmem<D, G>) + 1024;
    static bool attr = false;
    if (!attr) {
        cuda_check(cudaFuncSetAttribute(attn_decode_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)),
                   "cudaFuncSetAttribute(decode smem)");
        attr = true;
    }
    attn_decode_kernel<D, G><<<p.n_items, kDecWarps * 32, smem, st>>>(maps[1], maps[2], p);
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
    sm100_prepare_maps(p, shape, cache, total_tokens);
    const auto* maps = reinterpret_cast<const CUtensorMap*>(cache.maps);
    if (shape.head_size == 128) launch_decode_d<128>(p, maps, stream);
    else launch_decode_d<64>(p, maps, stream);
}

} // namespace pb
