// Single-token (decode) spans with a GQA group of 1..16 query heads: tcgen05 split-KV path.
//
// Semantics: single_token_attention, /root/reference/proj/src/attention.cpp:134-188 (one query
// row per head against the whole context).  Why tensor cores for a memory-bound op: with G
// query heads per kv head every K/V byte feeds 2*G flops; at G = 8 the SIMT path needs ~1000
// issue slots per 8 KB page and cannot keep up with HBM (profiles/r1_variants.md).  Here the
// arithmetic is two tiny MMAs per 128-row kv tile and the SMs only stream bytes:
//   * one work unit = (span, kv head, page range), the same split-KV units as the SIMT path,
//     taken from a global ticket in LPT order by the TMA warp and handed to the other roles
//     through a shared ring; partials of split spans are merged by the last-arriving unit;
//   * S^T = K . Q^T   (M = 128 kv rows, N = 16 padded query heads, K = D): the kv rows are the
//     TMEM lanes, so every softmax thread owns one kv row and all heads of it;
//   * O^T += V^T . P^T (M = D, N = 16, K = 128 kv rows): V straight from the TMA-staged page
//     tile as an MN-major A operand, P^T (bf16) written by the softmax threads into a K-major
//     SWIZZLE_128B B tile;
//   * a 3-stage K/V ring of 128-row tiles (8 pages x 2 halves x K,V TMA boxes) runs ahead
//     across unit boundaries; S is double-buffered in TMEM so S(j+1) overlaps softmax(j);
//   * per tile, the per-head max is a warp xor-reduction plus a 4-warp exchange in shared
//     memory; O is rescaled lazily (only when a head's max grows by more than 2^8).
// Warp roles (192 threads, one CTA per SM): warp 0 TMA producer, warp 1 MMA issuer,
// warps 2..5 softmax + epilogue (TMEM lane quadrants 2, 3, 0, 1).
#pragma once

#include "attn_internal.hpp"
#include "pb_common.hpp"
#include "sm100_attn.hpp"
#include "sm100_ptx.cuh"

#include <cuda.h>
#include <cuda_bf16.h>
#include <math_constants.h>

#include <algorithm>

namespace pb {
namespace dtc {

using namespace pb::sm100;

constexpr int kDtThreads = 224;     // TMA K warp, MMA warp, 4 softmax warps, TMA V warp
constexpr int kKvRows = 128;         // kv rows per tile
constexpr int kN = 16;               // padded query heads (N of both MMAs)
#ifndef PB_DEC_K_STAGES
#define PB_DEC_K_STAGES 3
#endif
#ifndef PB_DEC_V_STAGES
#define PB_DEC_V_STAGES 3
#endif
constexpr int kKStages = PB_DEC_K_STAGES;  // K ring depth
constexpr int kVStages = PB_DEC_V_STAGES;  // V ring depth
constexpr int kRing = 4;             // work-unit ring
constexpr uint32_t kTmemCols = 64;   // S^T buffers [0,16) [16,32), O^T [32,48)
constexpr uint32_t kColO = 32;
constexpr float kThr = 8.f;          // lazy rescale threshold (log2 domain)
constexpr uint32_t kHalf = kKvRows * 128;          // one 64-dim half of a kv tile (16 KB)
constexpr uint32_t kStageTx = 2u * kHalf;          // one of K or V, two halves (D = 128)

struct __align__(1024) DtSmem {
    uint8_t k[kKStages][2][kHalf];   // [stage][half][row][128 B], SW128 K-major (A of S^T)
    uint8_t v[kVStages][2][kHalf];   // same layout, read as the MN-major A of O^T
    uint8_t q[2][2][kN * 128];      // [unit parity][half][head][128 B], SW128 K-major (B of S^T)
    uint8_t pt[2][2][kN * 128];     // [tile parity][kv half][head][128 B], SW128 K-major (B of O^T)
    float red[2][4][kN];            // [tile parity][warp quadrant][head] max exchange
    float redl[4][kN];              // [warp quadrant][head] epilogue sum exchange
    int32_t flag;
    // separate K and V rings with their own producer warps: a K stage is free as soon as S
    // has read it, so K runs further ahead and more bytes are in flight per CTA
    uint64_t k_full[kKStages], k_empty[kKStages], v_full[kVStages], v_empty[kVStages];
    uint64_t q_full[2], q_empty[2];
    // p_full / pv_done per tile parity: the softmax may run one tile ahead of the MMA warp's
    // p_full wait (it no longer waits for PV(j-1) before releasing P(j)), so a single barrier
    // could be lapped; per parity every wait is at most one phase behind
    uint64_t s_full[2], p_full[2], pv_done[2], o_empty;
    uint64_t item_full[kRing], item_empty[kRing];
    uint64_t drain;                 // MMA issuer: every commit of the pass has landed
    int32_t item_ring[kRing];
    uint32_t tmem_base;
};

__device__ __forceinline__ void bar_softmax() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
// bar_softmax with an OR-reduction of one predicate over the four softmax warps
__device__ __forceinline__ bool bar_softmax_any(bool v) {
    uint32_t r;
    asm volatile("{\n\t.reg .pred pi, po;\n\t"
                 "setp.ne.u32 pi, %1, 0;\n\t"
                 "bar.red.or.pred po, 1, 128, pi;\n\t"
                 "selp.u32 %0, 1, 0, po;\n\t}"
                 : "=r"(r)
                 : "r"(static_cast<uint32_t>(v))
                 : "memory");
    return r != 0;
}

#ifndef PB_TILE_TRACE
#define PB_TILE_TRACE 0
#endif
// Diagnostics build only (-DPB_TILE_TRACE=1): per-tile clock64 stamps of the first 8 CTAs, in
// the layout of sm100_attn.cu's tile trace (roles: 0 softmax, 2 MMA, 3 K producer, 4 V
// producer); scripts/trace_decode.py reads them.  Compiles to nothing by default.
__device__ __forceinline__ unsigned long long* dt_trace_slot(unsigned long long* tr, int role, uint32_t ev) {
    if (!PB_TILE_TRACE || !tr || blockIdx.x >= 8 || ev >= 1024) return nullptr;
    return tr + 148 * 2 * 4 + ((static_cast<size_t>(blockIdx.x) * 6 + role) * 1024 + ev) * 8;
}
__device__ __forceinline__ unsigned long long dt_clk() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    return t;
}

// max over the warp in one instruction (sm_100a redux.sync on f32)
__device__ __forceinline__ float warp_max_f32(float v) {
    float r;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
    return r;
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void st_shared_u16(uint32_t addr, uint16_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void st_shared_zero16(uint32_t addr) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(addr), "r"(0) : "memory");
}

__device__ __forceinline__ int unit_tiles(const WorkItem& w, int chunk) {
    const int np = (w.kv_end - w.kv_begin + chunk - 1) / chunk;
    return (np * chunk + kKvRows - 1) / kKvRows;
}

// thread 0 only: the decode pipeline's barriers
__device__ __forceinline__ void decode_cta_init(DtSmem& s) {
    for (int i = 0; i < kKStages; ++i) {
        mbar_init(&s.k_full[i], 1);
        mbar_init(&s.k_empty[i], 1);
    }
    for (int i = 0; i < kVStages; ++i) {
        mbar_init(&s.v_full[i], 1);
        mbar_init(&s.v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
        mbar_init(&s.q_full[i], 1);
        mbar_init(&s.q_empty[i], 1);
        mbar_init(&s.s_full[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
        mbar_init(&s.p_full[i], 128);
        mbar_init(&s.pv_done[i], 1);
    }
    mbar_init(&s.o_empty, 128);
    for (int i = 0; i < kRing; ++i) {
        mbar_init(&s.item_full[i], 1);
        mbar_init(&s.item_empty[i], 1 + 4 + 1); // MMA thread + 4 softmax warps + V producer
    }
    mbar_init(&s.drain, 1);
}

// thread 0 only, pipeline drained: release the barriers' memory for another layout
__device__ __forceinline__ void decode_cta_inval(DtSmem& s) {
    for (int i = 0; i < kKStages; ++i) {
        mbar_inval(&s.k_full[i]);
        mbar_inval(&s.k_empty[i]);
    }
    for (int i = 0; i < kVStages; ++i) {
        mbar_inval(&s.v_full[i]);
        mbar_inval(&s.v_empty[i]);
    }
    for (int i = 0; i < 2; ++i) {
        mbar_inval(&s.q_full[i]);
        mbar_inval(&s.q_empty[i]);
        mbar_inval(&s.s_full[i]);
    }
    for (int i = 0; i < 2; ++i) {
        mbar_inval(&s.p_full[i]);
        mbar_inval(&s.pv_done[i]);
    }
    mbar_inval(&s.o_empty);
    for (int i = 0; i < kRing; ++i) {
        mbar_inval(&s.item_full[i]);
        mbar_inval(&s.item_empty[i]);
    }
    mbar_inval(&s.drain);
}

// One CTA of the decode pipeline.  Roles: warp w_prod = TMA producer of q and K (and the
// unit ticket), w_prodv = TMA producer of V, w_mma = MMA issuer, w_sm0 .. w_sm0+3 = softmax +
// epilogue (must cover the four TMEM lane quadrants); other warps fall through.  Units come from `items` through the global `ticket`.  TMEM columns
// [tmem, tmem + 48) are used.
template <int G>
__device__ __forceinline__ void decode_cta_run(DtSmem& s, const uint32_t tmem, const CUtensorMap* tm_q,
                                               const CUtensorMap* tm_k, const CUtensorMap* tm_v, const AttnParams& p,
                                               const WorkItem* items, const int n_items, int* ticket, const int w_prod,
                                               const int w_mma, const int w_sm0, const int w_prodv) {
    constexpr int D = 128;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int g = p.group;
    const int chunk = p.chunk;
    const int ppt = kKvRows / chunk;
    if (warp == w_prod) {
        // ============================ TMA producer ============================
        if (elect_one()) {
            int stage = 0;
            uint32_t kph = 0;
            const int oob_row = p.n_slots * chunk;
            int it = 0;
            uint32_t kt_ev = 0;
            for (;; ++it) {
                const int slot = it % kRing;
                if (it >= kRing) mbar_wait(&s.item_empty[slot], ((it / kRing) - 1) & 1);
                int item = atomicAdd(ticket, 1);
                if (item >= n_items) item = -1;
                s.item_ring[slot] = item;
                mbar_arrive(&s.item_full[slot]);
                if (item < 0) break;
                const WorkItem w = items[item];
                const SpanDev sp = p.spans[w.span];
                const int qb = it & 1;
                if (it >= 2) mbar_wait(&s.q_empty[qb], ((it >> 1) - 1) & 1);
                mbar_arrive_expect_tx(&s.q_full[qb], 2u * 128u * static_cast<uint32_t>(g));
                for (int h = 0; h < 2; ++h)
                    tma_load_3d(s.q[qb][h], tm_q, &s.q_full[qb], h * 64, w.kvh * g, sp.query_start);
                const int32_t* table = p.block_tables + sp.bt_off + w.kv_begin / chunk;
                const int np = (w.kv_end - w.kv_begin + chunk - 1) / chunk;
                const int nt = (np + ppt - 1) / ppt;
                for (int j = 0; j < nt; ++j) {
                    // the tile's block-table entries in one round trip, before the ring wait
                    int rows[16];
#pragma unroll
                    for (int pg = 0; pg < 16; ++pg) {
                        const int page = j * ppt + pg;
                        rows[pg] = (pg < ppt && page < np) ? __ldg(table + page) * chunk : oob_row;
                    }
                    unsigned long long* tk = dt_trace_slot(p.trace, 3, kt_ev++);
                    if (tk) tk[0] = dt_clk();
                    mbar_wait(&s.k_empty[stage], kph ^ 1);
                    if (tk) tk[1] = dt_clk();
                    mbar_arrive_expect_tx(&s.k_full[stage], kStageTx);
#pragma unroll
                    for (int pg = 0; pg < 16; ++pg)
                        if (pg < ppt)
                            for (int h = 0; h < 2; ++h)
                                tma_load_3d(s.k[stage][h] + pg * chunk * 128, tm_k, &s.k_full[stage], h * 64, w.kvh, rows[pg]);
                    if (++stage == kKStages) { stage = 0; kph ^= 1; }
                }
            }
        }
    } else if (warp == w_prodv) {
        // ============================ TMA producer (V) ========================
        if (elect_one()) {
            int stage = 0;
            uint32_t vph = 0;
            const int oob_row = p.n_slots * chunk;
            uint32_t vt_ev = 0;
            for (int it = 0;; ++it) {
                const int slot = it % kRing;
                mbar_wait(&s.item_full[slot], (it / kRing) & 1);
                const int item = *reinterpret_cast<volatile int32_t*>(&s.item_ring[slot]);
                mbar_arrive(&s.item_empty[slot]);
                if (item < 0) break;
                const WorkItem w = items[item];
                const SpanDev sp = p.spans[w.span];
                const int32_t* table = p.block_tables + sp.bt_off + w.kv_begin / chunk;
                const int np = (w.kv_end - w.kv_begin + chunk - 1) / chunk;
                const int nt = (np + ppt - 1) / ppt;
                for (int j = 0; j < nt; ++j) {
                    int rows[16];
#pragma unroll
                    for (int pg = 0; pg < 16; ++pg) {
                        const int page = j * ppt + pg;
                        rows[pg] = (pg < ppt && page < np) ? __ldg(table + page) * chunk : oob_row;
                    }
                    unsigned long long* tv = dt_trace_slot(p.trace, 4, vt_ev++);
                    if (tv) tv[0] = dt_clk();
                    mbar_wait(&s.v_empty[stage], vph ^ 1);
                    if (tv) tv[1] = dt_clk();
                    mbar_arrive_expect_tx(&s.v_full[stage], kStageTx);
#pragma unroll
                    for (int pg = 0; pg < 16; ++pg)
                        if (pg < ppt)
                            for (int h = 0; h < 2; ++h)
                                tma_load_3d(s.v[stage][h] + pg * chunk * 128, tm_v, &s.v_full[stage], h * 64, w.kvh, rows[pg]);
                    if (++stage == kVStages) { stage = 0; vph ^= 1; }
                }
            }
        }
    } else if (warp == w_mma) {
        // ============================ MMA issuer =============================
        if (elect_one()) {
            constexpr uint32_t idesc_s = umma_idesc_bf16(128, kN, false, false);
            constexpr uint32_t idesc_o = umma_idesc_bf16(128, kN, true, false);
            int stage = 0;   // K ring position (the tile S is issued for)
            uint32_t kph = 0;
            int vstage = 0;  // V ring position (the tile PV is issued for)
            uint32_t vph = 0;
            uint32_t T = 0; // tiles issued by this CTA (all units)
            auto issue_s = [&](int qb, uint32_t tile) {
                const uint64_t ad = umma_desc_sw128(smem_u32(s.k[stage][0]), 16, 1024);
                const uint64_t bd = umma_desc_sw128(smem_u32(s.q[qb][0]), 16, 1024);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t oa = ((kk >> 2) * kHalf + (kk & 3) * 32) >> 4;
                    const uint32_t ob = ((kk >> 2) * (kN * 128) + (kk & 3) * 32) >> 4;
                    umma_bf16_ss(tmem + (tile & 1) * kN, ad + oa, bd + ob, idesc_s, kk > 0);
                }
                umma_commit(&s.s_full[tile & 1]);
                umma_commit(&s.k_empty[stage]); // K is read by S only
                if (++stage == kKStages) { stage = 0; kph ^= 1; }
            };
            for (int it = 0;; ++it) {
                const int slot = it % kRing;
                mbar_wait(&s.item_full[slot], (it / kRing) & 1);
                const int item = *reinterpret_cast<volatile int32_t*>(&s.item_ring[slot]);
                mbar_arrive(&s.item_empty[slot]);
                if (item < 0) {
                    umma_commit(&s.drain); // the last commit arrivals land before barriers are reused
                    mbar_wait(&s.drain, 0);
                    break;
                }
                const WorkItem w = items[item];
                const int nt = unit_tiles(w, chunk);
                const int qb = it & 1;
                mbar_wait(&s.q_full[qb], (it >> 1) & 1);
                mbar_wait(&s.k_full[stage], kph);
                tc_fence_after();
                issue_s(qb, T);
                for (int j = 0; j < nt; ++j, ++T) {
                    unsigned long long* tm = dt_trace_slot(p.trace, 2, T);
                    if (tm) tm[0] = dt_clk();
                    if (j + 1 < nt) { // S(j+1) overlaps softmax(j)
                        mbar_wait(&s.k_full[stage], kph);
                        tc_fence_after();
                        issue_s(qb, T + 1);
                    }
                    if (tm) tm[1] = dt_clk();
                    mbar_wait(&s.p_full[T & 1], (T >> 1) & 1);
                    if (tm) tm[2] = dt_clk();
                    if (j == 0 && it > 0) mbar_wait(&s.o_empty, (it - 1) & 1);
                    mbar_wait(&s.v_full[vstage], vph);
                    if (tm) tm[3] = dt_clk();
                    tc_fence_after();
                    const uint64_t ad = umma_desc_sw128(smem_u32(s.v[vstage][0]), kHalf, 1024);
                    const uint64_t bd = umma_desc_sw128(smem_u32(s.pt[T & 1][0]), 16, 1024);
#pragma unroll
                    for (int kk = 0; kk < kKvRows / 16; ++kk) {
                        const uint32_t ob = ((kk >> 2) * (kN * 128) + (kk & 3) * 32) >> 4;
                        umma_bf16_ss(tmem + kColO, ad + kk * (2048 >> 4), bd + ob, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
                    }
                    umma_commit(&s.pv_done[T & 1]);
                    umma_commit(&s.v_empty[vstage]);
                    if (tm) {
                        tm[4] = dt_clk();
                        tm[6] = j;
                        tm[7] = item;
                    }
                    if (++vstage == kVStages) { vstage = 0; vph ^= 1; }
                }
                umma_commit(&s.q_empty[qb]);
            }
        }
    } else if (warp >= w_sm0 && warp < w_sm0 + 4) {
        // ===================== softmax + epilogue (4 warps) =====================
        const int quad = warp & 3;
        const int r = quad * 32 + lane;                     // kv row of the tile / output dim
        const uint32_t t_lane = tmem + (static_cast<uint32_t>(quad * 32) << 16);
        const float sl2 = p.scale_log2;
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out);
        uint32_t T = 0;
        // P^T element (head h, kv row r): kv half r/64, 16-B chunk ((r%64)/8) ^ (h%8), 2 B each
        const uint32_t pt_row = static_cast<uint32_t>((r >> 6) * (kN * 128) + (r & 7) * 2);
        const uint32_t pt_c16 = static_cast<uint32_t>((r & 63) >> 3);
        for (int it = 0;; ++it) {
            const int slot = it % kRing;
            mbar_wait(&s.item_full[slot], (it / kRing) & 1);
            const int item = *reinterpret_cast<volatile int32_t*>(&s.item_ring[slot]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.item_empty[slot]);
            if (item < 0) break;
            const WorkItem w = items[item];
            const SpanDev sp = p.spans[w.span];
            const int nt = unit_tiles(w, chunk);
            float m_run[G], l_thr[G];
#pragma unroll
            for (int h = 0; h < G; ++h) {
                m_run[h] = -CUDART_INF_F;
                l_thr[h] = 0.f;
            }
            for (int j = 0; j < nt; ++j, ++T) {
                unsigned long long* ts = (warp == w_sm0 && lane == 0) ? dt_trace_slot(p.trace, 0, T) : nullptr;
                if (ts) ts[0] = dt_clk();
                mbar_wait(&s.s_full[T & 1], (T >> 1) & 1);
                if (ts) ts[1] = dt_clk();
                tc_fence_after();
                uint32_t sr[16];
                tmem_ld16(t_lane + (T & 1) * kN, sr);
                tmem_ld_wait();
                const int kv = w.kv_begin + j * kKvRows + r;
                const bool valid = kv < w.kv_end;
                float x[G], mt[G];
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    x[h] = (valid && h < g) ? __uint_as_float(sr[h]) * sl2 : -CUDART_INF_F;
                    mt[h] = warp_max_f32(x[h]);
                }
                // The heads' maxima over the tile only matter when one grows past the lazy
                // threshold: a barrier OR-reduction asks whether any warp sees that; usually
                // none does and the 4-warp exchange is skipped (same results either way).
                bool want = false;
#pragma unroll
                for (int h = 0; h < G; ++h) want |= mt[h] > m_run[h] + kThr;
                bool rescale = false;
                float corr[G];
#pragma unroll
                for (int h = 0; h < G; ++h) corr[h] = 1.f;
                if (bar_softmax_any(want)) {
                    if (lane < G) {
                        float v = mt[0];
#pragma unroll
                        for (int h = 1; h < G; ++h) v = lane == h ? mt[h] : v;
                        s.red[T & 1][quad][lane] = v;
                    }
                    bar_softmax();
#pragma unroll
                    for (int h = 0; h < G; ++h) {
                        const float m4 = fmaxf(fmaxf(s.red[T & 1][0][h], s.red[T & 1][1][h]),
                                               fmaxf(s.red[T & 1][2][h], s.red[T & 1][3][h]));
                        const bool grow = m4 > m_run[h] + kThr; // uniform across the 128 threads
                        const float m_new = grow ? m4 : m_run[h];
                        corr[h] = grow ? ex2(m_run[h] - m_new) : 1.f;
                        rescale |= grow && j > 0;
                        m_run[h] = m_new;
                    }
                }
                if (ts) ts[2] = dt_clk();
                const uint32_t ptb = smem_u32(s.pt[T & 1][0]) + pt_row;
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    if (h < g) {
                        const float pr = valid ? ex2(x[h] - m_run[h]) : 0.f;
                        l_thr[h] = l_thr[h] * corr[h] + pr;
                        const __nv_bfloat16 b = __float2bfloat16_rn(pr);
                        st_shared_u16(ptb + h * 128 + ((pt_c16 ^ (h & 7)) << 4), *reinterpret_cast<const uint16_t*>(&b));
                    }
                }
                if (ts) ts[4] = dt_clk();
                if (!valid && j + 1 == nt) {
                    // rows past the unit's end in a fetched page may hold anything (stale or
                    // never-written pool rows): zero their V so 0 * NaN cannot reach O
                    const int stg = static_cast<int>(T % kVStages);
                    // V arrives on its own ring: wait until this tile's V landed before zeroing
                    // (its next reuse needs PV(T), so the parity wait is exact)
                    mbar_wait(&s.v_full[stg], (T / kVStages) & 1);
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int c = 0; c < 8; ++c) st_shared_zero16(smem_u32(s.v[stg][h]) + r * 128 + c * 16);
                }
                if (rescale) {
                    // O may be rescaled once PV(j-1) is complete.  S(j) landing already proves
                    // PV(j-2) complete (S(j) is issued after it), so this parity wait is exact;
                    // without a rescale nothing waits for PV(j-1) (P^T is double-buffered and
                    // its buffer's previous reader, PV(j-2), is done)
                    mbar_wait(&s.pv_done[(T - 1) & 1], ((T - 1) >> 1) & 1);
                    {
                        tc_fence_after();
                        uint32_t o[16];
                        tmem_ld16(t_lane + kColO, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int h = 0; h < G; ++h) o[h] = __float_as_uint(__uint_as_float(o[h]) * corr[h]);
                        tmem_st16(t_lane + kColO, o);
                        tmem_st_wait();
                    }
                }
                if (ts) ts[5] = dt_clk();
                fence_proxy_async_smem();
                if (ts) ts[6] = dt_clk();
                tc_fence_before();
                mbar_arrive(&s.p_full[T & 1]);
                if (ts) {
                    ts[3] = dt_clk();
                    ts[7] = item;
                }
            }
            // ---------------- epilogue: O^T lane r = output dim r ----------------
            mbar_wait(&s.pv_done[(T - 1) & 1], ((T - 1) >> 1) & 1);
            tc_fence_after();
            uint32_t o[16];
            tmem_ld16(t_lane + kColO, o);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&s.o_empty);
            // l: per-thread partial sums -> per head (warp reduce + 4-warp exchange)
            float lsum[G];
#pragma unroll
            for (int h = 0; h < G; ++h) {
                float v = l_thr[h];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                lsum[h] = v;
            }
            if (lane < G) {
                float v = lsum[0];
#pragma unroll
                for (int h = 1; h < G; ++h) v = lane == h ? lsum[h] : v;
                s.redl[quad][lane] = v;
            }
            bar_softmax();
            float L[G];
#pragma unroll
            for (int h = 0; h < G; ++h) L[h] = (s.redl[0][h] + s.redl[1][h]) + (s.redl[2][h] + s.redl[3][h]);
            __nv_bfloat16* orow = out + (static_cast<size_t>(sp.query_start) * p.n_head + static_cast<size_t>(w.kvh) * g) * D;
            if (w.n_parts <= 1) {
#pragma unroll
                for (int h = 0; h < G; ++h)
                    if (h < g) orow[static_cast<size_t>(h) * D + r] = __float2bfloat16_rn(__uint_as_float(o[h]) / L[h]);
            } else {
                const int part = w.part_base + w.part_idx;
#pragma unroll
                for (int h = 0; h < G; ++h)
                    if (h < g) {
                        p.part_o[(static_cast<size_t>(part) * g + h) * D + r] = __uint_as_float(o[h]);
                        if (r == 0) {
                            p.part_ml[(static_cast<size_t>(part) * g + h) * 2 + 0] = m_run[h];
                            p.part_ml[(static_cast<size_t>(part) * g + h) * 2 + 1] = L[h];
                        }
                    }
                __threadfence();
                bar_softmax();
                if (r == 0) s.flag = atomicAdd(&p.counters[w.group], 1) == w.n_parts - 1;
                bar_softmax();
                if (s.flag) {
                    // merge: loads of all heads (and 4 parts) in flight per step
                    __threadfence();
                    const int np = w.n_parts;
                    const float* ml = p.part_ml + static_cast<size_t>(w.part_base) * g * 2;
                    const float* po = p.part_o + static_cast<size_t>(w.part_base) * g * D + r;
                    float M[G], Ls[G], O[G];
#pragma unroll
                    for (int h = 0; h < G; ++h) {
                        M[h] = -CUDART_INF_F;
                        Ls[h] = 0.f;
                        O[h] = 0.f;
                    }
#pragma unroll 4
                    for (int q = 0; q < np; ++q)
#pragma unroll
                        for (int h = 0; h < G; ++h)
                            if (h < g) M[h] = fmaxf(M[h], __ldcg(ml + (q * g + h) * 2));
#pragma unroll 4
                    for (int q = 0; q < np; ++q)
#pragma unroll
                        for (int h = 0; h < G; ++h)
                            if (h < g) {
                                const float f = ex2(__ldcg(ml + (q * g + h) * 2) - M[h]);
                                Ls[h] = fmaf(f, __ldcg(ml + (q * g + h) * 2 + 1), Ls[h]);
                                O[h] = fmaf(f, __ldcg(po + static_cast<size_t>(q * g + h) * D), O[h]);
                            }
#pragma unroll
                    for (int h = 0; h < G; ++h)
                        if (h < g) orow[static_cast<size_t>(h) * D + r] = __float2bfloat16_rn(O[h] / Ls[h]);
                    if (r == 0) p.counters[w.group] = 0; // self-reset for the next launch
                }
            }
        }
    }
}

} // namespace dtc
} // namespace pb
