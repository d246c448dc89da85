// sm_100a tile path of the fused ragged paged attention: multi-token spans (prefill, prompt
// and dropped-prefix recompute spans) on the 5th-generation tensor cores.
//
// Semantics: paged_multi_token_attention, /root/reference/proj/src/attention.cpp:73-132
// (token i of a span sees [0, causal_offset+i], head h reads kv head h/group, softmax with
// max subtraction).  B200 design:
//   * one work item = (span, kv head, block of 2 x 128/group query tokens) = two M=128 query
//     tiles A and B that share every K/V tile loaded; the GQA group is packed into M
//     (rows = tokens x heads-of-the-group), PAPER.md:708-717 fuses QK^T, mask, softmax, PV;
//   * persistent CTAs, 3 warpgroups: WG0 / WG1 = softmax + correction + epilogue of query
//     tiles A / B (one TMEM lane = one query row per thread, 224 registers via setmaxnreg),
//     WG2 = warp 8 TMA producer + warp 9 MMA issuer (one elected thread,
//     tcgen05.mma.cta_group::1.kind::f16) at 56 registers;
//   * TMEM: S_A | S_B | O_A | O_B (4 x 128 columns).  P (bf16) is written back over S with
//     tcgen05.st and fed to the PV MMA straight from TMEM (A operand in TMEM), so P never
//     touches shared memory;
//   * MMA order per KV tile j: PV_A(j), S_A(j+1), PV_B(j), S_B(j+1): while one softmax group
//     works on its scores the tensor core runs the other group's two MMAs (ping-pong);
//   * KV pages are gathered straight from the paged pools by TMA: a 128-row KV tile is
//     128/page_tokens box loads {64 dims, 1 kv head, page_tokens rows} at row coordinate
//     block_table[p] * page_tokens (SWIZZLE_128B); pages past the span's table are fetched
//     out of bounds, which TMA zero-fills;
//   * O is rescaled lazily (only when a row's running max grows by more than 2^8).
#include "attn_internal.hpp"
#include "pb_common.hpp"
#include "sm100_attn.hpp"
#include "sm100_ptx.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <math_constants.h>

#include <algorithm>
#include <cstring>

namespace pb {

namespace {

using namespace pb::sm100;

constexpr int kThreads = 384; // WG0/WG1 softmax of tiles A/B, WG2: TMA warp, MMA warp, 2 spare
constexpr int kTileRows = 128;        // M rows per query tile and kv rows per kv tile
constexpr uint32_t kTmemCols = 512;   // S_A [0,128) S_B [128,256) O_A [256,384) O_B [384,512)
constexpr uint32_t kColO = 256;
#ifndef PB_SETMAXNREG
#define PB_SETMAXNREG 1 // 1: rebalance registers, WG2 (TMA + MMA warps) down, softmax groups up
#endif
constexpr bool kUseSetMaxNReg = PB_SETMAXNREG != 0;
#ifndef PB_REG_LO
#define PB_REG_LO 88  // WG2 after setmaxnreg.dec
#endif
#ifndef PB_REG_HI
#define PB_REG_HI 208 // softmax groups after setmaxnreg.inc (128*LO + 256*HI <= 64K)
#endif
constexpr float kRescaleThreshold = 8.0f; // log2 domain: rescale only if max grows by > 2^8
#ifndef PB_POLY_EVERY
#define PB_POLY_EVERY 0 // one exp2 pair in N on the FMA pipe; 0 = all on MUFU (measured fastest, see profiles/)
#endif
#ifndef PB_P_HALF
#define PB_P_HALF 0     // 1: release P in two halves (measured slower: profiles/r1_variants.md)
#endif
#ifndef PB_LD_SPLIT
#define PB_LD_SPLIT 0   // 1: overlap the second half of the S read with the first half's max
#endif

constexpr int kItemRing = 4; // work items fetched ahead by the TMA warp
constexpr int kMaxPpt = 16;   // pages per 128-row kv tile (page_tokens >= 8)
constexpr int kDecN = 16;     // decode units: padded query heads (N of S^T = K Q^T and O^T = V^T P^T)
constexpr uint32_t kDecPtBytes = 2 * kDecN * 128; // one P^T buffer: [kv half][head][128 B]

template <int D>
struct __align__(1024) Smem {
    uint8_t q[2][kTileRows * D * 2];  // tiles A, B: [D/64][128 rows][128 B] K-major SW128
    uint8_t k[2][kTileRows * D * 2];  // 2-stage ring, same layout
    uint8_t v[2][kTileRows * D * 2];  // 2-stage ring; read as MN-major SW128 B operand
    uint64_t q_full, q_empty;
    uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
    uint64_t s_full[2], p_half[2], p_full[2], o_ready[2], o_empty[2]; // per query tile
    uint64_t item_full[kItemRing], item_empty[kItemRing];   // dynamic tile scheduler ring
    int32_t item_ring[kItemRing];
    // decode units (fused launch): S^T double buffer, P^T ready, PV done; P^T lives in the
    // q[1] region, q rows in the q[0] region (decode units do not use query tile B)
    uint64_t d_s_full[2], d_p_full, d_pv_done;
    float d_red[2][4][kDecN];
    float d_redl[4][kDecN];
    int32_t d_flag;
    uint32_t tmem_base;
};

__device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Query-tile geometry of one work item.
struct ItemTiles {
    int nt[2];     // query tokens in tile A / B (B may be empty)
    int ntiles[2]; // kv tiles each query tile needs (0 when empty)
    int n_kv;      // kv tiles loaded for the item
};

__device__ __forceinline__ ItemTiles item_tiles(const WorkItem& w, const SpanDev& sp, int tpt) {
    ItemTiles r;
    r.nt[0] = min(w.nt, tpt);
    r.nt[1] = w.nt - r.nt[0];
    r.ntiles[0] = ceil_div(sp.causal_offset + w.t0 + r.nt[0], kTileRows);
    r.ntiles[1] = r.nt[1] > 0 ? ceil_div(sp.causal_offset + w.t0 + w.nt, kTileRows) : 0;
    r.n_kv = max(r.ntiles[0], r.ntiles[1]);
    return r;
}

__device__ __forceinline__ int dec_pages(const WorkItem& w, int chunk) {
    return (w.kv_end - w.kv_begin + chunk - 1) / chunk;
}
__device__ __forceinline__ int dec_tiles(const WorkItem& w, int chunk) {
    return (dec_pages(w, chunk) * chunk + kTileRows - 1) / kTileRows;
}
__device__ __forceinline__ void bar_group0() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
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

// A operand in TMEM (P, bf16), B from shared memory (V).
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

template <int D, int GD>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fused_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                            const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_qd,
                            const AttnParams p) {
    constexpr int KH = D / 64;                  // 64-dim halves (one 128 B swizzle row each)
    constexpr uint32_t kHalfBytes = kTileRows * 128;
    constexpr uint32_t kTileBytes = kTileRows * D * 2;
    extern __shared__ uint8_t smem_raw[];
    Smem<D>& s = *reinterpret_cast<Smem<D>*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5;
    const int g = p.group;
    const int tpt = kTileRows / g;         // query tokens per query tile
    const int chunk = p.chunk;
    const int ppt = kTileRows / chunk;     // pages per kv tile

    if (threadIdx.x == 0) {
        mbar_init(&s.q_full, 1);
        mbar_init(&s.q_empty, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s.k_full[i], 1);
            mbar_init(&s.k_empty[i], 1);
            mbar_init(&s.v_full[i], 1);
            mbar_init(&s.v_empty[i], 1);
            mbar_init(&s.s_full[i], 1);
            mbar_init(&s.p_half[i], 128);
            mbar_init(&s.p_full[i], 128);
            mbar_init(&s.o_ready[i], 1);
            mbar_init(&s.o_empty[i], 128);
        }
        for (int i = 0; i < kItemRing; ++i) {
            mbar_init(&s.item_full[i], 1);
            mbar_init(&s.item_empty[i], 1 + 8); // MMA thread + the 8 softmax warps
        }
        mbar_init(&s.d_s_full[0], 1);
        mbar_init(&s.d_s_full[1], 1);
        mbar_init(&s.d_p_full, 128);
        mbar_init(&s.d_pv_done, 1);
        mbar_fence_init();
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        tma_prefetch(&tm_qd);
    }
    if (warp == 9) tmem_alloc<kTmemCols>(&s.tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem_base;
    const int wg = warp >> 2;
    if (wg == 2) {
    if (kUseSetMaxNReg) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(PB_REG_LO) : "memory");
    if (warp == 8) {
        // ============================ TMA producer ============================
        if (elect_one()) {
            int it = 0, kst = 0, vst = 0;
            uint32_t kph = 0, vph = 0;
            const uint32_t q_bytes = KH * 128u * static_cast<uint32_t>(g * tpt);
            const int oob_row = p.n_slots * chunk;
            // Dynamic tile scheduler: the TMA warp takes the next item (items are in LPT order)
            // from a global ticket when it is ready to load it, and hands the index to the MMA
            // and softmax roles through a small shared ring.
            int* ticket = p.work_counter + 2; // [2] next item, [3] retired CTAs (self-resetting)
            for (;; ++it) {
                const int slot = it % kItemRing;
                if (it >= kItemRing) mbar_wait(&s.item_empty[slot], ((it / kItemRing) - 1) & 1);
                int item = atomicAdd(ticket, 1);
                if (item >= p.n_items) item = -1;
                s.item_ring[slot] = item;
                mbar_arrive(&s.item_full[slot]);
                if (item < 0) break;
                const WorkItem w = p.items[item];
                const SpanDev sp = p.spans[w.span];
                if (it > 0) mbar_wait(&s.q_empty, (it - 1) & 1);
                const int32_t* table;
                int n_pages, n_kv;
                if (w.type == kWorkDecode) {
                    // decode unit: the g query rows of one token into the q[0] region, then the
                    // unit's page range
                    mbar_arrive_expect_tx(&s.q_full, KH * 128u * static_cast<uint32_t>(g));
                    for (int h = 0; h < KH; ++h)
                        tma_load_3d(s.q[0] + h * kHalfBytes, &tm_qd, &s.q_full, h * 64, w.kvh * g, sp.query_start);
                    table = p.block_tables + sp.bt_off + w.kv_begin / chunk;
                    n_pages = dec_pages(w, chunk);
                    n_kv = dec_tiles(w, chunk);
                } else {
                    const ItemTiles T = item_tiles(w, sp, tpt);
                    mbar_arrive_expect_tx(&s.q_full, q_bytes * (T.nt[1] > 0 ? 2u : 1u));
                    for (int t = 0; t < 2; ++t)
                        if (T.nt[t] > 0)
                            for (int h = 0; h < KH; ++h)
                                tma_load_3d(s.q[t] + h * kHalfBytes, &tm_q, &s.q_full, h * 64, w.kvh * g,
                                            sp.query_start + w.t0 + t * tpt);
                    table = p.block_tables + sp.bt_off;
                    n_pages = sp.n_pages;
                    n_kv = T.n_kv;
                }
                for (int j = 0; j < n_kv; ++j) {
                    // the tile's block-table entries: independent loads issued together, before
                    // any barrier wait or TMA (one L2 round trip per tile, not one per page)
                    int rows[kMaxPpt];
#pragma unroll
                    for (int pg = 0; pg < kMaxPpt; ++pg) {
                        const int page = j * ppt + pg;
                        rows[pg] = (pg < ppt && page < n_pages) ? __ldg(table + page) * chunk : oob_row;
                    }
                    for (int which = 0; which < 2; ++which) {
                        uint64_t* full = which ? &s.v_full[vst] : &s.k_full[kst];
                        uint64_t* empty = which ? &s.v_empty[vst] : &s.k_empty[kst];
                        uint8_t* dst = which ? s.v[vst] : s.k[kst];
                        const CUtensorMap* tm = which ? &tm_v : &tm_k;
                        mbar_wait(empty, (which ? vph : kph) ^ 1);
                        mbar_arrive_expect_tx(full, kTileBytes);
#pragma unroll
                        for (int pg = 0; pg < kMaxPpt; ++pg)
                            if (pg < ppt)
                                for (int h = 0; h < KH; ++h)
                                    tma_load_3d(dst + h * kHalfBytes + pg * chunk * 128, tm, full, h * 64, w.kvh, rows[pg]);
                        if (which) {
                            if (++vst == 2) { vst = 0; vph ^= 1; }
                        } else {
                            if (++kst == 2) { kst = 0; kph ^= 1; }
                        }
                    }
                }
            }
            // the last CTA to retire re-arms the ticket for the next launch
            __threadfence();
            if (atomicAdd(ticket + 1, 1) == static_cast<int>(gridDim.x) - 1) {
                ticket[0] = 0;
                ticket[1] = 0;
            }
        }
    } else if (warp == 9) {
        // ============================ MMA issuer =============================
        if (elect_one()) {
            constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
            constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, false, true);
            int it = 0, kst = 0, vst = 0;
            uint32_t kph = 0, vph = 0;
            uint32_t n_p[2] = {0, 0}, n_oe[2] = {0, 0};
            uint32_t dT = 0; // decode kv tiles issued (S^T buffer / P^T buffer parity)
            for (;; ++it) {
                const int slot = it % kItemRing;
                mbar_wait(&s.item_full[slot], (it / kItemRing) & 1);
                const int item = *reinterpret_cast<volatile int32_t*>(&s.item_ring[slot]);
                mbar_arrive(&s.item_empty[slot]);
                if (item < 0) break;
                const WorkItem w = p.items[item];
                if (w.type == kWorkDecode) {
                    if constexpr (D == 128) {
                        // S^T = K Q^T (M = 128 kv rows, N = 16 heads) into S_A columns
                        // [16*(dT&1), +16); O^T += V^T P^T (M = d, N = 16) into O_A
                        constexpr uint32_t idesc_sd = umma_idesc_bf16(128, kDecN, false, false);
                        constexpr uint32_t idesc_od = umma_idesc_bf16(128, kDecN, true, false);
                        const int nt = dec_tiles(w, chunk);
                        auto issue_sd = [&](uint32_t tile) {
                            const uint64_t ad = umma_desc_sw128(smem_u32(s.k[kst]), 16, 1024);
                            const uint64_t bd = umma_desc_sw128(smem_u32(s.q[0]), 16, 1024);
#pragma unroll
                            for (int kk = 0; kk < D / 16; ++kk) {
                                const uint32_t off = ((kk >> 2) * kHalfBytes + (kk & 3) * 32) >> 4;
                                umma_bf16_ss(tmem + (tile & 1) * kDecN, ad + off, bd + off, idesc_sd, kk > 0);
                            }
                            umma_commit(&s.d_s_full[tile & 1]);
                            umma_commit(&s.k_empty[kst]);
                            if (++kst == 2) { kst = 0; kph ^= 1; }
                        };
                        mbar_wait(&s.q_full, it & 1);
                        mbar_wait(&s.k_full[kst], kph);
                        tc_fence_after();
                        issue_sd(dT);
                        for (int j = 0; j < nt; ++j, ++dT) {
                            if (j + 1 < nt) { // S^T(j+1) overlaps softmax(j)
                                mbar_wait(&s.k_full[kst], kph);
                                tc_fence_after();
                                issue_sd(dT + 1);
                            }
                            mbar_wait(&s.d_p_full, dT & 1);
                            if (j == 0) {
                                mbar_wait(&s.o_empty[0], (n_oe[0] & 1) ^ 1);
                                ++n_oe[0];
                            }
                            mbar_wait(&s.v_full[vst], vph);
                            tc_fence_after();
                            const uint64_t ad = umma_desc_sw128(smem_u32(s.v[vst]), kHalfBytes, 1024);
                            const uint64_t bd = umma_desc_sw128(smem_u32(s.q[1]) + (dT & 1) * kDecPtBytes, 16, 1024);
#pragma unroll
                            for (int kk = 0; kk < kTileRows / 16; ++kk) {
                                const uint32_t ob = ((kk >> 2) * (kDecN * 128) + (kk & 3) * 32) >> 4;
                                umma_bf16_ss(tmem + kColO, ad + kk * (2048 >> 4), bd + ob, idesc_od,
                                             (j > 0 || kk > 0) ? 1u : 0u);
                            }
                            umma_commit(&s.d_pv_done);
                            umma_commit(&s.v_empty[vst]);
                            if (++vst == 2) { vst = 0; vph ^= 1; }
                        }
                        umma_commit(&s.q_empty);
                    }
                    continue;
                }
                const SpanDev sp = p.spans[w.span];
                const ItemTiles T = item_tiles(w, sp, tpt);
                mbar_wait(&s.q_full, it & 1);
                tc_fence_after();
                // S_t = Q_t K^T for the kv tile in stage kst
                // descriptors are advanced by adding (byte offset >> 4) to the start-address
                // field (no carry: shared addresses < 256 KB), which keeps register use low
                auto issue_s = [&](int t) {
                    const uint64_t qd = umma_desc_sw128(smem_u32(s.q[t]), 16, 1024);
                    const uint64_t kd = umma_desc_sw128(smem_u32(s.k[kst]), 16, 1024);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off = ((kk >> 2) * kHalfBytes + (kk & 3) * 32) >> 4;
                        umma_bf16_ss(tmem + t * 128, qd + off, kd + off, idesc_s, kk > 0);
                    }
                    umma_commit(&s.s_full[t]);
                };
                // S for kv tile 0
                mbar_wait(&s.k_full[kst], kph);
                tc_fence_after();
                for (int t = 0; t < 2; ++t)
                    if (T.ntiles[t] > 0) issue_s(t);
                umma_commit(&s.k_empty[kst]);
                if (++kst == 2) { kst = 0; kph ^= 1; }
                for (int j = 0; j < T.n_kv; ++j) {
                    mbar_wait(&s.v_full[vst], vph);
                    bool k_next_ready = false;
                    for (int t = 0; t < 2; ++t) {
                        if (j >= T.ntiles[t]) continue;
                        if (j == 0) {
                            mbar_wait(&s.o_empty[t], (n_oe[t] & 1) ^ 1);
                            ++n_oe[t];
                        }
                        const uint64_t vd = umma_desc_sw128(smem_u32(s.v[vst]), kHalfBytes, 1024);
                        // kv rows 0..63 as soon as the first half of P_t is in TMEM, then 64..127
                        mbar_wait(&s.p_half[t], n_p[t] & 1);
                        tc_fence_after();
#pragma unroll
                        for (int kk = 0; kk < kTileRows / 32; ++kk)
                            umma_bf16_ts(tmem + kColO + t * 128, tmem + t * 128 + kk * 8, vd + kk * (2048 >> 4),
                                         idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
                        mbar_wait(&s.p_full[t], n_p[t] & 1);
                        ++n_p[t];
                        tc_fence_after();
#pragma unroll
                        for (int kk = kTileRows / 32; kk < kTileRows / 16; ++kk)
                            umma_bf16_ts(tmem + kColO + t * 128, tmem + t * 128 + kk * 8, vd + kk * (2048 >> 4),
                                         idesc_o, 1u);
                        if (j + 1 == T.ntiles[t]) umma_commit(&s.o_ready[t]);
                        if (j + 1 < T.ntiles[t]) {
                            if (!k_next_ready) {
                                mbar_wait(&s.k_full[kst], kph);
                                tc_fence_after();
                                k_next_ready = true;
                            }
                            issue_s(t);
                        }
                    }
                    umma_commit(&s.v_empty[vst]);
                    if (++vst == 2) { vst = 0; vph ^= 1; }
                    if (j + 1 < T.n_kv) {
                        if (!k_next_ready) { // no query tile needed it (cannot happen; keep rings in step)
                            mbar_wait(&s.k_full[kst], kph);
                        }
                        umma_commit(&s.k_empty[kst]);
                        if (++kst == 2) { kst = 0; kph ^= 1; }
                    }
                }
                umma_commit(&s.q_empty);
            }
        }
    }
    } else {
        if (kUseSetMaxNReg) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(PB_REG_HI) : "memory");
        // ============ softmax / correction / epilogue (one group per query tile) ============
        const int t = wg;                           // query tile of this warpgroup
        const int quad = warp & 3;                  // TMEM lane quadrant of this warp
        const int row = quad * 32 + (threadIdx.x & 31);
        const uint32_t t_lane = tmem + (static_cast<uint32_t>(quad * 32) << 16);
        const uint32_t col_s = t * 128;
        const uint32_t col_o = kColO + t * 128;
        const float sl2 = p.scale_log2;
        uint32_t n_s = 0, n_o = 0;
        uint32_t kv_seen = 0; // kv tiles loaded for earlier items (V ring position)
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out);
        uint32_t dT = 0;      // decode kv tiles consumed (group 0 only)
        // ---- decode unit (group 0): thread `row` owns kv row `row` of each S^T tile and
        // output dim `row` of O^T (semantics: single_token_attention, attention.cpp:134-188)
        auto decode_unit = [&](const WorkItem& w, const SpanDev& sp, int nt, uint32_t kvb) {
            const int lane = threadIdx.x & 31;
            const uint32_t pt_row = static_cast<uint32_t>((row >> 6) * (kDecN * 128) + (row & 7) * 2);
            const uint32_t pt_c16 = static_cast<uint32_t>((row & 63) >> 3);
            float m_run[GD], l_thr[GD];
#pragma unroll
            for (int h = 0; h < GD; ++h) {
                m_run[h] = -CUDART_INF_F;
                l_thr[h] = 0.f;
            }
            for (int j = 0; j < nt; ++j, ++dT) {
                mbar_wait(&s.d_s_full[dT & 1], (dT >> 1) & 1);
                tc_fence_after();
                uint32_t sr[16];
                tmem_ld16(t_lane + (dT & 1) * kDecN, sr);
                tmem_ld_wait();
                const int kv = w.kv_begin + j * kTileRows + row;
                const bool ok = kv < w.kv_end;
                float x[GD], mt[GD];
#pragma unroll
                for (int h = 0; h < GD; ++h) {
                    x[h] = (ok && h < g) ? __uint_as_float(sr[h]) * sl2 : -CUDART_INF_F;
                    float m = x[h];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                    mt[h] = m;
                }
                if (lane < GD) {
                    float v = mt[0];
#pragma unroll
                    for (int h = 1; h < GD; ++h) v = lane == h ? mt[h] : v;
                    s.d_red[dT & 1][quad][lane] = v;
                }
                bar_group0();
                bool rescale = false;
                float corr[GD];
#pragma unroll
                for (int h = 0; h < GD; ++h) {
                    const float m4 = fmaxf(fmaxf(s.d_red[dT & 1][0][h], s.d_red[dT & 1][1][h]),
                                           fmaxf(s.d_red[dT & 1][2][h], s.d_red[dT & 1][3][h]));
                    const bool grow = m4 > m_run[h] + kRescaleThreshold; // uniform over the group
                    const float m_new = grow ? m4 : m_run[h];
                    corr[h] = grow ? ex2(m_run[h] - m_new) : 1.f;
                    rescale |= grow && j > 0;
                    m_run[h] = m_new;
                }
                const uint32_t ptb = smem_u32(s.q[1]) + (dT & 1) * kDecPtBytes + pt_row;
#pragma unroll
                for (int h = 0; h < GD; ++h) {
                    if (h < g) {
                        const float pr = ok ? ex2(x[h] - m_run[h]) : 0.f;
                        l_thr[h] = l_thr[h] * corr[h] + pr;
                        const __nv_bfloat16 b = __float2bfloat16_rn(pr);
                        st_shared_u16(ptb + h * 128 + ((pt_c16 ^ (h & 7)) << 4), *reinterpret_cast<const uint16_t*>(&b));
                    }
                }
                if (!ok && j + 1 == nt) {
                    // fetched rows past the unit's end may hold anything: zero their V
                    uint8_t* vrow = s.v[(kvb + j) & 1] + row * 128;
#pragma unroll
                    for (int h = 0; h < KH; ++h)
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            *reinterpret_cast<uint4*>(vrow + h * kHalfBytes + c * 16) = make_uint4(0, 0, 0, 0);
                }
                if (j > 0) {
                    mbar_wait(&s.d_pv_done, (dT - 1) & 1); // PV(j-1) done: O^T may be rescaled
                    if (rescale) {
                        tc_fence_after();
                        uint32_t o[16];
                        tmem_ld16(t_lane + kColO, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int h = 0; h < GD; ++h) o[h] = __float_as_uint(__uint_as_float(o[h]) * corr[h]);
                        tmem_st16(t_lane + kColO, o);
                        tmem_st_wait();
                    }
                }
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(&s.d_p_full);
            }
            // epilogue: O^T lane `row` = output dim `row`
            mbar_wait(&s.d_pv_done, (dT - 1) & 1);
            tc_fence_after();
            uint32_t o[16];
            tmem_ld16(t_lane + kColO, o);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&s.o_empty[0]);
            float lsum[GD];
#pragma unroll
            for (int h = 0; h < GD; ++h) {
                float v = l_thr[h];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                lsum[h] = v;
            }
            if (lane < GD) {
                float v = lsum[0];
#pragma unroll
                for (int h = 1; h < GD; ++h) v = lane == h ? lsum[h] : v;
                s.d_redl[quad][lane] = v;
            }
            bar_group0();
            float L[GD];
#pragma unroll
            for (int h = 0; h < GD; ++h)
                L[h] = (s.d_redl[0][h] + s.d_redl[1][h]) + (s.d_redl[2][h] + s.d_redl[3][h]);
            __nv_bfloat16* orow = out + (static_cast<size_t>(sp.query_start) * p.n_head + static_cast<size_t>(w.kvh) * g) * D;
            if (w.n_parts <= 1) {
#pragma unroll
                for (int h = 0; h < GD; ++h)
                    if (h < g) orow[static_cast<size_t>(h) * D + row] = __float2bfloat16_rn(__uint_as_float(o[h]) / L[h]);
                return;
            }
            const int part = w.part_base + w.part_idx;
#pragma unroll
            for (int h = 0; h < GD; ++h)
                if (h < g) {
                    p.part_o[(static_cast<size_t>(part) * g + h) * D + row] = __uint_as_float(o[h]);
                    if (row == 0) {
                        p.part_ml[(static_cast<size_t>(part) * g + h) * 2 + 0] = m_run[h];
                        p.part_ml[(static_cast<size_t>(part) * g + h) * 2 + 1] = L[h];
                    }
                }
            __threadfence();
            bar_group0();
            if (row == 0) s.d_flag = atomicAdd(&p.counters[w.group], 1) == w.n_parts - 1;
            bar_group0();
            if (!s.d_flag) return;
            // last split of the group: merge (loads of all heads and 4 parts in flight per step)
            __threadfence();
            const int np = w.n_parts;
            const float* ml = p.part_ml + static_cast<size_t>(w.part_base) * g * 2;
            const float* po = p.part_o + static_cast<size_t>(w.part_base) * g * D + row;
            float M[GD], Ls[GD], O[GD];
#pragma unroll
            for (int h = 0; h < GD; ++h) {
                M[h] = -CUDART_INF_F;
                Ls[h] = 0.f;
                O[h] = 0.f;
            }
#pragma unroll 4
            for (int q = 0; q < np; ++q)
#pragma unroll
                for (int h = 0; h < GD; ++h)
                    if (h < g) M[h] = fmaxf(M[h], __ldcg(ml + (q * g + h) * 2));
#pragma unroll 4
            for (int q = 0; q < np; ++q)
#pragma unroll
                for (int h = 0; h < GD; ++h)
                    if (h < g) {
                        const float f = ex2(__ldcg(ml + (q * g + h) * 2) - M[h]);
                        Ls[h] = fmaf(f, __ldcg(ml + (q * g + h) * 2 + 1), Ls[h]);
                        O[h] = fmaf(f, __ldcg(po + static_cast<size_t>(q * g + h) * D), O[h]);
                    }
#pragma unroll
            for (int h = 0; h < GD; ++h)
                if (h < g) orow[static_cast<size_t>(h) * D + row] = __float2bfloat16_rn(O[h] / Ls[h]);
            if (row == 0) p.counters[w.group] = 0; // self-reset for the next launch
        };
        for (int it = 0;; ++it) {
            const int slot = it % kItemRing;
            mbar_wait(&s.item_full[slot], (it / kItemRing) & 1);
            const int item = *reinterpret_cast<volatile int32_t*>(&s.item_ring[slot]);
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&s.item_empty[slot]);
            if (item < 0) break;
            const WorkItem w = p.items[item];
            const SpanDev sp = p.spans[w.span];
            if (w.type == kWorkDecode) {
                const int ntd = dec_tiles(w, chunk);
                const uint32_t kvb = kv_seen;
                kv_seen += static_cast<uint32_t>(ntd);
                if constexpr (D == 128) {
                    if (t == 0) decode_unit(w, sp, ntd, kvb);
                }
                continue;
            }
            const ItemTiles T = item_tiles(w, sp, tpt);
            const int n_tiles = T.ntiles[t];
            const uint32_t kv_base = kv_seen;
            kv_seen += static_cast<uint32_t>(T.n_kv);
            if (n_tiles == 0) continue;
            // rows of the span's last page past its context may hold anything (stale or
            // never-written pool memory): this group zeroes them in the V stage of the item's
            // last kv tile before its PV reads it (tile A when it reaches that tile, else B),
            // so 0 * NaN cannot reach O
            const bool zero_owner = (t == 0) ? (T.ntiles[0] == T.n_kv) : (T.ntiles[0] < T.n_kv);
            const int t_local = row / g;
            const bool valid = t_local < T.nt[t] && row < g * tpt;
            const int tok0 = w.t0 + t * tpt;           // first span-relative token of this tile
            const int allowed = sp.causal_offset + tok0 + (valid ? t_local : 0) + 1;
            float m_run = -CUDART_INF_F, l_run = 0.f;
            for (int j = 0; j < n_tiles; ++j) {
                mbar_wait(&s.s_full[t], n_s & 1);
                ++n_s;
                tc_fence_after();
                if (p.ablate == 1) { // profiling: tensor-core + pipeline bound (P left as S bits)
                    tc_fence_before();
                    mbar_arrive(&s.p_half[t]);
                    mbar_arrive(&s.p_full[t]);
                    l_run = 1.f;
                    continue;
                }
                float x[128];
                const int kv0 = j * kTileRows;
                const bool diag = kv0 + kTileRows > allowed;
                float pm[8];
#if PB_LD_SPLIT
                // two halves: the second half's TMEM read is in flight while the first half's
                // max runs (the wait carries the registers so no use is hoisted above it)
                tmem_ld32(t_lane + col_s, *reinterpret_cast<uint32_t(*)[32]>(&x[0]));
                tmem_ld32(t_lane + col_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&x[32]));
                tmem_ld_wait_dep(*reinterpret_cast<uint32_t(*)[32]>(&x[0]));
                tmem_ld_wait_dep(*reinterpret_cast<uint32_t(*)[32]>(&x[32]));
                tmem_ld32(t_lane + col_s + 64, *reinterpret_cast<uint32_t(*)[32]>(&x[64]));
                tmem_ld32(t_lane + col_s + 96, *reinterpret_cast<uint32_t(*)[32]>(&x[96]));
                if (diag) {
#pragma unroll
                    for (int c = 0; c < 64; ++c) x[c] = (kv0 + c < allowed) ? x[c] : -CUDART_INF_F;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) pm[u] = x[u];
#pragma unroll
                for (int c = 8; c < 64; ++c) pm[c & 7] = fmaxf(pm[c & 7], x[c]);
                tmem_ld_wait_dep(*reinterpret_cast<uint32_t(*)[32]>(&x[64]));
                tmem_ld_wait_dep(*reinterpret_cast<uint32_t(*)[32]>(&x[96]));
                if (diag) {
#pragma unroll
                    for (int c = 64; c < 128; ++c) x[c] = (kv0 + c < allowed) ? x[c] : -CUDART_INF_F;
                }
#pragma unroll
                for (int c = 64; c < 128; ++c) pm[c & 7] = fmaxf(pm[c & 7], x[c]);
#else
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    tmem_ld32(t_lane + col_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&x[c * 32]));
                tmem_ld_wait();
                // causal mask (only tiles that cross this row's boundary) + running max
                if (diag) {
#pragma unroll
                    for (int c = 0; c < 128; ++c) x[c] = (kv0 + c < allowed) ? x[c] : -CUDART_INF_F;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) pm[u] = x[u];
#pragma unroll
                for (int c = 8; c < 128; ++c) pm[c & 7] = fmaxf(pm[c & 7], x[c]);
#endif
                const float mt = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                                       fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7]))) * sl2;
                const bool grow = mt > m_run + kRescaleThreshold;
                const float m_new = grow ? mt : m_run;
                const float corr = grow ? ex2(m_run - m_new) : 1.f;
                // S_t(j) landing implies PV_t(j-1) completed (in-order tensor pipe, the commit for
                // s_full was issued after it): O_t may be rescaled now, before any of P_t(j) is
                // released to the tensor core
                if (j > 0 && __any_sync(0xffffffffu, grow)) {
#pragma unroll
                    for (int c = 0; c < D / 32; ++c) {
                        uint32_t o[32];
                        tmem_ld32(t_lane + col_o + c * 32, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
                        tmem_st32(t_lane + col_o + c * 32, o);
                    }
                }
                if (zero_owner && j + 1 == T.n_kv) {
                    const int kv = kv0 + row;
                    if (kv >= sp.context_len && kv < sp.n_pages * chunk) {
                        uint8_t* vrow = s.v[(kv_base + j) & 1] + row * 128;
#pragma unroll
                        for (int h = 0; h < KH; ++h)
#pragma unroll
                            for (int c = 0; c < 8; ++c)
                                *reinterpret_cast<uint4*>(vrow + h * kHalfBytes + c * 16) = make_uint4(0, 0, 0, 0);
                        fence_proxy_async_smem();
                    }
                }
                float2 ps[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) ps[u] = make_float2(0.f, 0.f);
                uint32_t pk[32];
                const float2 sl2x2 = make_float2(sl2, sl2), negm = make_float2(-m_new, -m_new);
#pragma unroll
                for (int c = 0; c < 128; c += 2) {
                    // exp2((s - max) * log2e / scale) on packed pairs (FFMA2 / FADD2) and MUFU
                    const float2 a = fma2(make_float2(x[c], x[c + 1]), sl2x2, negm);
                    float2 e;
                    if (p.ablate == 2) { // profiling: no exponentials
                        e = a;
                    } else if (PB_POLY_EVERY > 0 && ((c >> 1) % (PB_POLY_EVERY > 0 ? PB_POLY_EVERY : 1)) ==
                                                        PB_POLY_EVERY - 1) {
                        e = exp2_poly3_x2(a);
                    } else {
                        e.x = ex2(a.x);
                        e.y = ex2(a.y);
                    }
                    ps[(c >> 1) & 3] = add2(ps[(c >> 1) & 3], e);
                    pk[(c >> 1) & 31] = pack_bf16x2(e.x, e.y);
                    if (c == 62 || c == 126) {
                        // P (bf16) over S_t's columns; with PB_P_HALF the first half is released
                        // to the tensor core (PV kv rows 0..63) while the second is computed
                        tmem_st32(t_lane + col_s + (c == 62 ? 0 : 32), pk);
                        if (PB_P_HALF || c == 126) {
                            tmem_st_wait();
                            tc_fence_before();
                            if (c == 126 && !PB_P_HALF) mbar_arrive(&s.p_half[t]);
                            mbar_arrive(c == 62 ? &s.p_half[t] : &s.p_full[t]);
                        }
                    }
                }
                const float2 s2 = add2(add2(ps[0], ps[1]), add2(ps[2], ps[3]));
                const float sum = s2.x + s2.y;
                l_run = l_run * corr + sum;
                m_run = m_new;
            }
            // epilogue: O / l -> bf16 -> global
            mbar_wait(&s.o_ready[t], n_o & 1);
            ++n_o;
            tc_fence_after();
            const float inv_l = 1.f / l_run;
            const int h = w.kvh * g + (row % g);
            __nv_bfloat16* orow = out + (static_cast<size_t>(sp.query_start + tok0 + t_local) * p.n_head + h) * D;
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                uint32_t o[32];
                tmem_ld32(t_lane + col_o + c * 32, o);
                tmem_ld_wait();
                if (valid) {
#pragma unroll
                    for (int e = 0; e < 32; e += 8) {
                        uint4 v;
                        v.x = pack_bf16x2(__uint_as_float(o[e + 0]) * inv_l, __uint_as_float(o[e + 1]) * inv_l);
                        v.y = pack_bf16x2(__uint_as_float(o[e + 2]) * inv_l, __uint_as_float(o[e + 3]) * inv_l);
                        v.z = pack_bf16x2(__uint_as_float(o[e + 4]) * inv_l, __uint_as_float(o[e + 5]) * inv_l);
                        v.w = pack_bf16x2(__uint_as_float(o[e + 6]) * inv_l, __uint_as_float(o[e + 7]) * inv_l);
                        *reinterpret_cast<uint4*>(orow + c * 32 + e) = v;
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&s.o_empty[t]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
}

// ------------------------------------------------------------------ host side

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q),
                   "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
        if (!f || q != cudaDriverEntryPointSuccess) fail(PB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    return fn;
}

void encode_3d(CUtensorMap* m, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1_bytes,
               uint64_t s2_bytes, uint32_t b0, uint32_t b1, uint32_t b2) {
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {s1_bytes, s2_bytes};
    cuuint32_t box[3] = {b0, b1, b2};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(PB_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
}

int g_sms = 0;

template <int D, int GD>
void launch_fused(const AttnParams& p, const CUtensorMap* maps, cudaStream_t st) {
    const size_t smem = sizeof(Smem<D>) + 1024;
    static bool attr_set = false;
    if (!attr_set) {
        cuda_check(cudaFuncSetAttribute(attn_fused_sm100_kernel<D, GD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)),
                   "cudaFuncSetAttribute(fused smem)");
        attr_set = true;
    }
    if (g_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int grid = std::min(p.n_items, g_sms);
    attn_fused_sm100_kernel<D, GD><<<grid, kThreads, smem, st>>>(maps[0], maps[1], maps[2], maps[3], p);
    cuda_check(cudaGetLastError(), "attn_fused_sm100 launch");
    count_launch();
}

} // namespace

bool sm100_supports(int head_size, int chunk, int group) {
    return (head_size == 64 || head_size == 128) && chunk >= 8 && chunk <= 128 && (128 % chunk) == 0 &&
           group >= 1 && group <= 128;
}

int sm100_tile_tokens(int group) { return 2 * (kTileRows / group); } // two query tiles per item

void sm100_prepare_maps(const AttnParams& p, const pb_attn_shape& shape, Sm100Cache& cache, int64_t total_tokens) {
    const int D = shape.head_size;
    const int g = shape.n_head / shape.n_kv_head;
    if (!cache.valid || cache.q != p.q || cache.k != p.k_pages || cache.v != p.v_pages ||
        cache.total_tokens != total_tokens) {
        auto* m = reinterpret_cast<CUtensorMap*>(cache.maps);
        encode_3d(&m[0], p.q, D, shape.n_head, std::max<int64_t>(total_tokens, 1), D * 2ull,
                  static_cast<uint64_t>(shape.n_head) * D * 2, 64, g, kTileRows / g);
        const uint64_t rows = static_cast<uint64_t>(shape.n_slots) * shape.chunk_size;
        encode_3d(&m[1], p.k_pages, D, shape.n_kv_head, std::max<uint64_t>(rows, 1), D * 2ull,
                  static_cast<uint64_t>(shape.n_kv_head) * D * 2, 64, 1, shape.chunk_size);
        encode_3d(&m[2], p.v_pages, D, shape.n_kv_head, std::max<uint64_t>(rows, 1), D * 2ull,
                  static_cast<uint64_t>(shape.n_kv_head) * D * 2, 64, 1, shape.chunk_size);
        // decode rows: the g query heads of one kv head for one token
        encode_3d(&m[3], p.q, D, shape.n_head, std::max<int64_t>(total_tokens, 1), D * 2ull,
                  static_cast<uint64_t>(shape.n_head) * D * 2, 64, g, 1);
        cache.q = p.q;
        cache.k = p.k_pages;
        cache.v = p.v_pages;
        cache.total_tokens = total_tokens;
        cache.valid = true;
    }
}

void launch_attn_sm100(const AttnParams& p, const pb_attn_shape& shape, Sm100Cache& cache, int64_t total_tokens,
                       cudaStream_t stream) {
    if (p.n_items <= 0) return;
    sm100_prepare_maps(p, shape, cache, total_tokens);
    const int D = shape.head_size;
    const auto* maps = reinterpret_cast<const CUtensorMap*>(cache.maps);
    if (D == 128 && p.group > 8) launch_fused<128, 16>(p, maps, stream);
    else if (D == 128) launch_fused<128, 8>(p, maps, stream);
    else launch_fused<64, 8>(p, maps, stream);
}

void sm100_cache_release(Sm100Cache& cache) { cache.valid = false; }

} // namespace pb
