// The fused ragged paged attention launch for sm_100a: multi-token spans (prefill, prompt
// and dropped-prefix recompute spans) as tcgen05 tiles, single-token spans as tcgen05
// split-KV units (decode_tc_cta.cuh), from two persistent queues in one kernel.
//
// Semantics: paged_multi_token_attention, /root/reference/proj/src/attention.cpp:73-132
// (token i of a span sees [0, causal_offset+i], head h reads kv head h/group, softmax with
// max subtraction).  Tile pipeline:
//   * one work item = (span, kv head, block of 2 x 128/group query tokens) = two M=128 query
//     tiles A and B that share every K/V tile loaded; the GQA group is packed into M
//     (rows = tokens x heads-of-the-group); PAPER.md:708-717 fuses QK^T, mask, softmax, PV;
//   * persistent CTAs, 3 warpgroups: WG0 / WG1 = softmax + correction + epilogue of query
//     tiles A / B (one TMEM lane = one query row per thread, 208 registers via setmaxnreg),
//     WG2 = warp 8 TMA producer + warp 9 MMA issuer (one elected thread,
//     tcgen05.mma.cta_group::1.kind::f16) at 88 registers;
//   * kv tiles of 128 rows, so S = Q K^T runs as M=128 N=128 instructions: at N=64 both
//     shared-memory operands (6 KB per K=16 step) exceed what the tensor core reads per
//     clock and the instruction runs at 2/3 rate (scripts/microbench/mma_rate.cu,
//     profiles/r2_tile_pipeline.md); TMEM: S_A | S_B | O_A | O_B (128 columns each);
//   * P (bf16) is written back over the first 64 columns of its S buffer with tcgen05.st and
//     fed to the PV MMA from TMEM; per kv tile j the MMA issuer runs PV_A(j), S_A(j+1),
//     PV_B(j), S_B(j+1): the tensor pipe executes one thread's MMAs in order, so S_t(j+1)
//     overwrites P_t(j) only after PV_t(j) has read it, and its completion (s_full) also
//     proves PV_t(j) done, which is what the lazy O rescale of tile j+1 needs.  Softmax A
//     overlaps the tensor work of tile B and vice versa (ping-pong);
//   * KV pages are gathered straight from the paged pools by TMA: a kv tile is
//     128/page_tokens box loads {64 dims, 1 kv head, page_tokens rows} per 64-dim half at row
//     block_table[p] * page_tokens (SWIZZLE_128B); pages past the span's table are fetched
//     out of bounds, which TMA zero-fills;
//   * O is rescaled lazily (only when a row's running max grows by more than 2^8).
// DESIGN.md §3 has the measurements behind each choice and the pipeline invariants.
#include "attn_internal.hpp"
#include "pb_common.hpp"
#include "sm100_attn.hpp"
#include "sm100_ptx.cuh"
#include "decode_tc_cta.cuh"
#include "append_prologue.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <math_constants.h>

#include <algorithm>
#include <cstring>
#include <mutex>

namespace pb {

namespace {

using namespace pb::sm100;

constexpr int kSoftWG = 2;                    // softmax warpgroups (query tiles A, B)
constexpr int kThreads = 128 * (kSoftWG + 1); // + one warpgroup: TMA warp, MMA warp, 2 spare
constexpr int kProdWarp = 4 * kSoftWG;
constexpr int kMmaWarp = kProdWarp + 1;
constexpr int kProdVWarp = kProdWarp + 2; // V tiles have their own producer: K(j+1) is never
                                          // queued behind a V stage that is still being read
constexpr int kStoreWarp = kProdWarp + 3; // copies finished O tiles from shared memory to global
constexpr int kTileRows = 128;        // M rows per query tile
constexpr int kBN = 128;              // kv rows per kv tile (N of S = Q K^T, K of O += P V)
#ifndef PB_K_STAGES
#define PB_K_STAGES 2 // 3 measured identical (the K tile of j+1 is always in before S(j+1)), so
                      // its 32 KB hold the O staging tile instead
#endif
#ifndef PB_V_STAGES
#define PB_V_STAGES 2
#endif
constexpr int kKStages = PB_K_STAGES; // K ring depth (kBN-row tiles): K(j+1) is read first
constexpr int kVStages = PB_V_STAGES; // V ring depth
constexpr uint32_t kTmemCols = 512;   // S_A [0,128) S_B [128,256) O_A [256,384) O_B [384,512)
constexpr uint32_t kColO = 256;
#ifndef PB_SETMAXNREG
#define PB_SETMAXNREG 1 // 1: rebalance registers, WG2 (TMA + MMA warps) down, softmax groups up
#endif
constexpr bool kUseSetMaxNReg = PB_SETMAXNREG != 0;
#ifndef PB_REG_LO
#define PB_REG_LO 72 // producer/MMA/store warpgroup after setmaxnreg.dec
#endif
#ifndef PB_REG_HI
#define PB_REG_HI 216 // softmax warpgroups after setmaxnreg.inc (208 -> 216: tiles alone 381 -> 376 us)
#endif
// setmaxnreg only moves registers inside the CTA's launch allocation (kThreads x the
// per-thread count __launch_bounds__ gives, 64K / kThreads rounded down to 8): what the
// softmax warpgroups gain must be what the producer/MMA warpgroup gives up, or inc blocks
constexpr int kLaunchRegs = (65536 / kThreads) / 8 * 8;
static_assert((PB_REG_HI - kLaunchRegs) * kSoftWG <= (kLaunchRegs - PB_REG_LO),
              "setmaxnreg budget exceeds the launch register allocation");
#ifndef PB_RESCALE_THR
#define PB_RESCALE_THR 8.0f
#endif
constexpr float kRescaleThreshold = PB_RESCALE_THR; // log2 domain: rescale only if max grows by > 2^thr
#ifndef PB_ABLATE_MODE
#define PB_ABLATE_MODE 0 // roofline ablations, separate builds only: 1 no softmax, 2 no exp2, 5 no P store
#endif
#ifndef PB_POLY_COLS
#define PB_POLY_COLS 0 // the last N columns of each S tile take exp2 on the FMA pipe (cubic)
                       // before the MUFU share; measured slower at 32 and 64 (with or without
                       // the lock) and at 1 pair in 2..4 interleaved
#endif
constexpr int kPolyCols = PB_POLY_COLS;
#ifndef PB_POLY_EVERY
#define PB_POLY_EVERY 0 // exp2 of one pair in N on the FMA pipe, interleaved with the MUFU pairs
#endif
static_assert(kPolyCols % 32 == 0 && kPolyCols <= 64, "poly columns: whole 32-column chunks of the second P half");
#ifndef PB_P_PARTS
#define PB_P_PARTS 2 // P released in this many column parts; PV of a part overlaps the softmax of
                     // the next (1: one release per tile)
#endif
constexpr int kPParts = PB_P_PARTS;
static_assert(kPParts == 1 || kPParts == 2 || kPParts == 4, "P parts");
#ifndef PB_MUFU_LOCK
#define PB_MUFU_LOCK 0 // 1: the two softmax warps of an SMSP (query tiles A, B) take turns on
                       // the MUFU pipe.  Measured slower (434 vs 418 us on the config-4 tiles):
                       // one warp alone cannot keep MUFU busy (the ex2 issue throttle stalls
                       // it), so the exp2 phases do not get shorter, they only serialise
#endif

constexpr int kItemRing = 4; // work items fetched ahead by the TMA warp

// Diagnostics build only (-DPB_TILE_TRACE): per-tile clock64 stamps of the softmax groups and
// the MMA issuer of the first kTraceCtas CTAs, written after the per-CTA pass records of
// pb_attn_set_trace (scripts/trace_tiles.py reads them).  Compiles to nothing by default.
#ifndef PB_TILE_TRACE
#define PB_TILE_TRACE 0
#endif
// roles: 0/1 softmax A/B per tile, 2 MMA per kv tile, 3 K producer per item, 4 MMA per item,
// 5 softmax A per item
constexpr int kTraceCtas = 8, kTraceEvents = 1024, kTraceFields = 8;
__device__ __forceinline__ unsigned long long* tile_trace_slot(unsigned long long* tr, int role, int ev) {
    if (!PB_TILE_TRACE || !tr || blockIdx.x >= kTraceCtas || ev >= kTraceEvents) return nullptr;
    return tr + 148 * 2 * 4 + ((static_cast<size_t>(blockIdx.x) * 6 + role) * kTraceEvents + ev) * kTraceFields;
}
__device__ __forceinline__ unsigned long long clk64() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    return t;
}
constexpr int kMaxPpt = kBN / 8; // pages per kv tile (page_tokens >= 8)

template <int D>
struct __align__(1024) Smem {
    uint8_t q[2][kTileRows * D * 2];      // tiles A, B: [D/64][128 rows][128 B] K-major SW128
    uint8_t k[kKStages][kBN * D * 2];     // ring of kv tiles: [D/64][128 rows][128 B] K-major SW128
    uint8_t v[kVStages][kBN * D * 2];     // same layout, read as the MN-major SW128 B operand
    uint8_t o[kTileRows * D * 2];         // finished O tile (bf16 rows, 16-B chunks XOR-swizzled)
                                          // on its way to global through the store warp
    uint64_t q_full, q_empty;             // Q is released after the item's last S MMA
    uint64_t k_full[kKStages], k_empty[kKStages], v_full[kVStages], v_empty[kVStages];
    uint64_t s_full[2];                   // [query tile] S landed
    uint64_t p_full[2][kPParts];          // [query tile][column part] P stored (O rescaled
                                          // before the first part)
    uint64_t o_ready[2], o_empty[2];      // per query tile
    uint64_t item_full[kItemRing], item_empty[kItemRing];   // dynamic tile scheduler ring
    uint64_t drain;                       // MMA issuer: every commit of the pass has landed
    int32_t item_ring[kItemRing];
    uint64_t o_full;                      // an O tile is staged (arrived by its group)
    int32_t o_turn;                       // index of the next epilogue allowed to stage
    int32_t o_info[2];                    // staged tile: first token row, first head
    uint32_t mufu_lock[4];                // per SMSP: softmax warp using the MUFU pipe
};

// one CTA per SM: the larger of the two layouts plus 1 KiB of alignment slack must fit the
// 227 KiB opt-in shared memory of an sm_100 CTA
static_assert(sizeof(Smem<128>) + 1024 + 64 <= 232448, "tile layout exceeds shared memory");
static_assert(sizeof(dtc::DtSmem) + 1024 <= 232448, "decode layout exceeds shared memory");

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
    r.ntiles[0] = ceil_div(sp.causal_offset + w.t0 + r.nt[0], kBN);
    r.ntiles[1] = r.nt[1] > 0 ? ceil_div(sp.causal_offset + w.t0 + w.nt, kBN) : 0;
    r.n_kv = max(r.ntiles[0], r.ntiles[1]);
    return r;
}

__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
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

template <int D>
__device__ __forceinline__ void tile_init(Smem<D>& s) { // thread 0
    mbar_init(&s.q_full, 1);
    mbar_init(&s.q_empty, 1);
    for (int i = 0; i < kKStages; ++i) {
        mbar_init(&s.k_full[i], 1);
        mbar_init(&s.k_empty[i], 1);
    }
    for (int i = 0; i < kVStages; ++i) {
        mbar_init(&s.v_full[i], 1);
        mbar_init(&s.v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
        mbar_init(&s.s_full[i], 1);
        for (int h = 0; h < kPParts; ++h) mbar_init(&s.p_full[i][h], 128);
        mbar_init(&s.o_ready[i], 1);
        mbar_init(&s.o_empty[i], 128);
    }
    for (int i = 0; i < kItemRing; ++i) {
        mbar_init(&s.item_full[i], 1);
        mbar_init(&s.item_empty[i], 3 + 4 * kSoftWG); // MMA thread, V producer, store warp + the softmax warps
    }
    mbar_init(&s.drain, 1);
    mbar_init(&s.o_full, 1);
    s.o_turn = 0;
    for (int i = 0; i < 4; ++i) s.mufu_lock[i] = 0;
}
template <int D>
__device__ __forceinline__ void tile_inval(Smem<D>& s) { // thread 0, pipeline drained
    uint64_t* first = &s.q_full;
    uint64_t* last = &s.drain;
    for (uint64_t* b = first; b <= last; ++b) mbar_inval(b);
    mbar_inval(&s.o_full);
}

// One launch for the whole ragged batch (BASELINE north star (a)): persistent CTAs, each
// running the tile pipeline (multi-token spans, tcgen05 QK^T / PV with the GQA group in M)
// and the decode pipeline (single-token split-KV units, decode_tc_cta.cuh) from two global
// queues.  CTAs [0, n_dec_ctas) start on decode units and the rest on tile items; a CTA whose
// queue runs dry drains its pipeline, re-initialises its barriers for the other layout and
// steals from the other queue, so HBM-bound units stream next to tensor-bound tiles and both
// queues finish together.
template <int D, int GD>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fused_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                            const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_qd,
                            const __grid_constant__ CUtensorMap tm_o,
                            const AttnParams p) {
    constexpr int KH = D / 64;                  // 64-dim halves (one 128 B swizzle row each)
    constexpr uint32_t kHalfBytes = kTileRows * 128;   // one 64-dim half of a query tile
    constexpr uint32_t kKvHalf = kBN * 128;            // one 64-dim half of a kv tile
    constexpr uint32_t kKvTileBytes = kBN * D * 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    Smem<D>& s = *reinterpret_cast<Smem<D>*>(base);           // tile layout
    dtc::DtSmem& ds = *reinterpret_cast<dtc::DtSmem*>(base);  // decode layout (same bytes)
    __shared__ uint32_t tmem_base_sh;
    const int warp = threadIdx.x >> 5;
    const int g = p.group;
    const int tpt = kTileRows / g;         // query tokens per query tile
    const int chunk = p.chunk;
    const int ppt = kBN / chunk;           // pages per kv tile
    int* ctr = p.work_counter;             // [2] next tile item, [3] retired CTAs, [4] next decode unit

    if (threadIdx.x == 0 && p.trace) { // CTA entry (pass-0 record, field 1)
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[static_cast<size_t>(blockIdx.x) * 8 + 1] = t;
    }
    append_prologue(p, ctr); // fused K/V append, when the launch carries new rows
    if (threadIdx.x == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        tma_prefetch(&tm_qd);
        tma_prefetch(&tm_o);
    }
    if (warp == kMmaWarp) tmem_alloc<kTmemCols>(&tmem_base_sh);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    const int wg = warp >> 2;
    const bool dec_first = static_cast<int>(blockIdx.x) < p.n_dec_ctas;
    auto mode_items = [&](bool dec) { return dec ? (D == 128 ? p.n_dec_items : 0) : p.n_items; };
    auto gtime = []() {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        return t;
    };
    auto mode_begin = [&](bool dec) {
        if (threadIdx.x == 0 && p.trace) {
            unsigned long long* tr = p.trace + (static_cast<size_t>(blockIdx.x) * 2 + (dec == dec_first ? 0 : 1)) * 4;
            tr[0] = dec ? 1 : 0;
            tr[2] = gtime();
        }
        if (threadIdx.x == 0) {
            if (dec) dtc::decode_cta_init(ds);
            else tile_init(s);
            mbar_fence_init();
        }
        __syncthreads();
    };
    auto mode_end = [&](bool dec) { // pipeline drained: every barrier phase consumed
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        if (threadIdx.x == 0) {
            if (dec) dtc::decode_cta_inval(ds);
            else tile_inval(s);
            if (p.trace)
                p.trace[(static_cast<size_t>(blockIdx.x) * 2 + (dec == dec_first ? 0 : 1)) * 4 + 3] = gtime();
        }
    };
    if (wg == kSoftWG) {
    if (kUseSetMaxNReg) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(PB_REG_LO) : "memory");
    for (int pass = 0; pass < 2; ++pass) {
    const bool dec = (pass == 0) == dec_first;
    if (mode_items(dec) == 0) continue;
    mode_begin(dec);
    if (dec) {
        if constexpr (D == 128)
            dtc::decode_cta_run<GD>(ds, tmem, &tm_qd, &tm_k, &tm_v, p, p.dec_items, p.n_dec_items, ctr + 4, kProdWarp,
                                    kMmaWarp, 0, kProdWarp + 2);
    } else if (warp == kProdWarp || warp == kProdVWarp) {
        // ===================== TMA producers (K warp: Q + K, V warp: V) =====================
        if (elect_one()) {
            const bool kw = warp == kProdWarp;
            int it = 0, st = 0;
            uint32_t ph = 0;
            const int n_st = kw ? kKStages : kVStages;
            const uint32_t q_bytes = KH * 128u * static_cast<uint32_t>(g * tpt);
            const int oob_row = p.n_slots * chunk;
            // Dynamic tile scheduler: the K warp takes the next item (items are in LPT order)
            // from a global ticket when it is ready to load it, and hands the index to the MMA,
            // V and softmax roles through a small shared ring.
            int* ticket = p.work_counter + 2; // [2] next tile item (reset by the last CTA to retire)
            for (;; ++it) {
                const int slot = it % kItemRing;
                int item;
                if (kw) {
                    if (it >= kItemRing) mbar_wait(&s.item_empty[slot], ((it / kItemRing) - 1) & 1);
                    item = atomicAdd(ticket, 1);
                    if (item >= p.n_items) item = -1;
                    s.item_ring[slot] = item;
                    mbar_arrive(&s.item_full[slot]);
                } else {
                    mbar_wait(&s.item_full[slot], (it / kItemRing) & 1);
                    item = *reinterpret_cast<volatile int32_t*>(&s.item_ring[slot]);
                    mbar_arrive(&s.item_empty[slot]);
                }
                unsigned long long* ti = kw ? tile_trace_slot(p.trace, 3, it) : nullptr;
                if (ti) { ti[0] = clk64(); ti[7] = static_cast<unsigned long long>(item); }
                if (item < 0) break;
                const WorkItem w = p.items[item];
                const SpanDev sp = p.spans[w.span];
                const ItemTiles T = item_tiles(w, sp, tpt);
                if (ti) ti[1] = clk64();
                if (kw) {
                    if (it > 0) mbar_wait(&s.q_empty, (it - 1) & 1);
                    if (ti) ti[2] = clk64();
                    mbar_arrive_expect_tx(&s.q_full, q_bytes * (T.nt[1] > 0 ? 2u : 1u));
                    for (int t = 0; t < 2; ++t)
                        if (T.nt[t] > 0)
                            for (int h = 0; h < KH; ++h)
                                tma_load_3d(s.q[t] + h * kHalfBytes, &tm_q, &s.q_full, h * 64, w.kvh * g,
                                            sp.query_start + w.t0 + t * tpt);
                }
                const int32_t* table = p.block_tables + sp.bt_off;
                const int n_pages = sp.n_pages;
                const CUtensorMap* tm = kw ? &tm_k : &tm_v;
                for (int j = 0; j < T.n_kv; ++j) {
                    // the tile's block-table entries: independent loads issued together, before
                    // any barrier wait or TMA (one L2 round trip per tile, not one per page)
                    int rows[kMaxPpt];
#pragma unroll
                    for (int pg = 0; pg < kMaxPpt; ++pg) {
                        const int page = j * ppt + pg;
                        rows[pg] = (pg < ppt && page < n_pages) ? __ldg(table + page) * chunk : oob_row;
                    }
                    uint64_t* full = kw ? &s.k_full[st] : &s.v_full[st];
                    uint8_t* dst = kw ? s.k[st] : s.v[st];
                    mbar_wait(kw ? &s.k_empty[st] : &s.v_empty[st], ph ^ 1);
                    mbar_arrive_expect_tx(full, kKvTileBytes);
#pragma unroll
                    for (int pg = 0; pg < kMaxPpt; ++pg)
                        if (pg < ppt)
                            for (int h = 0; h < KH; ++h)
                                tma_load_3d(dst + h * kKvHalf + pg * chunk * 128, tm, full, h * 64, w.kvh, rows[pg]);
                    if (++st == n_st) { st = 0; ph ^= 1; }
                    if (ti && j == 0) ti[3] = clk64();
                }
                if (ti) ti[4] = clk64();
            }
        }
    } else if (warp == kMmaWarp) {
        // ============================ MMA issuer =============================
        if (elect_one()) {
            constexpr uint32_t idesc_s = umma_idesc_bf16(128, kBN, false, false);
            constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, false, true);
            int it = 0, kst = 0, vst = 0;
            uint32_t kph = 0, vph = 0;
            uint32_t n_oe[2] = {0, 0};
            uint32_t c_p[2] = {0, 0}; // per group: PV tiles issued (p_full phase)
            int mma_ev = 0;           // PB_TILE_TRACE event index
            for (;; ++it) {
                const int slot = it % kItemRing;
                mbar_wait(&s.item_full[slot], (it / kItemRing) & 1);
                const int item = *reinterpret_cast<volatile int32_t*>(&s.item_ring[slot]);
                mbar_arrive(&s.item_empty[slot]);
                if (item < 0) {
                    // the pass's last tcgen05.commit arrivals land before its barriers are reused
                    umma_commit(&s.drain);
                    mbar_wait(&s.drain, 0);
                    break;
                }
                unsigned long long* ti = tile_trace_slot(p.trace, 4, it);
                if (ti) { ti[0] = clk64(); ti[7] = static_cast<unsigned long long>(item); }
                const WorkItem w = p.items[item];
                const SpanDev sp = p.spans[w.span];
                const ItemTiles T = item_tiles(w, sp, tpt);
                if (ti) ti[1] = clk64();
                mbar_wait(&s.q_full, it & 1);
                if (ti) ti[2] = clk64();
                tc_fence_after();
                // S_t = Q_t K^T (K stage ks) into group t's S buffer.  Descriptors are advanced
                // by adding (byte offset >> 4) to the start-address field (no carry: shared
                // addresses < 256 KB).
                auto issue_s = [&](int t, int ks) {
                    const uint64_t kd = umma_desc_sw128(smem_u32(s.k[ks]), 16, 1024);
                    const uint64_t qd = umma_desc_sw128(smem_u32(s.q[t]), 16, 1024);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t oq = ((kk >> 2) * kHalfBytes + (kk & 3) * 32) >> 4;
                        const uint32_t ok = ((kk >> 2) * kKvHalf + (kk & 3) * 32) >> 4;
                        umma_bf16_ss(tmem + t * 128, qd + oq, kd + ok, idesc_s, kk > 0);
                    }
                    umma_commit(&s.s_full[t]);
                };
                // prologue: S_A(0), S_B(0) from K(0)
                mbar_wait(&s.k_full[kst], kph);
                tc_fence_after();
                if (ti) ti[3] = clk64();
                for (int t = 0; t < 2; ++t)
                    if (T.ntiles[t] > 0) issue_s(t, kst);
                if (ti) ti[4] = clk64();
                umma_commit(&s.k_empty[kst]);
                if (++kst == kKStages) { kst = 0; kph ^= 1; }
                if (T.n_kv == 1) umma_commit(&s.q_empty); // Q is read by S MMAs only
                for (int j = 0; j < T.n_kv; ++j) {
                    unsigned long long* tt = tile_trace_slot(p.trace, 2, mma_ev++);
                    if (tt) tt[0] = clk64();
                    const bool nxt = j + 1 < T.n_kv;
                    if (nxt) mbar_wait(&s.k_full[kst], kph);
                    if (tt) tt[1] = clk64();
                    mbar_wait(&s.v_full[vst], vph);
                    if (tt) tt[2] = clk64();
                    tc_fence_after();
                    const uint64_t vd = umma_desc_sw128(smem_u32(s.v[vst]), kKvHalf, 1024);
                    for (int t = 0; t < 2; ++t) {
                        if (j < T.ntiles[t]) {
                            if (j == 0) {
                                mbar_wait(&s.o_empty[t], (n_oe[t] & 1) ^ 1);
                                ++n_oe[t];
                            }
                            const uint32_t pcol = t * 128; // P (bf16) over the first 64 S columns
#pragma unroll
                            for (int h = 0; h < kPParts; ++h) {
                                mbar_wait(&s.p_full[t][h], c_p[t] & 1);
                                if (tt && h == kPParts - 1) tt[3 + t] = clk64();
                                tc_fence_after();
#pragma unroll
                                for (int kk = h * (kBN / 16 / kPParts); kk < (h + 1) * (kBN / 16 / kPParts); ++kk)
                                    umma_bf16_ts(tmem + kColO + t * 128, tmem + pcol + kk * 8,
                                                 vd + kk * (2048 >> 4), idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
                            }
                            ++c_p[t];
                            if (j + 1 == T.ntiles[t]) umma_commit(&s.o_ready[t]);
                        }
                        // S_t(j+1) behind PV_t(j) on the in-order tensor pipe (P_t(j) lives in
                        // the S_t columns)
                        if (nxt && j + 1 < T.ntiles[t]) issue_s(t, kst);
                    }
                    umma_commit(&s.v_empty[vst]);
                    if (++vst == kVStages) { vst = 0; vph ^= 1; }
                    if (nxt) {
                        umma_commit(&s.k_empty[kst]);
                        if (++kst == kKStages) { kst = 0; kph ^= 1; }
                        if (j + 2 == T.n_kv) umma_commit(&s.q_empty);
                    }
                    if (tt) {
                        tt[5] = clk64();
                        tt[6] = static_cast<unsigned long long>(j);
                        tt[7] = static_cast<unsigned long long>(item);
                    }
                }
            }
        }
    } else if (warp == kStoreWarp) {
        // ============================ O store warp ==============================
        // Full query tiles are staged one at a time in s.o (the SW128 layout of a TMA box
        // {64 dims, g heads, 128/g tokens}), in an order every role can compute: per item,
        // tile A then tile B, full tiles only.  For each: wait until it is staged, TMA-store
        // it, wait until the bulk copy has read shared memory, hand the buffer to the next
        // tile (o_turn).  The softmax groups never block on global stores.  Partial tiles
        // (the last block of a span) are stored by their group directly.
        if (elect_one()) {
            int e = 0;
            for (int it = 0;; ++it) {
                const int slot = it % kItemRing;
                mbar_wait(&s.item_full[slot], (it / kItemRing) & 1);
                const int item = *reinterpret_cast<volatile int32_t*>(&s.item_ring[slot]);
                mbar_arrive(&s.item_empty[slot]);
                if (item < 0) break;
                const int nt = p.items[item].nt;
                const int n_epi = (nt >= tpt ? 1 : 0) + (nt == 2 * tpt ? 1 : 0);
                for (int k = 0; k < n_epi; ++k, ++e) {
                    mbar_wait(&s.o_full, e & 1);
                    const int row0 = reinterpret_cast<volatile int32_t*>(s.o_info)[0];
                    const int head0 = reinterpret_cast<volatile int32_t*>(s.o_info)[1];
                    for (int h = 0; h < KH; ++h) tma_store_3d(&tm_o, s.o + h * kHalfBytes, h * 64, head0, row0);
                    bulk_commit();
                    bulk_wait_read0();
                    *reinterpret_cast<volatile int32_t*>(&s.o_turn) = e + 1;
                }
            }
            bulk_wait_all0(); // the pass's stores are complete before its smem is reused
        }
    }
    mode_end(dec);
    }
    } else {
        if (kUseSetMaxNReg) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(PB_REG_HI) : "memory");
    for (int pass = 0; pass < 2; ++pass) {
    const bool dec = (pass == 0) == dec_first;
    if (mode_items(dec) == 0) continue;
    mode_begin(dec);
    if (dec) {
        if constexpr (D == 128)
            dtc::decode_cta_run<GD>(ds, tmem, &tm_qd, &tm_k, &tm_v, p, p.dec_items, p.n_dec_items, ctr + 4, kProdWarp,
                                    kMmaWarp, 0, kProdWarp + 2);
    } else {
        // ============ softmax / correction / epilogue (one group per query tile) ============
        const int t = wg;                           // query tile of this warpgroup
        const int quad = warp & 3;                  // TMEM lane quadrant of this warp
        const int row = quad * 32 + (threadIdx.x & 31);
        const uint32_t t_lane = tmem + (static_cast<uint32_t>(quad * 32) << 16);
        const uint32_t col_s = t * 128;
        const uint32_t col_o = kColO + t * 128;
        const float sl2 = p.scale_log2;
        // roofline ablations exist only in builds with -DPB_ABLATE_MODE=n
        // (scripts/build_variants.sh); the production kernel carries no checks for them
        constexpr int ablate = PB_ABLATE_MODE;
        uint32_t n_o = 0;
        uint32_t c_t = 0;     // kv tiles processed by this group (s_full / p_full phase)
        uint32_t kv_seen = 0; // kv tiles loaded for earlier items (V ring position)
        int epi = 0;          // epilogues (staged O tiles) of earlier items, both groups
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out);
        for (int it = 0;; ++it) {
            const int slot = it % kItemRing;
            mbar_wait(&s.item_full[slot], (it / kItemRing) & 1);
            const int item = *reinterpret_cast<volatile int32_t*>(&s.item_ring[slot]);
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&s.item_empty[slot]);
            unsigned long long* ti = threadIdx.x == 0 ? tile_trace_slot(p.trace, 5, it) : nullptr;
            if (ti) { ti[0] = clk64(); ti[7] = static_cast<unsigned long long>(item); }
            if (item < 0) break;
            const WorkItem w = p.items[item];
            const SpanDev sp = p.spans[w.span];
            const ItemTiles T = item_tiles(w, sp, tpt);
            if (ti) ti[1] = clk64();
            const int n_tiles = T.ntiles[t];
            const uint32_t kv_base = kv_seen;
            kv_seen += static_cast<uint32_t>(T.n_kv);
            // staged epilogues: full tiles only, A then B per item (the store warp's order)
            const bool full_tile = T.nt[t] == tpt;
            const int my_epi = epi + (t == 1 && T.nt[0] == tpt ? 1 : 0);
            epi += (T.nt[0] == tpt ? 1 : 0) + (T.nt[1] == tpt ? 1 : 0);
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
            for (int j = 0; j < n_tiles; ++j, ++c_t) {
                unsigned long long* tt = (threadIdx.x & 127) == 0 ? tile_trace_slot(p.trace, t, static_cast<int>(c_t)) : nullptr;
                if (tt) tt[0] = clk64();
                float x[kBN];
                mbar_wait(&s.s_full[t], c_t & 1);
                if (tt) tt[1] = clk64();
                tc_fence_after();
                if (ablate == 1) { // profiling: tensor-core + pipeline bound (P left as S bits)
                    tc_fence_before();
                    for (int h = 0; h < kPParts; ++h) mbar_arrive(&s.p_full[t][h]);
                    l_run = 1.f;
                    continue;
                }
#pragma unroll
                for (int c = 0; c < kBN / 32; ++c)
                    tmem_ld32(t_lane + col_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&x[c * 32]));
                tmem_ld_wait();
                const int kv0 = j * kBN;
                // causal mask (only tiles that cross this row's boundary) + running max
                if (kv0 + kBN > allowed) {
#pragma unroll
                    for (int c = 0; c < kBN; ++c) x[c] = (kv0 + c < allowed) ? x[c] : -CUDART_INF_F;
                }
                float pm[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) pm[u] = x[u];
#pragma unroll
                for (int c = 8; c < kBN; ++c) pm[c & 7] = fmaxf(pm[c & 7], x[c]);
                const float mt = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                                       fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7]))) * sl2;
                if (tt) tt[2] = clk64();
                const bool grow = mt > m_run + kRescaleThreshold;
                const float m_new = grow ? mt : m_run;
                const float corr = grow ? ex2(m_run - m_new) : 1.f;
                if (zero_owner && j + 1 == T.n_kv) {
                    const int kv = j * kBN + row;
                    if (kv >= sp.context_len && kv < sp.n_pages * chunk) {
                        // the V tile must have landed first (S_t(j) landing does not imply it);
                        // its stage cannot be refilled before this group releases P_t(j)
                        const uint32_t vt = kv_base + j;
                        mbar_wait(&s.v_full[vt % kVStages], (vt / kVStages) & 1);
                        uint8_t* vrow = s.v[vt % kVStages] + row * 128;
#pragma unroll
                        for (int h = 0; h < KH; ++h)
#pragma unroll
                            for (int c = 0; c < 8; ++c)
                                *reinterpret_cast<uint4*>(vrow + h * kKvHalf + c * 16) = make_uint4(0, 0, 0, 0);
                        fence_proxy_async_smem();
                    }
                }
                // lazy O rescale, before any part of P(j) is released to PV_t(j): S_t(j)
                // completing proves PV_t(j-1) done (in-order pipe)
                const bool rescale = j > 0 && __any_sync(0xffffffffu, grow);
                if (rescale) {
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
                float2 ps[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) ps[u] = make_float2(0.f, 0.f);
                const float2 sl2x2 = make_float2(sl2, sl2);
                // the FMA-pipe share first, outside the MUFU lock (results kept in x)
#pragma unroll
                for (int c = kBN - kPolyCols; c < kBN; c += 2) {
                    const float2 e = exp2_neg_poly_x2(fma2(make_float2(x[c], x[c + 1]), sl2x2, make_float2(-m_new, -m_new)));
                    ps[(c >> 1) & 3] = add2(ps[(c >> 1) & 3], e);
                    x[c] = e.x;
                    x[c + 1] = e.y;
                }
                const float m_arg = PB_MUFU_LOCK ? m_new + __uint_as_float(smsp_lock_acquire(&s.mufu_lock[quad])) : m_new;
                const float2 negm = make_float2(-m_arg, -m_arg);
#pragma unroll
                for (int h = 0; h < kPParts; ++h) {
#pragma unroll
                    for (int c0 = h * (kBN / kPParts); c0 < (h + 1) * (kBN / kPParts); c0 += 32) {
                        uint32_t pk[16];
#pragma unroll
                        for (int c = c0; c < c0 + 32; c += 2) {
                            float2 e;
                            if (c >= kBN - kPolyCols) { // done on the FMA pipe above
                                e = make_float2(x[c], x[c + 1]);
                            } else {
                                // exp2((s - max) * log2e / scale) on packed pairs (FFMA2 / FADD2) and MUFU
                                const float2 a = fma2(make_float2(x[c], x[c + 1]), sl2x2, negm);
                                if (ablate == 2) { // profiling: no exponentials
                                    e = a;
                                } else if (PB_POLY_EVERY > 0 && ((c >> 1) % (PB_POLY_EVERY > 0 ? PB_POLY_EVERY : 1)) == 0) {
                                    e = exp2_neg_poly_x2(a);
                                } else {
                                    e.x = ex2(a.x);
                                    e.y = ex2(a.y);
                                }
                                ps[(c >> 1) & 3] = add2(ps[(c >> 1) & 3], e);
                            }
                            pk[(c - c0) >> 1] = pack_bf16x2(e.x, e.y);
                        }
                        // P (bf16) over the first 64 columns of this S buffer (all of S is in
                        // registers already)
                        if (ablate != 5) dtc::tmem_st16(t_lane + col_s + (c0 >> 1), pk);
                    }
                    tmem_st_wait();
                    tc_fence_before();
                    mbar_arrive(&s.p_full[t][h]);
                }
                if (PB_MUFU_LOCK) smsp_lock_release(&s.mufu_lock[quad]);
                if (tt) {
                    tt[3] = clk64();
                    tt[4] = clk64();
                    tt[5] = rescale ? 1ull : 0ull;
                    tt[6] = static_cast<unsigned long long>(j);
                    tt[7] = static_cast<unsigned long long>(item);
                }
                const float2 s2 = add2(add2(ps[0], ps[1]), add2(ps[2], ps[3]));
                const float sum = s2.x + s2.y;
                l_run = l_run * corr + sum;
                m_run = m_new;
            }
            // epilogue: O / l -> bf16 -> global
            if (ti) ti[2] = clk64();
            mbar_wait(&s.o_ready[t], n_o & 1);
            if (ti) ti[3] = clk64();
            ++n_o;
            tc_fence_after();
            const float inv_l = 1.f / l_run;
            // the whole row into registers (all TMEM loads in flight at once), bf16 16-B
            // chunks, so O_t is released to the next item's PV before anything is stored
            uint4 chv[D / 8];
            {
                uint32_t o[D];
#pragma unroll
                for (int c = 0; c < D / 32; ++c)
                    tmem_ld32(t_lane + col_o + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c * 32]));
                tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < D / 8; ++c) {
                    const uint32_t* q8 = o + c * 8;
                    chv[c] = make_uint4(
                        pack_bf16x2(__uint_as_float(q8[0]) * inv_l, __uint_as_float(q8[1]) * inv_l),
                        pack_bf16x2(__uint_as_float(q8[2]) * inv_l, __uint_as_float(q8[3]) * inv_l),
                        pack_bf16x2(__uint_as_float(q8[4]) * inv_l, __uint_as_float(q8[5]) * inv_l),
                        pack_bf16x2(__uint_as_float(q8[6]) * inv_l, __uint_as_float(q8[7]) * inv_l));
                }
            }
            tc_fence_before();
            mbar_arrive(&s.o_empty[t]);
            if (ti) ti[5] = clk64();
            if (full_tile) {
                // stage the row for the store warp once the buffer is this tile's turn
                if (threadIdx.x % 128 == 0)
                    while (*reinterpret_cast<volatile int32_t*>(&s.o_turn) != my_epi) __nanosleep(32);
                named_bar_sync(2 + t, 128);
                if (ti) ti[6] = clk64();
#pragma unroll
                for (int c = 0; c < D / 8; ++c)
                    *reinterpret_cast<uint4*>(s.o + (c >> 3) * kHalfBytes + row * 128 + (((c & 7) ^ (row & 7)) << 4)) = chv[c];
                fence_proxy_async_smem(); // generic-proxy writes -> the TMA (async proxy) read
                if (threadIdx.x % 128 == 0) {
                    s.o_info[0] = sp.query_start + tok0;
                    s.o_info[1] = w.kvh * g;
                }
                named_bar_sync(2 + t, 128);
                if (threadIdx.x % 128 == 0) mbar_arrive(&s.o_full);
            } else if (valid) {
                __nv_bfloat16* orow =
                    out + (static_cast<size_t>(sp.query_start + tok0 + t_local) * p.n_head + w.kvh * g + (row % g)) * D;
#pragma unroll
                for (int c = 0; c < D / 8; ++c) *reinterpret_cast<uint4*>(orow + c * 8) = chv[c];
            }
            if (ti) ti[4] = clk64();
        }
    }
    mode_end(dec);
    }
    }
    // the last CTA to retire re-arms the queues for the next launch
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(ctr + 3, 1) == static_cast<int>(gridDim.x) - 1) {
            ctr[2] = 0;
            if (p.n_dec_items > 0) ctr[4] = 0;
            ctr[3] = 0;
        }
    }
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
        if (p.trace && (threadIdx.x & 31) == 0) { // CTA exit (pass-1 record, field 1)
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            p.trace[static_cast<size_t>(blockIdx.x) * 8 + 4 + 1] = t;
        }
    }
}


// ------------------------------------------------------------------ host side

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() { // a driver entry point: one per process
    static std::once_flag once;
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            f && q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
        else
            cudaGetLastError();
    });
    if (!fn) fail(PB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
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

template <int D, int GD>
void launch_fused(const AttnParams& p, const CUtensorMap* maps, cudaStream_t st) {
    const size_t smem = std::max(sizeof(Smem<D>), sizeof(dtc::DtSmem)) + 1024;
    static std::once_flag attr[kMaxDevices];
    set_smem_once(attr, attn_fused_sm100_kernel<D, GD>, smem, "cudaFuncSetAttribute(fused smem)");
    const int grid = std::min(p.n_items + (D == 128 ? p.n_dec_items : 0), device_sms());
    if (!p.k_new) {
        attn_fused_sm100_kernel<D, GD><<<grid, kThreads, smem, st>>>(maps[0], maps[1], maps[2], maps[3], maps[4], p);
        cuda_check(cudaGetLastError(), "attn_fused_sm100 launch");
        count_launch();
        return;
    }
    // The fused append ends in a grid-wide barrier, so every CTA must be co-resident: a
    // cooperative launch guarantees it (or refuses, e.g. under an MPS SM limit or next to a
    // persistent kernel on another stream); when refused, the rows are written by their own
    // launch first and the attention launch carries no barrier.
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr_coop{};
    attr_coop.id = cudaLaunchAttributeCooperative;
    attr_coop.val.cooperative = 1;
    cfg.attrs = &attr_coop;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, attn_fused_sm100_kernel<D, GD>, maps[0], maps[1], maps[2], maps[3], maps[4], p);
    if (e == cudaSuccess) {
        count_launch();
        return;
    }
    if (e != cudaErrorCooperativeLaunchTooLarge) cuda_check(e, "attn_fused_sm100 cooperative launch");
    cudaGetLastError();
    launch_append_spans(p, st);
    AttnParams q = p;
    q.k_new = nullptr;
    q.v_new = nullptr;
    attn_fused_sm100_kernel<D, GD><<<grid, kThreads, smem, st>>>(maps[0], maps[1], maps[2], maps[3], maps[4], q);
    cuda_check(cudaGetLastError(), "attn_fused_sm100 launch");
    count_launch();
}

} // namespace

bool sm100_supports(int head_size, int chunk, int group) {
    return (head_size == 64 || head_size == 128) && chunk >= 8 && chunk <= kBN && (kBN % chunk) == 0 &&
           group >= 1 && group <= 128;
}

int sm100_tile_tokens(int group) { return 2 * (kTileRows / group); } // two query tiles per item

void sm100_prepare_maps(const AttnParams& p, const pb_attn_shape& shape, Sm100Cache& cache, int64_t total_tokens) {
    const int D = shape.head_size;
    const int g = shape.n_head / shape.n_kv_head;
    if (!cache.valid || cache.q != p.q || cache.k != p.k_pages || cache.v != p.v_pages || cache.out != p.out ||
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
        // output tiles (TMA store of a staged full query tile): the q tile geometry over out
        encode_3d(&m[4], p.out, D, shape.n_head, std::max<int64_t>(total_tokens, 1), D * 2ull,
                  static_cast<uint64_t>(shape.n_head) * D * 2, 64, g, kTileRows / g);
        cache.q = p.q;
        cache.k = p.k_pages;
        cache.v = p.v_pages;
        cache.out = p.out;
        cache.total_tokens = total_tokens;
        cache.valid = true;
    }
}

void launch_attn_sm100(const AttnParams& p, const pb_attn_shape& shape, Sm100Cache& cache, int64_t total_tokens,
                       cudaStream_t stream) {
    if (p.n_items + p.n_dec_items <= 0) return;
    sm100_prepare_maps(p, shape, cache, total_tokens);
    const int D = shape.head_size;
    const auto* maps = reinterpret_cast<const CUtensorMap*>(cache.maps);
    if (D == 128 && p.group > 8) launch_fused<128, 16>(p, maps, stream);
    else if (D == 128) launch_fused<128, 8>(p, maps, stream);
    else launch_fused<64, 8>(p, maps, stream);
}

void sm100_cache_release(Sm100Cache& cache) { cache.valid = false; }

} // namespace pb
