/*
 * pensieve_b200.h — C-ABI of the B200-native Pensieve hot path.
 *
 * Plain pointers and sizes only (no torch / C++ types).  Every entry point names the
 * reference interface it replaces (paths relative to /root/reference/proj).  Device
 * pointers are caller-owned; `stream` is a cudaStream_t passed as void* (NULL = legacy
 * default stream).  Calls are asynchronous on `stream` unless stated otherwise.
 *
 * Errors: every function returns pb_status; the codes map 1:1 onto the reference's
 * exception classes (include/kvsim/errors.hpp).  Validation happens before any mutation
 * or launch, exactly like the reference (which validates, then throws without side
 * effects).  pb_last_error() returns the message of the calling thread's last failure.
 */
#ifndef PENSIEVE_B200_H
#define PENSIEVE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum pb_status {
    PB_OK = 0,
    PB_ERR_DIMENSION_MISMATCH = 1,        /* kvsim::DimensionMismatch  errors.hpp:76-79 */
    PB_ERR_NUMERIC = 2,                   /* kvsim::NumericError       errors.hpp:82-85 */
    PB_ERR_ERROR = 3,                     /* kvsim::Error (base)       errors.hpp:12-15 */
    PB_ERR_INSUFFICIENT_DEVICE_MEMORY = 4,/* errors.hpp:23-26 */
    PB_ERR_INSUFFICIENT_HOST_MEMORY = 5,  /* errors.hpp:29-32 */
    PB_ERR_INVALID_CHUNK_STATE = 6,       /* errors.hpp:41-44 */
    PB_ERR_UNKNOWN_CONVERSATION = 7,      /* errors.hpp:34-37 */
    PB_ERR_CONFIG = 8,                    /* kvsim::ConfigError */
    PB_ERR_NOT_ENOUGH_EVICTABLE = 9,      /* kvsim::NotEnoughEvictable */
    PB_ERR_TRACE_MISSING = 10,            /* kvsim::TraceMissing */
    PB_ERR_CANNOT_SUSPEND_ALL = 11,       /* kvsim::CannotSuspendAll */
    PB_ERR_CUDA = 20,                     /* CUDA runtime/driver failure (no ref analogue) */
    PB_ERR_UNSUPPORTED = 21               /* shape outside what the kernels were built for */
} pb_status;

typedef enum pb_dtype { PB_F32 = 0, PB_BF16 = 1 } pb_dtype;

const char* pb_last_error(void);
const char* pb_version(void);
/* Number of kernel launches issued by this process so far (all pb_* kernels). */
uint64_t pb_launch_count(void);

/* ===================================================================== attention
 *
 * Layouts (identical to the reference):
 *   q, out : [total_tokens][n_head][head_size]              (RaggedQueryBatch::q,
 *                                                            include/kvsim/attention.hpp:53-65)
 *   pages  : [n_slots][chunk_size][n_kv_head][head_size]   (PagedKvStore keys / values,
 *                                                            include/kvsim/attention.hpp:33-49,
 *                                                            src/attention.cpp:60-71)
 *   spans  : SubRequest{query_start, query_len, context_len, causal_offset, block_table}
 *            (include/kvsim/batch.hpp:17-24); block tables as CSR: the slots of span s are
 *            block_tables[block_table_offsets[s] .. block_table_offsets[s+1]).
 * Semantics: query token i of span s attends to context positions [0, causal_offset+i];
 * query head h reads kv head h / (n_head / n_kv_head); scores are dot / scale
 * (src/attention.cpp:73-132).
 * dtype PB_F32 is the fp32 validation mode (fp32 SIMT, 1e-5 parity); PB_BF16 is the
 * production mode (bf16 storage, fp32 accumulation; tcgen05 tiles for multi-token spans,
 * split-KV SIMT for single-token spans).
 */
typedef struct pb_attn_shape {
    int32_t n_head;
    int32_t n_kv_head;
    int32_t head_size;
    int32_t chunk_size; /* tokens per page (= the reference's chunk_size) */
    int32_t n_slots;    /* pages in the pool */
    int32_t dtype;      /* pb_dtype of q, pages and out */
    double scale;       /* scores are divided by this (RaggedQueryBatch::scale) */
} pb_attn_shape;

typedef struct pb_attn_plan pb_attn_plan;

enum {
    PB_PLAN_SINGLE_TOKEN = 1, /* single_token_attention contract: every query_len == 1 */
    PB_PLAN_FORCE_SIMT = 2,   /* route every span through the SIMT kernel (diagnostics) */
    PB_PLAN_NO_SPLIT = 4,     /* never split a decode span's context across CTAs */
    PB_PLAN_SEPARATE_DECODE = 8, /* decode units in their own launch instead of the fused one */
    PB_PLAN_LPT_ORDER = 16       /* tile queue in strict LPT order (default: LPT below 8 items per
                                    SM, else grouped by span and kv head for L2 reuse); changes
                                    timing only, never the outputs */
};

/* Validates the batch exactly as check_batch (src/attention.cpp:23-48, minus the q
 * finiteness scan, which needs the data: see pb_attn_check_numerics) and builds the
 * host-side work list (prefill tiles + decode split units, heavy first).  The plan is
 * reusable across layers and calls.  Replaces the per-call
 * bookkeeping inside paged_multi_token_attention / single_token_attention. */
pb_status pb_attn_plan_create(const pb_attn_shape* shape, int32_t n_spans,
                              const int64_t* query_start, const int64_t* query_len,
                              const int64_t* context_len, const int64_t* causal_offset,
                              const int32_t* block_tables, const int64_t* block_table_offsets,
                              int64_t total_tokens, int32_t flags, pb_attn_plan** out);
/* Copies the plan's descriptors to the device on `stream` (first call allocates). */
pb_status pb_attn_plan_upload(pb_attn_plan* plan, void* stream);
/* Device workspace bytes pb_attn_run needs (split-KV partials + work-queue tickets).  The
 * tickets are zeroed on first use of a workspace buffer and are self-resetting after every
 * launch, so one workspace serves a whole layer loop and may be shared by several plans run
 * one after another; it must not be shared by two launches that can run at the same time
 * (give each stream its own).  The split-KV arrival counters live in the plan's own
 * descriptor buffer (zeroed by pb_attn_plan_upload), so runs of one plan are serialised:
 * run a plan on one stream at a time. */
size_t pb_attn_plan_workspace_bytes(const pb_attn_plan* plan);
/* Plan statistics: out[0] prefill tiles, [1] decode units, [2] split spans,
 * [3] algorithmic flops (4*n_head*d*sum allowed), [4] algorithmic bytes, [5] total tokens,
 * [6] SIMT tiles, [7] query rows covered by the work list (must equal tokens*n_head) */
void pb_attn_plan_stats(const pb_attn_plan* plan, double* out8);
/* The fused ragged paged attention launch(es) for one layer.  q, pages, out, workspace are
 * device pointers; the plan must have been uploaded.  Replaces
 * paged_multi_token_attention (src/attention.cpp:73-132) and single_token_attention
 * (:134-188) on the device. */
pb_status pb_attn_run(pb_attn_plan* plan, const void* q, const void* k_pages,
                      const void* v_pages, void* out, void* workspace, void* stream);
/* pb_attn_run with the paged K/V append fused in (the row-write loop of
 * qkv_project, src/attention.cpp:315-327): k_new / v_new hold the batch's new K/V rows
 * [total_tokens][n_kv_head][head_size] in query order; token i of span s is written to
 * position causal_offset[s] + i (page block_table[pos / chunk], row pos % chunk) before any
 * attention reads it.  Equivalent to pb_kv_append followed by pb_attn_run, in one launch on
 * the tcgen05 paths (a grid-wide barrier separates the writes from the reads). */
pb_status pb_attn_run_append(pb_attn_plan* plan, const void* q, const void* k_new, const void* v_new,
                             void* k_pages, void* v_pages, void* out, void* workspace, void* stream);
/* Layer loop with HOST q / out (the per-layer worker loop of PAPER.md:730-732 when the
 * projections live on the host side of the boundary): for l < n_layer, q_host[l] is copied
 * to the device, attended against k_pages[l] / v_pages[l] with the plan, and the result is
 * copied to out_host[l].  Layer l+1's H2D and layer l-1's D2H run on two copy streams while
 * layer l computes (two device staging buffers each for q and out, carved from `staging`,
 * pb_attn_stage_bytes(plan) bytes).  Asynchronous on `stream`: when `stream` completes,
 * every out_host[l] is written.  Host buffers should be pinned for the copies to overlap. */
size_t pb_attn_stage_bytes(const pb_attn_plan* plan);
/* The layer loop on device pointers: pb_attn_run(q[l], k_pages[l], v_pages[l], out[l]) for
 * l < n_layer, issued as ONE CUDA graph launch (the per-layer worker loop of
 * PAPER.md:730-732; each launch replaces paged_multi_token_attention / single_token_attention,
 * src/attention.cpp:73-188).  The graph is captured on the first call and replayed while the
 * pointers, n_layer, workspace and trace buffer stay the same (a change re-captures it); it
 * removes the per-launch gap between back-to-back layers.  Inside a caller's own stream
 * capture the launches are issued directly into the caller's graph.  Same stream and
 * workspace rules as pb_attn_run. */
pb_status pb_attn_run_layers(pb_attn_plan* plan, int32_t n_layer, const void* const* q,
                             const void* const* k_pages, const void* const* v_pages, void* const* out,
                             void* workspace, void* stream);
/* Diagnostics: when d_trace (device, >= 148 * 2 * 4 uint64) is set, the fused launch writes
 * per CTA and pass {mode (0 tile, 1 decode), items taken, begin ns, end ns}.  NULL disables. */
void pb_attn_set_trace(pb_attn_plan* plan, void* d_trace);
pb_status pb_attn_run_layers_host(pb_attn_plan* plan, int32_t n_layer, const void* const* q_host,
                                  void* const* out_host, const void* const* k_pages,
                                  const void* const* v_pages, void* staging, void* workspace,
                                  void* stream);
/* Optional device-side restatement of the reference's NumericError checks: q must be
 * finite (src/attention.cpp:30) and k_row[0] of every attended position must be finite
 * (:100-101).  Writes 0 / PB_ERR_NUMERIC into *d_flag (device int32). */
pb_status pb_attn_check_numerics(pb_attn_plan* plan, const void* q, const void* k_pages,
                                 int32_t* d_flag, void* stream);
void pb_attn_plan_destroy(pb_attn_plan* plan);

/* Host-buffer, synchronous mirrors of the reference's value-semantics API
 * (include/kvsim/attention.hpp:71-77).  q/keys/values/out are HOST fp32 arrays with the
 * reference layouts; with shape->dtype == PB_BF16 they are rounded to bf16 on upload and
 * the bf16 result is widened back.  Error behaviour matches the reference, including
 * NumericError for non-finite q / k_row[0]. */
pb_status pb_paged_multi_token_attention(const pb_attn_shape* shape, int32_t n_spans,
                                         const int64_t* query_start, const int64_t* query_len,
                                         const int64_t* context_len,
                                         const int64_t* causal_offset,
                                         const int32_t* block_tables,
                                         const int64_t* block_table_offsets,
                                         const float* q, int64_t total_tokens,
                                         const float* keys, const float* values, float* out);
pb_status pb_single_token_attention(const pb_attn_shape* shape, int32_t n_spans,
                                    const int64_t* query_start, const int64_t* query_len,
                                    const int64_t* context_len, const int64_t* causal_offset,
                                    const int32_t* block_tables,
                                    const int64_t* block_table_offsets, const float* q,
                                    int64_t total_tokens, const float* keys,
                                    const float* values, float* out);

/* ===================================================================== KV pages
 * A page is page_bytes contiguous bytes (chunk_size * n_kv_head * head_size elements) at
 * pool + slot * page_bytes: PagedKvStore::key_row addressing (src/attention.cpp:60-71).
 * Slot lists are DEVICE int32 arrays.  The reference moves no bytes; these
 * are the copies its bookkeeping implies (PagedKvCache::apply_evictions / restore,
 * src/paged_kv_cache.cpp:129-197). */

/* staging[i] = pool[slots[i]] for i < n, for n_layers layers: the pool of layer l starts at
 * pool + l * layer_stride; staging is [i][l] (page_bytes each) when layer_major == 0 and
 * [l][i] when layer_major == 1. */
pb_status pb_kv_gather_pages(const void* pool, int64_t layer_stride, int32_t n_layers,
                             int64_t page_bytes, const int32_t* d_slots, int64_t n,
                             void* staging, int32_t layer_major, void* stream);
/* pool[slots[i]] = staging[i] (inverse of gather, same layouts). */
pb_status pb_kv_scatter_pages(const void* staging, int64_t layer_stride, int32_t n_layers,
                              int64_t page_bytes, const int32_t* d_slots, int64_t n,
                              void* pool, int32_t layer_major, void* stream);
/* Paged K/V append (the write loop of qkv_project, src/attention.cpp:315-327): row i
 * (n_kv_head*head_size elements of `dtype`) goes to slot block_table[(start_pos+i)/chunk],
 * row (start_pos+i)%chunk, for i < n_rows, one span per entry of the CSR arrays.
 * k_rows/v_rows are [sum rows][n_kv*hs]; span s covers rows row_start[s]..+n_rows[s].
 * Out-of-range positions/slots are rejected on the host from the HOST copies of the
 * arrays (h_*) before the launch; d_* are the device copies the kernel reads. */
pb_status pb_kv_append(const pb_attn_shape* shape, int32_t n_spans, const int64_t* h_row_start,
                       const int64_t* h_n_rows, const int64_t* h_start_pos,
                       const int32_t* h_block_tables, const int64_t* h_bt_offsets,
                       const int64_t* d_row_start, const int64_t* d_n_rows,
                       const int64_t* d_start_pos, const int32_t* d_block_tables,
                       const int64_t* d_bt_offsets, const void* k_rows, const void* v_rows,
                       void* k_pages, void* v_pages, void* stream);

/* Deterministic synthetic fill: dst[i] = dtype(float(2*u01(draw first_draw+i) - 1)) where
 * draw j is the j-th (0-based) output of SplitMix64{seed} (src/workload.cpp:30-40).
 * Counter-based, so a GPU fill equals the sequential CPU stream bit for bit. */
pb_status pb_fill_splitmix_unit(void* dst, int32_t dtype, int64_t n, uint64_t seed,
                                uint64_t first_draw, void* stream);

/* ===================================================================== model byte arithmetic
 * kvsim::ModelConfig (include/kvsim/model_config.hpp; src/model_config.cpp:13-68).
 * chunk_bytes is per worker: kv_token_bytes * chunk_size / n_partitions (:36-40), i.e. the
 * bytes one rank's pools / host tier hold for one chunk under pb_shard_shape; a tier built
 * with page_bytes = chunk_size * (n_kv_head / n_partitions) * head_size * bytes_per_scalar has
 * pb_tier_chunk_bytes == pb_model_chunk_bytes. */
typedef struct pb_model_config {
    int32_t n_layer, hidden, n_head, n_kv_head, head_size, bytes_per_scalar, n_partitions;
} pb_model_config;
pb_status pb_model_validate(const pb_model_config* model);                  /* validate, :13-27 */
pb_status pb_model_kv_token_bytes(const pb_model_config* model, uint64_t* out); /* :29-34 */
pb_status pb_model_chunk_bytes(const pb_model_config* model, int32_t chunk_size, uint64_t* out); /* :36-40 */
pb_status pb_model_preset(const char* name, pb_model_config* out);          /* preset, :48-68 */

/* ===================================================================== multi-GPU shard
 * KV-head sharding: rank r of `world` owns kv heads
 * [r*n_kv/world, (r+1)*n_kv/world) and the query heads that read them, a contiguous block
 * (head h reads kv head h / group, src/attention.cpp:91).  Spans, block tables and slots are
 * identical on every rank; each rank builds its plan from the shard shape and runs it on its
 * own device (one host thread or process per GPU; every pb_* call works on the CUDA device
 * current on the calling thread, and a plan / tier belongs to the device current when it was
 * uploaded / created).  Requires n_kv_head % world == 0 (src/model_config.cpp:25-26). */
pb_status pb_shard_shape(const pb_attn_shape* full, int32_t rank, int32_t world, pb_attn_shape* out,
                         int32_t* first_head, int32_t* first_kv_head);

/* ===================================================================== CPU-tier swap engine
 * Pinned host tier [host_slot][layer][K|V][page] (one chunk = chunk_bytes contiguous,
 * src/model_config.cpp:36-40) and the ordered, layer-pipelined copies the reference only
 * models as a timeline (src/swap_engine.cpp:21-53):
 *   1. swap-out GATHER of device pages on compute_stream first (device slots vacated by
 *      swap-out may be refilled in the same step, src/paged_kv_cache.cpp:28-37);
 *   2. swap-in per layer on copy_stream: batched H2D into staging, scatter kernel into the
 *      pools, event per layer (pb_swap_wait_layer = "attention of layer l may start",
 *      PAPER.md:617-619);
 *   3. swap-out D2H after this step's swap-ins (schedule_swap_out_start, :50-53), on the
 *      tier's own stream so the next step's swap-ins and attention do not queue behind it.
 *      Host-slot hazards across steps are ordered by events: a swap-in waits for the newest
 *      D2H still in flight that writes the host slot it reads (any earlier step, not only
 *      the previous one), and a D2H waits for the previous step's swap-ins.  pb_swap_sync
 *      waits for everything, D2H included.
 * Within one step the moves follow the scheduler's order: every eviction precedes every
 * restore.  So
 *   * a chunk swapped out and restored in the same step (out dst == in src, same chunk id)
 *     is restored device-to-device from the swap-out staging, and its D2H is skipped (the
 *     host copy is dead: restore frees the host slot);
 *   * an out-move whose host slot a LATER out-move of the same step also writes is dead (its
 *     chunk was dropped from the host in between) and is skipped, so no two copies of one
 *     batch write the same host slot;
 *   * an out-move writing a host slot a restore of a DIFFERENT chunk reads (restore freed
 *     it) is a write-after-read: that D2H waits for the step's swap-ins.
 * A chunk restored and then evicted again in one step is not representable; callers net it
 * out (pb_sched never produces it).
 * Pools: k_pool / v_pool hold n_layer pools at layer_stride bytes apart, pages of
 * page_bytes.  Moves come from pb_cache_apply_evictions (device src -> host dst) and
 * pb_cache_restore (host src -> device dst). */
/* ---------------------------------------------------------------- pipeline event log
 * Device-timestamped events (%globaltimer ns) of the swap / attention pipeline, kinds in the
 * order of kvsim::EventKind (include/kvsim/event_log.hpp:14).  pb_evlog_mark enqueues a
 * stamp on a stream (it records when that stream reached the point); a tier with a log
 * attached stamps SWAP_IN_LAYER after each layer's pages landed and SWAP_OUT after the D2H.
 * pb_evlog_audit restates LayerDependencyAuditor (src/event_log.cpp:90-118). */
typedef enum pb_event_kind {
    PB_EV_SWAP_IN_LAYER = 0,
    PB_EV_SWAP_OUT = 1,
    PB_EV_ATTN_START = 2,
    PB_EV_STEP_END = 3
} pb_event_kind;
typedef struct pb_event_record {
    int64_t t_ns;
    int32_t kind;
    int32_t layer;
    int64_t req;
} pb_event_record;
typedef struct pb_event_log pb_event_log;
pb_status pb_evlog_create(int64_t capacity, pb_event_log** out);
void pb_evlog_destroy(pb_event_log* log);
pb_status pb_evlog_mark(pb_event_log* log, int32_t kind, int32_t layer, int64_t req, void* stream);
pb_status pb_evlog_read(pb_event_log* log, pb_event_record* out, int64_t cap, int64_t* n);
pb_status pb_evlog_reset(pb_event_log* log);
pb_status pb_evlog_audit(const pb_event_record* events, int64_t n, uint64_t* violations,
                         uint64_t* steps);
/* Per-step form: readiness of a layer = latest SWAP_IN_LAYER of that layer anywhere in the
 * step (events between STEP_ENDs), so an attention stamped before its swap-in is flagged. */
pb_status pb_evlog_audit_steps(const pb_event_record* events, int64_t n, uint64_t* violations,
                               uint64_t* steps);

typedef struct pb_kv_tier pb_kv_tier;
typedef struct pb_slot_move pb_slot_move; /* defined with the bookkeeping API below */
pb_status pb_tier_create(int32_t n_layer, int32_t host_slots, int64_t page_bytes,
                         int32_t max_chunks_per_step, pb_kv_tier** out);
void pb_tier_destroy(pb_kv_tier* tier);
void* pb_tier_host_base(pb_kv_tier* tier);
int64_t pb_tier_chunk_bytes(const pb_kv_tier* tier);
pb_status pb_swap_step(pb_kv_tier* tier, void* k_pool, void* v_pool, int64_t layer_stride,
                       const pb_slot_move* out_moves, int64_t n_out, const pb_slot_move* in_moves,
                       int64_t n_in, void* compute_stream, void* copy_stream);
pb_status pb_swap_wait_layer(pb_kv_tier* tier, int32_t layer, void* compute_stream);
/* Transfer policy (explicit, per tier; the defaults are the measured best on B200 and no
 * environment variable changes them):
 *   swap_in: PB_SWAP_IN_STAGED (default: batched H2D pieces into device staging + a scatter
 *            kernel) or PB_SWAP_IN_ZERO_COPY (one kernel per layer reading the mapped pinned
 *            tier);
 *   d2h:     PB_D2H_AFTER_SWAP_IN (default: own stream, after this step's swap-ins),
 *            PB_D2H_CONCURRENT (own stream, concurrent with the swap-ins unless a host slot
 *            hazard orders it) or PB_D2H_ON_COPY_STREAM (queued behind the swap-ins on
 *            copy_stream, the reference's literal order);
 *   layers_per_piece: layers per swap-in H2D piece, 1..n_layer (default 8; 0 keeps it). */
#define PB_SWAP_IN_STAGED 0
#define PB_SWAP_IN_ZERO_COPY 1
#define PB_D2H_ON_COPY_STREAM 0
#define PB_D2H_CONCURRENT 1
#define PB_D2H_AFTER_SWAP_IN 2
pb_status pb_tier_set_policy(pb_kv_tier* tier, int32_t swap_in, int32_t d2h, int32_t layers_per_piece);
pb_status pb_swap_sync(pb_kv_tier* tier);
/* Attach (or detach with NULL) an event log to the tier's transfers. */
pb_status pb_tier_set_event_log(pb_kv_tier* tier, pb_event_log* log);

/* ===================================================================== KV page bookkeeping
 * Two-tier slot allocator + per-conversation chunk index with the exact slot semantics of
 * kvsim::PagedKvCache (include/kvsim/paged_kv_cache.hpp:52-153, src/paged_kv_cache.cpp):
 * lowest slot ids first, device slots vacated by swap-out reused LIFO before free ones,
 * fill-partial-first appends, validate-before-mutate.  Block tables and slot lists are
 * bit-identical to the reference.  In addition every tier move reports its
 * (chunk, source slot, destination slot) triple, which the copy engine needs and the
 * reference discards.  Host-only; single writer. */
typedef struct pb_kv_cache pb_kv_cache;

typedef struct pb_slot_move {
    int64_t chunk;
    int32_t src_slot; /* slot in the tier the chunk left (-1: rematerialised from nothing) */
    int32_t dst_slot; /* slot in the tier it entered (-1: dropped) */
} pb_slot_move;

typedef struct pb_chunk_record { /* ChunkRecord, include/kvsim/chunk.hpp:23-33 */
    int64_t chunk_id, conv_id, start_offset, n_tokens;
    int32_t location; /* 0 device, 1 host, 2 dropped (ChunkLocationKind) */
    int32_t slot;
    double last_active;
} pb_chunk_record;

typedef struct pb_layout_segment { /* LayoutSegment, paged_kv_cache.hpp:20-27 */
    int32_t kind;     /* 0 resident (device), 1 swap-in (host), 2 recompute (dropped) */
    int32_t n_chunks;
    int64_t token_begin, token_end;
    int64_t first_chunk;
} pb_layout_segment;

/* PagedKvCache(chunk_size, device_slots, host_slots)        paged_kv_cache.cpp:12-26 */
pb_status pb_cache_create(int32_t chunk_size, int32_t device_slots, int32_t host_slots,
                          pb_kv_cache** out);
void pb_cache_destroy(pb_kv_cache* cache);
/* allocate(conv, n_tokens, now) -> created chunk ids         paged_kv_cache.cpp:53-96 */
pb_status pb_cache_allocate(pb_kv_cache* cache, int64_t conv, int64_t n_tokens, double now,
                            int64_t* created, int64_t cap, int64_t* n_created);
/* apply_evictions(victims, Host|Dropped); moves[i] for ids[i]  paged_kv_cache.cpp:129-172 */
pb_status pb_cache_apply_evictions(pb_kv_cache* cache, const int64_t* ids, int64_t n,
                                   int32_t to_host, pb_slot_move* moves);
/* restore(chunks): host slot -> device slot                   paged_kv_cache.cpp:174-197 */
pb_status pb_cache_restore(pb_kv_cache* cache, const int64_t* ids, int64_t n, pb_slot_move* moves);
/* rematerialize(chunks): dropped -> device slot               paged_kv_cache.cpp:199-220 */
pb_status pb_cache_rematerialize(pb_kv_cache* cache, const int64_t* ids, int64_t n,
                                 pb_slot_move* moves);
/* release_conversation(conv)                                  paged_kv_cache.cpp:224-246 */
pb_status pb_cache_release_conversation(pb_kv_cache* cache, int64_t conv);
/* touch / retain_on_finish(conv, now)                         paged_kv_cache.cpp:222-254 */
pb_status pb_cache_touch(pb_kv_cache* cache, int64_t conv, double now);
/* block_table(conv, context_tokens)                           paged_kv_cache.cpp:284-304 */
pb_status pb_cache_block_table(const pb_kv_cache* cache, int64_t conv, int64_t context_tokens,
                               int32_t* out, int64_t cap, int64_t* n);
/* layout(conv)                                                paged_kv_cache.cpp:98-127 */
pb_status pb_cache_layout(const pb_kv_cache* cache, int64_t conv, pb_layout_segment* segs,
                          int64_t cap, int64_t* n, int64_t* total_tokens);
/* conversation_chunks(conv) with their records                paged_kv_cache.hpp:104 */
pb_status pb_cache_conversation_chunks(const pb_kv_cache* cache, int64_t conv,
                                       pb_chunk_record* out, int64_t cap, int64_t* n);
/* chunk(id)                                                   paged_kv_cache.hpp:103 */
pb_status pb_cache_chunk(const pb_kv_cache* cache, int64_t id, pb_chunk_record* out);
/* collect_chunks(kind, exclude) in (conv, offset) order       paged_kv_cache.cpp:270-282 */
pb_status pb_cache_collect_chunks(const pb_kv_cache* cache, int32_t location,
                                  const int64_t* exclude_convs, int64_t n_exclude, int64_t* ids,
                                  int64_t cap, int64_t* n);
/* counts[8]: device capacity, free, reclaimable, allocated; host capacity, free, allocated;
 * chunk size */
void pb_cache_counts(const pb_kv_cache* cache, int64_t* counts8);
int32_t pb_cache_has_conversation(const pb_kv_cache* cache, int64_t conv);
int64_t pb_cache_total_tokens(const pb_kv_cache* cache, int64_t conv);
/* append_chunks_needed(conv, add)                             paged_kv_cache.cpp:306-312 */
int32_t pb_cache_append_chunks_needed(const pb_kv_cache* cache, int64_t conv, int64_t add);
/* verify(): PB_ERR_ERROR on any invariant violation           paged_kv_cache.cpp:341-396 */
pb_status pb_cache_verify(const pb_kv_cache* cache);
/* dump() text; returns its length, writes at most cap-1 chars  paged_kv_cache.cpp:314-339 */
int64_t pb_cache_dump(const pb_kv_cache* cache, char* buf, int64_t cap);

/* ===================================================================== step planner
 * The reference Scheduler (include/kvsim/scheduler.hpp:88-179, src/scheduler.cpp) over a
 * pb_kv_cache: FCFS admission with reserve, prefix-drop span construction
 * (plan_request :162-230), rematerialize -> restore -> allocate (commit_admission
 * :232-258), eviction with host-overflow drops (:71-160), suspension (:292-350) and batch
 * assembly (build_batch :352-420).  Spans and block tables are bit-identical to the
 * reference; every plan also carries the slot moves for pb_swap_step. */
typedef struct pb_scheduler pb_scheduler;
typedef struct pb_sched_params { /* SchedulerParams, scheduler.hpp:75-82 */
    int32_t split_mode; /* 0 unified (prefill + decode in one plan), 1 split */
    int32_t policy;     /* 0 pensieve retention value, 1 LRU */
    int32_t stateful;   /* retain KV across turns */
    int64_t token_budget;
    double swap_threshold;
    double reserve_fraction;
} pb_sched_params;
void pb_sched_default_params(pb_sched_params* params);
/* cost profile: anchors (context_len, seconds per 32-token chunk), cost_model.hpp:170-177 */
pb_status pb_sched_create(pb_kv_cache* cache, const int64_t* anchor_len, const double* anchor_sec,
                          int32_t n_anchors, double c_other, double per_token_other,
                          const pb_sched_params* params, pb_scheduler** out);
/* synthetic_profile(k_attn, ...), cost_model.cpp:77-85 */
pb_status pb_sched_create_synthetic(pb_kv_cache* cache, double k_attn, double c_other,
                                    double per_token_other, const pb_sched_params* params,
                                    pb_scheduler** out);
void pb_sched_destroy(pb_scheduler* sched);
pb_status pb_sched_enqueue(pb_scheduler* sched, int64_t req_id, int64_t conv_id, int32_t turn,
                           double arrival, int64_t prompt, int64_t output);
pb_status pb_sched_append_history(pb_scheduler* sched, int64_t conv, int64_t tokens);
/* begin_step -> maybe_swap_out -> admit -> ensure_generation_capacity -> build_batch */
pb_status pb_sched_step(pb_scheduler* sched, double now, int32_t* n_plans);
/* info[8]: n_spans, total tokens, block-table entries, swap_in, swap_out, recompute tokens,
 * in_moves, out_moves */
pb_status pb_sched_plan_info(const pb_scheduler* sched, int32_t plan, int64_t* info8);
pb_status pb_sched_plan_spans(const pb_scheduler* sched, int32_t plan, int64_t* req_id,
                              int64_t* query_start, int64_t* query_len, int64_t* context_len,
                              int64_t* causal_offset, int32_t* block_tables, int64_t* bt_offsets);
pb_status pb_sched_plan_moves(const pb_scheduler* sched, int32_t plan, pb_slot_move* in_moves,
                              pb_slot_move* out_moves);
/* complete_plan(plan, end_time)                                 scheduler.cpp:433-457 */
pb_status pb_sched_complete(pb_scheduler* sched, int32_t plan, double end_time, int64_t* finished,
                            int64_t cap, int64_t* n_finished);
/* plan_request without mutation; info[9] = input, recompute, pending, n_rematerialize,
 * n_swap_in, append_slots, device_hit, host_hit, n_spans; spans as (q_len, ctx, offset) */
pb_status pb_sched_plan_request(const pb_scheduler* sched, int64_t req_id, int64_t conv_id,
                                int64_t prompt, int64_t output, int64_t generated,
                                int32_t suspended, int64_t* info9, int64_t* span3, int64_t cap);
int64_t pb_sched_queue_size(const pb_scheduler* sched);
int64_t pb_sched_running_size(const pb_scheduler* sched);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* PENSIEVE_B200_H */
