/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the ragged paged attention hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this
 * library, and only as the checker.  The product (paper_2312_05516_b200) never links
 * or calls it.
 *
 * Plain-C99 restatement of the reference kvsim attention module
 * (/root/reference/proj/src/attention.cpp).  Every function keeps the reference's loop
 * order and its fp32-in / double-accumulate arithmetic so that, on the same inputs,
 * results are bit-identical to the reference (checked by tests/test_oracle.py against
 * the reference compiled into oracle/_ref by oracle/Makefile, and against the golden
 * vectors in tests/golden/).
 *
 * Status codes are the ones declared in include/pensieve_b200.h (PB_*); they are
 * repeated here so the oracle has no dependency on the product.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_DIMENSION_MISMATCH 1 /* kvsim::DimensionMismatch */
#define OR_NUMERIC 2            /* kvsim::NumericError */
#define OR_ERROR 3              /* kvsim::Error (e.g. out-of-range slot) */

/* ------------------------------------------------------------------ SplitMix64
 * Follows /root/reference/proj/src/workload.cpp:30-40 (SplitMix64::next / u01). */
uint64_t oracle_splitmix_next(uint64_t *state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

double oracle_splitmix_u01(uint64_t *state) {
    return (double)(oracle_splitmix_next(state) >> 11) * (1.0 / 9007199254740992.0);
}

/* float(2*u01 - 1): the fixture draw of proj/tests/test_attention.cpp:19 and
 * proj/tests/acceptance.cpp:98 (both evaluate 2*u-1 in double, then round). */
void oracle_fill_unit(uint64_t *state, float *dst, int64_t n) {
    for (int64_t i = 0; i < n; ++i) dst[i] = (float)(2.0 * oracle_splitmix_u01(state) - 1.0);
}

/* ------------------------------------------------------------------ validation
 * Follows check_batch, proj/src/attention.cpp:23-48 (same check order, so the same
 * error class wins when several are violated). */
static int check_batch(int n_head, int head_size, double scale, int store_n_kv_head,
                       int store_head_size, int chunk, int n_slots, const float *q,
                       int64_t q_elems, int n_spans, const int64_t *query_start,
                       const int64_t *query_len, const int64_t *context_len,
                       const int64_t *causal_offset, const int32_t *bt,
                       const int64_t *bt_off) {
    if (!(n_head > 0 && head_size > 0)) return OR_DIMENSION_MISMATCH;
    if (!(store_n_kv_head > 0 && store_head_size == head_size)) return OR_DIMENSION_MISMATCH;
    if (n_head % store_n_kv_head != 0) return OR_DIMENSION_MISMATCH;
    if (!(scale > 0)) return OR_DIMENSION_MISMATCH;
    for (int64_t i = 0; i < q_elems; ++i)
        if (!isfinite(q[i])) return OR_NUMERIC;
    int64_t expect = 0;
    for (int s = 0; s < n_spans; ++s) {
        if (!(query_len[s] >= 0)) return OR_DIMENSION_MISMATCH;
        if (query_start[s] != expect) return OR_DIMENSION_MISMATCH;
        if (context_len[s] != causal_offset[s] + query_len[s]) return OR_DIMENSION_MISMATCH;
        if (!(causal_offset[s] >= 0)) return OR_DIMENSION_MISMATCH;
        int64_t need = (context_len[s] + chunk - 1) / chunk;
        if (bt_off[s + 1] - bt_off[s] != need) return OR_DIMENSION_MISMATCH;
        for (int64_t j = bt_off[s]; j < bt_off[s + 1]; ++j)
            if (bt[j] < 0 || bt[j] >= n_slots) return OR_ERROR;
        expect += query_len[s];
    }
    int64_t total = (int64_t)n_head * head_size > 0 ? q_elems / ((int64_t)n_head * head_size) : 0;
    if (expect != total) return OR_DIMENSION_MISMATCH;
    return OR_OK;
}

/* Row address in the paged store: (slot*chunk + row) * n_kv*hs, as
 * PagedKvStore::key_row, proj/src/attention.cpp:60-71. */
static inline const float *store_row(const float *pool, int32_t slot, int64_t row, int chunk,
                                     int row_elems) {
    return pool + ((size_t)slot * chunk + (size_t)row) * (size_t)row_elems;
}

/* Follows paged_multi_token_attention, proj/src/attention.cpp:73-132.
 * single_token != 0 restates single_token_attention (:134-188): same checks plus
 * query_len == 1 on every span; identical arithmetic (it is mathematically the same
 * loop with allowed == context_len). */
int oracle_paged_attention(int single_token, int n_head, int n_kv_head, int head_size,
                           int chunk, int n_slots, double scale, const float *q,
                           int64_t q_elems, int n_spans, const int64_t *query_start,
                           const int64_t *query_len, const int64_t *context_len,
                           const int64_t *causal_offset, const int32_t *bt,
                           const int64_t *bt_off, const float *keys, const float *values,
                           float *out) {
    int st = check_batch(n_head, head_size, scale, n_kv_head, head_size, chunk, n_slots, q,
                         q_elems, n_spans, query_start, query_len, context_len, causal_offset,
                         bt, bt_off);
    if (st != OR_OK) return st;
    if (single_token)
        for (int s = 0; s < n_spans; ++s)
            if (query_len[s] != 1) return OR_DIMENSION_MISMATCH;
    const int hs = head_size;
    const int group = n_head / n_kv_head;
    const int row_elems = n_kv_head * hs;
    memset(out, 0, sizeof(float) * (size_t)q_elems);
    int64_t max_ctx = 1;
    for (int s = 0; s < n_spans; ++s)
        if (context_len[s] > max_ctx) max_ctx = context_len[s];
    double *scores = (double *)malloc(sizeof(double) * (size_t)max_ctx);
    if (!scores) return OR_ERROR;

    for (int s = 0; s < n_spans; ++s) {
        const int32_t *table = bt + bt_off[s];
        for (int64_t i = 0; i < query_len[s]; ++i) {
            const int64_t allowed = causal_offset[s] + i + 1; /* causal prefix */
            const float *q_tok = q + (size_t)(query_start[s] + i) * n_head * hs;
            float *o_tok = out + (size_t)(query_start[s] + i) * n_head * hs;
            for (int h = 0; h < n_head; ++h) {
                const int kvh = h / group;
                const float *q_head = q_tok + (size_t)h * hs;
                double max_score = -HUGE_VAL;
                for (int64_t p = 0; p < allowed; ++p) {
                    const float *k_row =
                        store_row(keys, table[p / chunk], p % chunk, chunk, row_elems) +
                        (size_t)kvh * hs;
                    if (!isfinite(k_row[0])) {
                        free(scores);
                        return OR_NUMERIC;
                    }
                    double dot = 0.0;
                    for (int d = 0; d < hs; ++d) dot += (double)q_head[d] * (double)k_row[d];
                    double sc = dot / scale;
                    scores[p] = sc;
                    if (sc > max_score) max_score = sc;
                }
                double denom = 0.0;
                for (int64_t p = 0; p < allowed; ++p) {
                    double w = exp(scores[p] - max_score);
                    scores[p] = w;
                    denom += w;
                }
                float *o_head = o_tok + (size_t)h * hs;
                for (int d = 0; d < hs; ++d) {
                    double acc = 0.0;
                    for (int64_t p = 0; p < allowed; ++p) {
                        const float *v_row =
                            store_row(values, table[p / chunk], p % chunk, chunk, row_elems) +
                            (size_t)kvh * hs;
                        acc += scores[p] * (double)v_row[d];
                    }
                    o_head[d] = (float)(acc / denom);
                }
            }
        }
    }
    free(scores);
    return OR_OK;
}

/* Follows dense_attention, proj/src/attention.cpp:190-245 (contiguous k/v rows of
 * n_kv*hs floats). */
int oracle_dense_attention(const float *q, const float *k, const float *v, int64_t q_len,
                           int64_t kv_len, int64_t causal_offset, int n_head, int n_kv_head,
                           int head_size, double scale, float *out) {
    if (!(n_head > 0 && n_kv_head > 0 && head_size > 0 && n_head % n_kv_head == 0))
        return OR_DIMENSION_MISMATCH;
    if (causal_offset + q_len > kv_len) return OR_DIMENSION_MISMATCH;
    const int64_t qn = q_len * n_head * head_size, kn = kv_len * n_kv_head * head_size;
    for (int64_t i = 0; i < qn; ++i)
        if (!isfinite(q[i])) return OR_NUMERIC;
    for (int64_t i = 0; i < kn; ++i)
        if (!isfinite(k[i]) || !isfinite(v[i])) return OR_NUMERIC;
    const int group = n_head / n_kv_head;
    double *row = (double *)malloc(sizeof(double) * (size_t)(kv_len > 0 ? kv_len : 1));
    if (!row) return OR_ERROR;
    for (int64_t i = 0; i < q_len; ++i) {
        int64_t allowed = causal_offset + i + 1;
        for (int h = 0; h < n_head; ++h) {
            const int kvh = h / group;
            const float *q_head = q + ((size_t)i * n_head + h) * head_size;
            double max_s = -HUGE_VAL;
            for (int64_t p = 0; p < allowed; ++p) {
                const float *k_row = k + ((size_t)p * n_kv_head + kvh) * head_size;
                double dot = 0.0;
                for (int d = 0; d < head_size; ++d) dot += (double)q_head[d] * (double)k_row[d];
                row[p] = dot / scale;
                if (row[p] > max_s) max_s = row[p];
            }
            double denom = 0.0;
            for (int64_t p = 0; p < allowed; ++p) {
                row[p] = exp(row[p] - max_s);
                denom += row[p];
            }
            float *o_head = out + ((size_t)i * n_head + h) * head_size;
            for (int d = 0; d < head_size; ++d) {
                double acc = 0.0;
                for (int64_t p = 0; p < allowed; ++p)
                    acc += row[p] * (double)v[((size_t)p * n_kv_head + kvh) * head_size + d];
                o_head[d] = (float)(acc / denom);
            }
        }
    }
    free(row);
    return OR_OK;
}

/* ------------------------------------------------------------------ page movement
 * CPU restatement of the page copies the swap path performs.  The reference moves no
 * bytes; its page addressing is PagedKvStore::key_row
 * (proj/src/attention.cpp:60-71), its gather loop copyout_then_dense (:259-269).
 * A page is chunk*row_bytes contiguous bytes at slot*page_bytes. */
void oracle_gather_pages(const uint8_t *pool, int64_t page_bytes, const int32_t *slots,
                         int64_t n, uint8_t *staging) {
    for (int64_t i = 0; i < n; ++i)
        memcpy(staging + (size_t)i * page_bytes, pool + (size_t)slots[i] * page_bytes,
               (size_t)page_bytes);
}

void oracle_scatter_pages(const uint8_t *staging, int64_t page_bytes, const int32_t *slots,
                          int64_t n, uint8_t *pool) {
    for (int64_t i = 0; i < n; ++i)
        memcpy(pool + (size_t)slots[i] * page_bytes, staging + (size_t)i * page_bytes,
               (size_t)page_bytes);
}

/* K/V row write addressing of qkv_project, proj/src/attention.cpp:315-327:
 * position pos -> slot block_table[pos/chunk], row pos%chunk.  rows: n x row_elems. */
int oracle_append_rows(float *pool, int chunk, int n_slots, int row_elems, const int32_t *bt,
                       int64_t bt_len, int64_t start_pos, const float *rows, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        int64_t pos = start_pos + i;
        int64_t idx = pos / chunk;
        if (idx >= bt_len) return OR_DIMENSION_MISMATCH;
        int32_t slot = bt[idx];
        if (slot < 0 || slot >= n_slots) return OR_ERROR;
        memcpy(pool + ((size_t)slot * chunk + (size_t)(pos % chunk)) * row_elems,
               rows + (size_t)i * row_elems, sizeof(float) * (size_t)row_elems);
    }
    return OR_OK;
}
