// KV page movement kernels (HBM-bound integer/byte work):
//   * page gather / scatter between the paged pools and contiguous staging buffers — the
//     device half of CPU-tier swap-out / swap-in (PagedKvCache::apply_evictions / restore,
//     /root/reference/proj/src/paged_kv_cache.cpp:129-197; the reference itself moves no
//     bytes);
//   * paged K/V append — the row-write loop of qkv_project (src/attention.cpp:315-327);
//   * the counter-based SplitMix64 fill used to build bit-reproducible synthetic inputs
//     (src/workload.cpp:30-40);
//   * the optional device restatement of attention's NumericError checks.
//
// Copies move 16-byte vectors, one page per CTA-iteration, grid-stride over
// (layer, page) pairs with the grid sized to a multiple of the SM count.
#include "attn_internal.hpp"
#include "pb_common.hpp"

#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

namespace pb {

namespace {

int num_sms() { return device_sms(); }

// dst/src page index for item j = (layer l, page i)
template <bool kGather>
__global__ void __launch_bounds__(256) page_copy_kernel(const uint8_t* __restrict__ src,
                                                       uint8_t* __restrict__ dst,
                                                       const int32_t* __restrict__ slots,
                                                       int64_t n, int32_t n_layers,
                                                       int64_t layer_stride, int64_t page_bytes,
                                                       int32_t layer_major) {
    const int64_t vec_per_page = page_bytes / 16;
    const int64_t total = n * n_layers;
    for (int64_t job = blockIdx.x; job < total; job += gridDim.x) {
        const int64_t l = job / n;
        const int64_t i = job % n;
        const int64_t pool_off = l * layer_stride + static_cast<int64_t>(slots[i]) * page_bytes;
        const int64_t stage_off = (layer_major ? (l * n + i) : (i * n_layers + l)) * page_bytes;
        const int4* s = reinterpret_cast<const int4*>(src + (kGather ? pool_off : stage_off));
        int4* d = reinterpret_cast<int4*>(dst + (kGather ? stage_off : pool_off));
        // 4 independent 16 B loads in flight per thread before the stores
        int64_t v = threadIdx.x;
        for (; v + 3 * 256 < vec_per_page; v += 4 * 256) {
            int4 a = __ldcs(s + v), b = __ldcs(s + v + 256), c = __ldcs(s + v + 512), e = __ldcs(s + v + 768);
            __stcs(d + v, a);
            __stcs(d + v + 256, b);
            __stcs(d + v + 512, c);
            __stcs(d + v + 768, e);
        }
        for (; v < vec_per_page; v += 256) __stcs(d + v, __ldcs(s + v));
    }
}

template <typename T>
__global__ void __launch_bounds__(128) append_kernel(const T* __restrict__ k_rows,
                                                     const T* __restrict__ v_rows,
                                                     T* __restrict__ k_pages, T* __restrict__ v_pages,
                                                     const int64_t* __restrict__ row_start,
                                                     const int64_t* __restrict__ n_rows,
                                                     const int64_t* __restrict__ start_pos,
                                                     const int32_t* __restrict__ bt,
                                                     const int64_t* __restrict__ bt_off,
                                                     int32_t n_spans, int64_t total_rows,
                                                     int32_t chunk, int64_t row_elems) {
    for (int64_t r = blockIdx.x; r < total_rows; r += gridDim.x) {
        // span of row r: last span whose row_start <= r (row_start ascending)
        int lo = 0, hi = n_spans - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (row_start[mid] <= r) lo = mid; else hi = mid - 1;
        }
        const int64_t i = r - row_start[lo];
        if (i >= n_rows[lo]) continue;
        const int64_t pos = start_pos[lo] + i;
        const int32_t slot = bt[bt_off[lo] + pos / chunk];
        const int64_t dst = (static_cast<int64_t>(slot) * chunk + pos % chunk) * row_elems;
        const int64_t src = r * row_elems;
        for (int64_t e = threadIdx.x; e < row_elems; e += blockDim.x) {
            k_pages[dst + e] = k_rows[src + e];
            v_pages[dst + e] = v_rows[src + e];
        }
    }
}

__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t draw) {
    // draw-th output (0-based) of SplitMix64{seed}: state after draw+1 increments
    uint64_t z = seed + (draw + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

template <typename T>
__global__ void fill_kernel(T* dst, int64_t n, uint64_t seed, uint64_t first) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double u = static_cast<double>(splitmix_at(seed, first + i) >> 11) * (1.0 / 9007199254740992.0);
        const float f = static_cast<float>(2.0 * u - 1.0);
        if constexpr (sizeof(T) == 4) dst[i] = f;
        else dst[i] = __float2bfloat16_rn(f);
    }
}

__device__ __forceinline__ bool finite_elem(float x) { return isfinite(x); }
__device__ __forceinline__ bool finite_elem(__nv_bfloat16 x) { return isfinite(__bfloat162float(x)); }

// q fully finite (attention.cpp:30) and k_row[0] finite for every attended position of
// every kv head (attention.cpp:100-101).  One CTA per span plus a grid-stride q scan.
template <typename T>
__global__ void check_numerics_kernel(AttnParams p, int64_t q_elems, int32_t* flag) {
    const T* q = static_cast<const T*>(p.q);
    const T* k = static_cast<const T*>(p.k_pages);
    bool bad = false;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < q_elems;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        bad |= !finite_elem(q[i]);
    if (blockIdx.x < p.n_items) {
        const SpanDev sp = p.spans[blockIdx.x];
        if (sp.query_len > 0) {
            const int64_t n = static_cast<int64_t>(sp.context_len) * p.n_kv_head;
            for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
                const int pos = static_cast<int>(j / p.n_kv_head);
                const int kvh = static_cast<int>(j % p.n_kv_head);
                const int32_t slot = p.block_tables[sp.bt_off + pos / p.chunk];
                const int64_t off = ((static_cast<int64_t>(slot) * p.chunk + pos % p.chunk) * p.n_kv_head + kvh) *
                                    static_cast<int64_t>(p.head_size);
                bad |= !finite_elem(k[off]);
            }
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, PB_ERR_NUMERIC);
}

__global__ void set_flag_kernel(int32_t* flag, int32_t v) { *flag = v; }

} // namespace

void launch_check_numerics(const AttnParams& p, int dtype, int64_t q_elems, int32_t* d_flag,
                           cudaStream_t st) {
    set_flag_kernel<<<1, 1, 0, st>>>(d_flag, 0);
    const int grid = std::max(p.n_items, 1);
    if (dtype == PB_F32) check_numerics_kernel<float><<<grid, 256, 0, st>>>(p, q_elems, d_flag);
    else check_numerics_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(p, q_elems, d_flag);
    cuda_check(cudaGetLastError(), "check_numerics launch");
    count_launch(2);
}

} // namespace pb

using namespace pb;

namespace {

pb_status page_copy(bool gather, const void* src, int64_t layer_stride, int32_t n_layers,
                    int64_t page_bytes, const int32_t* d_slots, int64_t n, void* dst,
                    int32_t layer_major, void* stream) {
    return guarded([&] {
        if (n < 0 || n_layers < 0 || page_bytes < 0) fail(PB_ERR_DIMENSION_MISMATCH, "negative size");
        if (n == 0 || n_layers == 0 || page_bytes == 0) return;
        if (!src || !dst || !d_slots) fail(PB_ERR_ERROR, "null pointer");
        if (page_bytes % 16 != 0 || (reinterpret_cast<uintptr_t>(src) % 16) ||
            (reinterpret_cast<uintptr_t>(dst) % 16) || layer_stride % 16)
            fail(PB_ERR_UNSUPPORTED, "page copies need 16-byte aligned pages and buffers");
        const int64_t jobs = n * n_layers;
        const int grid = static_cast<int>(std::min<int64_t>(jobs, static_cast<int64_t>(num_sms()) * 8));
        auto* s = static_cast<const uint8_t*>(src);
        auto* d = static_cast<uint8_t*>(dst);
        if (gather)
            page_copy_kernel<true><<<grid, 256, 0, as_stream(stream)>>>(s, d, d_slots, n, n_layers,
                                                                       layer_stride, page_bytes, layer_major);
        else
            page_copy_kernel<false><<<grid, 256, 0, as_stream(stream)>>>(s, d, d_slots, n, n_layers,
                                                                        layer_stride, page_bytes, layer_major);
        cuda_check(cudaGetLastError(), "page copy launch");
        count_launch();
    });
}

} // namespace

extern "C" {

pb_status pb_kv_gather_pages(const void* pool, int64_t layer_stride, int32_t n_layers,
                             int64_t page_bytes, const int32_t* d_slots, int64_t n,
                             void* staging, int32_t layer_major, void* stream) {
    return page_copy(true, pool, layer_stride, n_layers, page_bytes, d_slots, n, staging,
                     layer_major, stream);
}

pb_status pb_kv_scatter_pages(const void* staging, int64_t layer_stride, int32_t n_layers,
                              int64_t page_bytes, const int32_t* d_slots, int64_t n,
                              void* pool, int32_t layer_major, void* stream) {
    return page_copy(false, staging, layer_stride, n_layers, page_bytes, d_slots, n, pool,
                     layer_major, stream);
}

pb_status pb_kv_append(const pb_attn_shape* shape, int32_t n_spans, const int64_t* h_row_start,
                       const int64_t* h_n_rows, const int64_t* h_start_pos,
                       const int32_t* h_bt, const int64_t* h_bt_off, const int64_t* d_row_start,
                       const int64_t* d_n_rows, const int64_t* d_start_pos, const int32_t* d_bt,
                       const int64_t* d_bt_off, const void* k_rows, const void* v_rows,
                       void* k_pages, void* v_pages, void* stream) {
    return guarded([&] {
        if (!shape) fail(PB_ERR_ERROR, "null shape");
        require(shape->n_kv_head > 0 && shape->head_size > 0 && shape->chunk_size > 0,
                "bad kv shape");
        // qkv_project's addressing checks (attention.cpp:315-322), before any write
        int64_t total = 0;
        for (int32_t s = 0; s < n_spans; ++s) {
            require(h_row_start[s] == total, "append rows must tile the row buffer");
            require(h_n_rows[s] >= 0 && h_start_pos[s] >= 0, "negative append span");
            const int64_t bt_len = h_bt_off[s + 1] - h_bt_off[s];
            if (h_n_rows[s] > 0) {
                const int64_t last = (h_start_pos[s] + h_n_rows[s] - 1) / shape->chunk_size;
                require(last < bt_len, "block table too short for written positions");
                for (int64_t j = h_start_pos[s] / shape->chunk_size; j <= last; ++j) {
                    const int32_t slot = h_bt[h_bt_off[s] + j];
                    if (slot < 0 || slot >= shape->n_slots)
                        fail(PB_ERR_ERROR, "block table references out-of-range slot " + std::to_string(slot));
                }
            }
            total += h_n_rows[s];
        }
        if (total == 0) return;
        const int64_t row_elems = static_cast<int64_t>(shape->n_kv_head) * shape->head_size;
        const int grid = static_cast<int>(std::min<int64_t>(total, static_cast<int64_t>(num_sms()) * 16));
        auto st = as_stream(stream);
        if (shape->dtype == PB_F32)
            append_kernel<float><<<grid, 128, 0, st>>>(
                static_cast<const float*>(k_rows), static_cast<const float*>(v_rows),
                static_cast<float*>(k_pages), static_cast<float*>(v_pages), d_row_start, d_n_rows,
                d_start_pos, d_bt, d_bt_off, n_spans, total, shape->chunk_size, row_elems);
        else
            append_kernel<__nv_bfloat16><<<grid, 128, 0, st>>>(
                static_cast<const __nv_bfloat16*>(k_rows), static_cast<const __nv_bfloat16*>(v_rows),
                static_cast<__nv_bfloat16*>(k_pages), static_cast<__nv_bfloat16*>(v_pages), d_row_start,
                d_n_rows, d_start_pos, d_bt, d_bt_off, n_spans, total, shape->chunk_size, row_elems);
        cuda_check(cudaGetLastError(), "append launch");
        count_launch();
    });
}

pb_status pb_fill_splitmix_unit(void* dst, int32_t dtype, int64_t n, uint64_t seed,
                                uint64_t first_draw, void* stream) {
    return guarded([&] {
        if (n <= 0) return;
        const int grid = num_sms() * 8;
        if (dtype == PB_F32)
            fill_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(static_cast<float*>(dst), n, seed, first_draw);
        else if (dtype == PB_BF16)
            fill_kernel<__nv_bfloat16><<<grid, 256, 0, as_stream(stream)>>>(static_cast<__nv_bfloat16*>(dst), n,
                                                                          seed, first_draw);
        else
            fail(PB_ERR_UNSUPPORTED, "dtype");
        cuda_check(cudaGetLastError(), "fill launch");
        count_launch();
    });
}

} // extern "C"
