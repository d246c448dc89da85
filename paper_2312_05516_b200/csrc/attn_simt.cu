// Generic SIMT ragged paged attention: the fp32 validation mode (PB_F32, 1e-5 parity with
// the double-accumulating reference) and the fallback for shapes the sm_100a tile kernel
// is not built for (head_size outside {64, 128}, page sizes that do not tile 128 rows).
//
// Semantics follow paged_multi_token_attention, /root/reference/proj/src/attention.cpp:73-132:
// token i of a span sees context positions [0, causal_offset + i]; query head h reads kv
// head h / group; softmax subtracts the running max.  Accumulation is fp32 (the reference
// accumulates in double; the 1e-5 bound in tests/test_attention_gpu.py covers the gap).
//
// One CTA (4 warps) per work item = (span, kv head, block of query tokens).  A warp owns
// one query row (token x head) at a time and walks the allowed context 32 positions per
// step: lane j scores position base+j (no reduction needed for the dot product), the
// warp agrees on the running max, and the PV update broadcasts each weight with one
// shuffle while lanes own output dimensions (coalesced V reads).
#include "attn_internal.hpp"
#include "pb_common.hpp"

#include <cuda_bf16.h>
#include <math_constants.h>

namespace pb {

namespace {

__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ void store_elem(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_elem(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr int kSimtWarps = 4;
constexpr int kMaxDimPerLane = 8; // head_size <= 256

template <typename T>
__global__ void __launch_bounds__(kSimtWarps * 32) attn_simt_kernel(AttnParams p) {
    extern __shared__ float q_smem[]; // [kSimtWarps][head_size]
    const WorkItem it = p.items[blockIdx.x];
    const SpanDev sp = p.spans[it.span];
    const int hs = p.head_size;
    const int g = p.group;
    const int chunk = p.chunk;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    float* qs = q_smem + warp * hs;
    const int32_t* table = p.block_tables + sp.bt_off;
    const size_t row_elems = static_cast<size_t>(p.n_kv_head) * hs;
    const T* q = static_cast<const T*>(p.q);
    const T* kp = static_cast<const T*>(p.k_pages) + static_cast<size_t>(it.kvh) * hs;
    const T* vp = static_cast<const T*>(p.v_pages) + static_cast<size_t>(it.kvh) * hs;
    T* out = static_cast<T*>(p.out);
    const int rows = it.nt * g;

    for (int r = warp; r < rows; r += kSimtWarps) {
        const int t = it.t0 + r / g;
        const int h = it.kvh * g + r % g;
        const size_t qoff = (static_cast<size_t>(sp.query_start + t) * p.n_head + h) * hs;
        for (int d = lane; d < hs; d += 32) qs[d] = to_f32(q[qoff + d]);
        __syncwarp();
        const int allowed = sp.causal_offset + t + 1;

        float m = -CUDART_INF_F;
        float l_lane = 0.f;
        float acc[kMaxDimPerLane];
#pragma unroll
        for (int k = 0; k < kMaxDimPerLane; ++k) acc[k] = 0.f;

        for (int base = 0; base < allowed; base += 32) {
            const int pos = base + lane;
            float s = -CUDART_INF_F;
            if (pos < allowed) {
                const int slot = table[pos / chunk];
                const T* kr = kp + (static_cast<size_t>(slot) * chunk + pos % chunk) * row_elems;
                float dot = 0.f;
#pragma unroll 8
                for (int d = 0; d < hs; ++d) dot = fmaf(qs[d], to_f32(kr[d]), dot);
                s = dot / p.scale; // score = dot / scale (attention.cpp:105)
            }
            const float m_new = fmaxf(m, warp_max(s));
            const float corr = expf(m - m_new); // 0 on the first step (m = -inf)
            const float w = pos < allowed ? expf(s - m_new) : 0.f;
            l_lane = l_lane * corr + w;
#pragma unroll
            for (int k = 0; k < kMaxDimPerLane; ++k) acc[k] *= corr;
            const int n = min(32, allowed - base);
            for (int j = 0; j < n; ++j) {
                const float wj = __shfl_sync(0xffffffffu, w, j);
                const int pj = base + j;
                const T* vr = vp + (static_cast<size_t>(table[pj / chunk]) * chunk + pj % chunk) * row_elems;
#pragma unroll
                for (int k = 0; k < kMaxDimPerLane; ++k) {
                    const int d = lane + 32 * k;
                    if (d < hs) acc[k] = fmaf(wj, to_f32(vr[d]), acc[k]);
                }
            }
            m = m_new;
        }
        const float inv_l = 1.f / warp_sum(l_lane);
#pragma unroll
        for (int k = 0; k < kMaxDimPerLane; ++k) {
            const int d = lane + 32 * k;
            if (d < hs) store_elem(out + qoff + d, acc[k] * inv_l);
        }
        __syncwarp();
    }
}

} // namespace

void launch_attn_simt(const AttnParams& p, int dtype, int n_items, cudaStream_t stream) {
    if (n_items <= 0) return;
    const size_t smem = sizeof(float) * kSimtWarps * p.head_size;
    if (dtype == PB_F32)
        attn_simt_kernel<float><<<n_items, kSimtWarps * 32, smem, stream>>>(p);
    else
        attn_simt_kernel<__nv_bfloat16><<<n_items, kSimtWarps * 32, smem, stream>>>(p);
    cuda_check(cudaGetLastError(), "attn_simt_kernel launch");
    count_launch();
}

} // namespace pb
