// Single-token (decode) spans, tcgen05 split-KV path: the stand-alone launch (decode-only
// batches, or PB_PLAN_SEPARATE_DECODE).  The pipeline itself is decode_tc_cta.cuh, shared with
// the fused launch (sm100_attn.cu).
#include "decode_tc_cta.cuh"
#include "append_prologue.cuh"
#include "pb_common.hpp"
#include "sm100_attn.hpp"

#include <algorithm>

namespace pb {

namespace {

using namespace pb::sm100;
using namespace pb::dtc;

template <int G>
__global__ void __launch_bounds__(kDtThreads, 1)
    attn_decode_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const AttnParams p) {
    extern __shared__ uint8_t smem_raw[];
    DtSmem& s = *reinterpret_cast<DtSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5;
    append_prologue(p, p.work_counter); // fused K/V append, when the launch carries new rows
    if (threadIdx.x == 0) {
        decode_cta_init(s);
        mbar_fence_init();
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
    }
    if (warp == 1) tmem_alloc<kTmemCols>(&s.tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem_base;
    int* ctr = p.work_counter; // [4] next unit, [5] retired CTAs (self-resetting)
    decode_cta_run<G>(s, tmem, &tm_q, &tm_k, &tm_v, p, p.items, p.n_items, ctr + 4, 0, 1, 2, 6);
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(ctr + 5, 1) == static_cast<int>(gridDim.x) - 1) {
            ctr[4] = 0;
            ctr[5] = 0;
        }
    }
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
}

__global__ void __launch_bounds__(256) append_spans_kernel(const AttnParams p) {
    append_rows(p, static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5),
                static_cast<int>((gridDim.x * blockDim.x) >> 5));
}

template <int G>
void launch_dt(const AttnParams& p, const CUtensorMap* maps, cudaStream_t st) {
    const size_t smem = sizeof(DtSmem) + 1024;
    static std::once_flag attr[kMaxDevices];
    set_smem_once(attr, attn_decode_tc_kernel<G>, smem, "cudaFuncSetAttribute(decode tc smem)");
    const int grid = std::max(1, std::min(device_sms(), p.n_items));
    if (!p.k_new) {
        attn_decode_tc_kernel<G><<<grid, kDtThreads, smem, st>>>(maps[3], maps[1], maps[2], p);
        cuda_check(cudaGetLastError(), "attn_decode_tc launch");
        count_launch();
        return;
    }
    // fused append: its grid barrier needs co-resident CTAs (cooperative launch), else the
    // rows get their own launch first (see launch_fused, sm100_attn.cu)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kDtThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute coop{};
    coop.id = cudaLaunchAttributeCooperative;
    coop.val.cooperative = 1;
    cfg.attrs = &coop;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, attn_decode_tc_kernel<G>, maps[3], maps[1], maps[2], p);
    if (e == cudaSuccess) {
        count_launch();
        return;
    }
    if (e != cudaErrorCooperativeLaunchTooLarge) cuda_check(e, "attn_decode_tc cooperative launch");
    cudaGetLastError();
    launch_append_spans(p, st);
    AttnParams q = p;
    q.k_new = nullptr;
    q.v_new = nullptr;
    attn_decode_tc_kernel<G><<<grid, kDtThreads, smem, st>>>(maps[3], maps[1], maps[2], q);
    cuda_check(cudaGetLastError(), "attn_decode_tc launch");
    count_launch();
}

} // namespace

void launch_append_spans(const AttnParams& p, cudaStream_t stream) {
    if (!p.k_new || p.total_tokens <= 0) return;
    const int grid = std::max(1, std::min(1184, (p.total_tokens + 7) / 8));
    append_spans_kernel<<<grid, 256, 0, stream>>>(p);
    cuda_check(cudaGetLastError(), "append launch");
    count_launch();
}

bool decode_tc_supports(int head_size, int chunk, int group) {
    return head_size == 128 && chunk >= 8 && chunk <= 128 && (128 % chunk) == 0 && group >= 1 && group <= kN;
}

void launch_attn_decode_tc(const AttnParams& p, const pb_attn_shape& shape, Sm100Cache& cache, int64_t total_tokens,
                           cudaStream_t stream) {
    if (p.n_items <= 0) return;
    sm100_prepare_maps(p, shape, cache, total_tokens);
    const auto* maps = reinterpret_cast<const CUtensorMap*>(cache.maps);
    if (p.group <= 8) launch_dt<8>(p, maps, stream);
    else launch_dt<16>(p, maps, stream);
}

} // namespace pb
