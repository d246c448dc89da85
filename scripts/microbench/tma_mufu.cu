// Microbenchmarks behind the tile-pipeline design (profiling only, not the product):
//  1. MUFU ex2 throughput: f32 vs bf16x2 vs f16x2 (per SM per clock);
//  2. TMA gather throughput from L2 with 16-row page boxes {64 dims, 1 kv head, 16 rows}
//     (the paged-KV tile loads of the fused kernel) vs 64-row boxes, 148 CTAs, 8-stage ring.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2312_05516_b200/csrc -o mb tma_mufu.cu -lcuda
#include "sm100_ptx.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
using namespace pb::sm100;

__global__ void k_f32(float* out, int iters) {
    float a[16];
    for (int i = 0; i < 16; ++i) a[i] = -(threadIdx.x + i) * 1e-3f;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i])); a[i] = y - 1.0f; }
    float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_bf16x2(float* out, int iters) {
    uint32_t a[16];
    for (int i = 0; i < 16; ++i) a[i] = 0xbf80bf80u - i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(a[i])); a[i] = y ^ 0x80008000u; }
    uint32_t s = 0; for (int i = 0; i < 16; ++i) s ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(s);
}
__global__ void k_f16x2(float* out, int iters) {
    uint32_t a[16];
    for (int i = 0; i < 16; ++i) a[i] = 0xbc00bc00u - i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(a[i])); a[i] = y ^ 0x80008000u; }
    uint32_t s = 0; for (int i = 0; i < 16; ++i) s ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(s);
}
// poly exp2 (FMA/ALU pipes) throughput, same shape as the kernel's exp2_neg_poly_x2
__global__ void k_poly(float* out, int iters) {
    float2 a[8];
    for (int i = 0; i < 8; ++i) a[i] = make_float2(-(threadIdx.x + i) * 1e-3f, -(threadIdx.x + 2 * i) * 1e-3f);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) { float2 y = exp2_neg_poly_x2(a[i]); a[i] = make_float2(y.x - 1.f, y.y - 1.f); }
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

constexpr int kStages = 8;
constexpr int kTileBytes = 16384; // one 64-row x 128-dim bf16 kv tile (K or V)

// one CTA: thread 0 issues TMA for kv tiles (rows_per_box rows per box), warp 1 lane 0 consumes
__global__ void __launch_bounds__(64, 1) k_tma(const __grid_constant__ CUtensorMap tm, const int* pages, int n_pages,
                                               int tiles, int rows_per_box, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t full[kStages], empty[kStages];
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        mbar_fence_init();
    }
    __syncthreads();
    const long long t0 = clock64();
    const int boxes = 64 / rows_per_box;
    if (threadIdx.x == 0) {
        uint32_t st = 0, ph = 0;
        for (int t = 0; t < tiles; ++t) {
            mbar_wait(&empty[st], ph ^ 1);
            mbar_arrive_expect_tx(&full[st], kTileBytes);
            for (int b = 0; b < boxes; ++b) {
                const int pg = pages[(blockIdx.x * 7919 + t * boxes + b) % n_pages];
                for (int h = 0; h < 2; ++h)
                    tma_load_3d(base + st * kTileBytes + h * 8192 + b * rows_per_box * 128, &tm, &full[st], h * 64,
                                (t + b) & 7, pg * rows_per_box);
            }
            if (++st == kStages) { st = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {
        uint32_t st = 0, ph = 0;
        for (int t = 0; t < tiles; ++t) {
            mbar_wait(&full[st], ph);
            mbar_arrive(&empty[st]);
            if (++st == kStages) { st = 0; ph ^= 1; }
        }
        cyc[blockIdx.x] = clock64() - t0;
    }
}

int main() {
    float* o;
    cudaMalloc(&o, 148 * 8 * 1024 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int iters = 4096, blocks = 148 * 4, threads = 512;
    for (int which = 0; which < 4; ++which) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            if (which == 0) k_f32<<<blocks, threads>>>(o, iters);
            if (which == 1) k_bf16x2<<<blocks, threads>>>(o, iters);
            if (which == 2) k_f16x2<<<blocks, threads>>>(o, iters);
            if (which == 3) k_poly<<<blocks, threads>>>(o, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double elems = double(blocks) * threads * iters * 16;
            if (rep == 2)
                printf("{\"bench\":\"exp2\",\"kind\":\"%s\",\"ms\":%.3f,\"gexp_per_s\":%.1f,\"exp_per_sm_per_clk_at_attr_clock\":%.2f}\n",
                       which == 0 ? "mufu f32" : which == 1 ? "mufu bf16x2" : which == 2 ? "mufu f16x2" : "poly f32x2 (FMA/ALU)",
                       ms, elems / ms / 1e6, elems / (ms * 1e-3) / 148 / (clk_khz * 1e3));
        }
    }
    // ---- TMA
    const int n_kv = 8, d = 128, n_rows = 1 << 16; // 128 MB pool region: [rows][8][128] bf16 = 2 KB rows
    void* pool;
    cudaMalloc(&pool, size_t(n_rows) * n_kv * d * 2);
    cudaMemset(pool, 0, size_t(n_rows) * n_kv * d * 2);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    unsigned long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    std::vector<unsigned long long> hc(148);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kTileBytes + 1024);
    for (int footprint_mb : {16, 512}) {
        for (int rpb : {16, 32, 64}) {
            CUtensorMap tm;
            cuuint64_t dims[3] = {uint64_t(d), uint64_t(n_kv), uint64_t(n_rows)};
            cuuint64_t strides[2] = {uint64_t(d) * 2, uint64_t(n_kv) * d * 2};
            cuuint32_t box[3] = {64, 1, uint32_t(rpb)};
            cuuint32_t es[3] = {1, 1, 1};
            enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, pool, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            const int rows_used = int(std::min<long long>(n_rows, (long long)footprint_mb * 1024 * 1024 / (n_kv * d * 2)));
            const int n_pages = rows_used / rpb;
            std::vector<int> hp(n_pages);
            srand(1);
            for (int i = 0; i < n_pages; ++i) hp[i] = rand() % n_pages;
            int* dp;
            cudaMalloc(&dp, n_pages * 4);
            cudaMemcpy(dp, hp.data(), n_pages * 4, cudaMemcpyHostToDevice);
            const int tiles = 4000;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                k_tma<<<148, 64, kStages * kTileBytes + 1024>>>(tm, dp, n_pages, tiles, rpb, cyc);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                cudaMemcpy(hc.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
                double mc = 0;
                for (auto c : hc) mc += double(c) / 148;
                if (rep == 2)
                    printf("{\"bench\":\"tma\",\"footprint_mb\":%d,\"rows_per_box\":%d,\"boxes_per_tile\":%d,\"ms\":%.3f,"
                           "\"tb_per_s\":%.2f,\"bytes_per_sm_clk\":%.1f,\"clk_per_box\":%.1f}\n",
                           footprint_mb, rpb, 2 * 64 / rpb, ms, 148.0 * tiles * kTileBytes / (ms * 1e-3) / 1e12,
                           double(tiles) * kTileBytes / mc, mc / (double(tiles) * 2 * 64 / rpb));
            }
            cudaFree(dp);
        }
    }
    printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
}
