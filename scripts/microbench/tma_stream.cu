// Microbenchmark (profiling only, not the product): how many bytes one SM can stream from HBM
// with TMA, as a function of the bytes it keeps in flight.  Each CTA (one per SM) streams its
// own 4 MiB region (no reuse, > L2 in total at 148 CTAs) in 16 KiB tiles through a ring of
// `stages` tiles: one thread issues a tile's boxes as soon as a stage is free and waits for the
// oldest tile.  Boxes are {64 bf16, 1, rows} of a [row][8][128] bf16 tensor (the paged-KV box
// shape, rows = 16 for 16-token pages) or {64, 8, rows/8} (8x larger boxes, same bytes).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2312_05516_b200/csrc -o tma_stream tma_stream.cu -lcuda
#include "sm100_ptx.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
using namespace pb::sm100;

constexpr int kTile = 16384;
constexpr int kMaxStages = 12;

__global__ void k_stream(const __grid_constant__ CUtensorMap tm, int stages, int tiles, int big, unsigned long long* cyc) {
    extern __shared__ uint8_t raw[];
    uint8_t* buf = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    __shared__ uint64_t full[kMaxStages];
    if (threadIdx.x != 0) return;
    for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
    mbar_fence_init();
    const int row0 = blockIdx.x * (tiles * 8);  // 8 rows of [8][128] bf16 (2 KB each) per 16 KB tile
    const long long t0 = clock64();
    auto issue = [&](int t) {
        const int st = t % stages;
        mbar_arrive_expect_tx(&full[st], kTile);
        uint8_t* dst = buf + st * kTile;
        if (big) {  // 2 boxes {64, 8 heads, 8 rows}: 8 KB each
            for (int h = 0; h < 2; ++h) tma_load_3d(dst + h * 8192, &tm, &full[st], h * 64, 0, row0 + t * 8);
        } else {    // 8 boxes {64, 1 head, 16 rows}: 2 KB each (heads 0..3 x halves)
            for (int b = 0; b < 8; ++b) tma_load_3d(dst + b * 2048, &tm, &full[st], (b & 1) * 64, b >> 1, row0 + t * 8);
        }
    };
    for (int t = 0; t < stages && t < tiles; ++t) issue(t);
    for (int t = 0; t < tiles; ++t) {
        mbar_wait(&full[t % stages], (t / stages) & 1);
        if (t + stages < tiles) issue(t + stages);
    }
    cyc[blockIdx.x] = clock64() - t0;
}

int main() {
    const int n_rows = 148 * 256 * 8 + 64;  // 148 CTAs x 256 tiles x 8 rows of 2 KB
    void* pool;
    cudaMalloc(&pool, size_t(n_rows) * 8 * 128 * 2);
    cudaMemset(pool, 0, size_t(n_rows) * 8 * 128 * 2);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    unsigned long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    std::vector<unsigned long long> hc(148);
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxStages * kTile + 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    for (int big : {0, 1}) {
        CUtensorMap tm;
        cuuint64_t dims[3] = {128, 8, uint64_t(n_rows)};
        cuuint64_t strides[2] = {128 * 2, 8 * 128 * 2};
        cuuint32_t box[3] = {64, big ? 8u : 1u, big ? 8u : 16u};
        cuuint32_t es[3] = {1, 1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, pool, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int grid : {8, 148}) {
            for (int stages : {2, 4, 6, 8, 12}) {
                const int tiles = 256;
                float ms = 0;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaEventRecord(a);
                    k_stream<<<grid, 32, kMaxStages * kTile + 1024>>>(tm, stages, tiles, big, cyc);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    cudaEventElapsedTime(&ms, a, b);
                }
                cudaMemcpy(hc.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
                double mc = 0;
                for (int i = 0; i < grid; ++i) mc += double(hc[i]) / grid;
                const double bytes = double(tiles) * kTile;
                printf("{\"bench\":\"tma_stream\",\"boxes_per_tile\":%d,\"grid\":%d,\"stages\":%d,\"inflight_kb\":%d,"
                       "\"gbs_per_cta\":%.1f,\"gbs_total\":%.0f,\"ms\":%.3f}\n",
                       big ? 2 : 8, grid, stages, stages * 16, bytes / (mc / (clk_khz * 1e3)) / 1e9,
                       grid * bytes / (ms * 1e-3) / 1e9, ms);
            }
        }
    }
    printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
}
