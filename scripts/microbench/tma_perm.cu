// Check (profiling/diagnostics only): does TMA accept a 4-D tensor map whose dims are listed
// in a non-stride order -- {d, token, head, slot} over a [slot][token][head][d] page pool --
// and deliver the box {64, 16 tokens, 8 heads, 1} head-major ([head][token][128 B]) into
// shared memory (SWIZZLE_128B)?  Prints PASS/FAIL.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2312_05516_b200/csrc -o tma_perm tma_perm.cu -lcuda
#include "sm100_ptx.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
using namespace pb::sm100;

__global__ void k_load(const __grid_constant__ CUtensorMap tm, int slot, uint16_t* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* buf = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
        mbar_arrive_expect_tx(&bar, 2 * 16384);
        for (int h = 0; h < 2; ++h)
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(buf + h * 16384)),
                         "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(&bar)), "r"(h * 64), "r"(0), "r"(0), "r"(slot)
                         : "memory");
        mbar_wait(&bar, 0);
    }
    __syncthreads();
    // un-swizzle: row r (= head*16 + token) of half h, element e
    for (int i = threadIdx.x; i < 2 * 128 * 64; i += blockDim.x) {
        const int h = i / (128 * 64), r = (i / 64) % 128, e = i % 64;
        const int chunk = (e >> 3) ^ (r & 7);
        out[i] = *reinterpret_cast<const uint16_t*>(buf + h * 16384 + r * 128 + chunk * 16 + (e & 7) * 2);
    }
}

int main() {
    const int n_slots = 4, chunk = 16, n_kv = 8, d = 128;
    std::vector<uint16_t> pool(size_t(n_slots) * chunk * n_kv * d);
    for (size_t i = 0; i < pool.size(); ++i) pool[i] = uint16_t(i * 2654435761u >> 16);
    uint16_t *dp, *dout;
    cudaMalloc(&dp, pool.size() * 2);
    cudaMemcpy(dp, pool.data(), pool.size() * 2, cudaMemcpyHostToDevice);
    cudaMalloc(&dout, 2 * 128 * 64 * 2);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[4] = {uint64_t(d), uint64_t(chunk), uint64_t(n_kv), uint64_t(n_slots)};
    cuuint64_t strides[3] = {uint64_t(n_kv) * d * 2, uint64_t(d) * 2, uint64_t(chunk) * n_kv * d * 2};
    cuuint32_t box[4] = {64, uint32_t(chunk), 8, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, dp, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", int(r));
    if (r != CUDA_SUCCESS) { printf("FAIL (encode rejected)\n"); return 1; }
    cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 16384 + 1024);
    const int slot = 2;
    k_load<<<1, 128, 2 * 16384 + 1024>>>(tm, slot, dout);
    std::vector<uint16_t> got(2 * 128 * 64);
    cudaError_t e = cudaMemcpy(got.data(), dout, got.size() * 2, cudaMemcpyDeviceToHost);
    printf("cuda: %s\n", cudaGetErrorString(e));
    int bad = 0;
    for (int h = 0; h < 2; ++h)
        for (int row = 0; row < 128; ++row)
            for (int el = 0; el < 64; ++el) {
                const int head = row / 16, tok = row % 16;
                const uint16_t want = pool[((size_t(slot) * chunk + tok) * n_kv + head) * d + h * 64 + el];
                if (got[(h * 128 + row) * 64 + el] != want) ++bad;
            }
    printf("%s (%d mismatches)\n", bad ? "FAIL" : "PASS", bad);
    return bad ? 1 : 0;
}
