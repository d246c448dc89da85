// Microbenchmark (profiling only, not the product): tcgen05.mma kind::f16 throughput per SM
// for the instruction shapes of the tile pipeline, one CTA per SM, one thread issuing a long
// stream of MMAs on resident operands (no TMA, no softmax):
//   SS  M=128 N=64  (S = Q K^T with 64-row kv tiles, both operands from shared memory)
//   SS  M=128 N=128 / N=256
//   TS  M=128 N=128 (O += P V, A = P from TMEM, B = V from shared memory, MN-major)
//   TS  M=128 N=64
// Prints MACs per SM per clock (clock64 on the issuing thread) vs the 4096 MAC/clk/SM
// nominal dense bf16 rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2312_05516_b200/csrc -o mma_rate mma_rate.cu
#include "sm100_ptx.cuh"
#include <cstdio>
#include <cstdint>
using namespace pb::sm100;

__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k_mma(long long* cyc, int iters) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint32_t tmem_sh;
    __shared__ uint64_t bar;
    uint8_t* a = base;                 // 128 rows x 128 dims bf16, SW128 K-major: [2][128][128 B]
    uint8_t* b = base + 32768;         // N rows x 128 dims (K-major) or 64 rows x N dims (MN-major)
    for (int i = threadIdx.x; i < (32768 + 65536) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(base)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x < 32) tmem_alloc<512>(&tmem_sh);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_sh;
    if (threadIdx.x == 0) {
        const uint32_t idesc = umma_idesc_bf16(128, N, false, TS);
        const uint64_t ad = umma_desc_sw128(smem_u32(a), 16, 1024);
        const uint64_t bd = TS ? umma_desc_sw128(smem_u32(b), 8192, 1024) : umma_desc_sw128(smem_u32(b), 16, 1024);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (TS) {
                // K = 64 kv rows per block: 4 instructions of K=16, A = P (bf16) at TMEM cols [0,32)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    umma_ts(tmem + 256, tmem + kk * 8, bd + kk * (2048 >> 4), idesc, 1u);
            } else {
                // K = 128 dims per block: 8 instructions of K=16
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t oa = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                    const uint32_t ob = ((kk >> 2) * (N * 128) + (kk & 3) * 32) >> 4;
                    umma_bf16_ss(tmem + 256, ad + oa, bd + ob, idesc, 1u);
                }
            }
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        cyc[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int N, bool TS>
void run(const char* name, long long* d_cyc, int sms) {
    const int iters = 4000;
    const size_t smem = 32768 + 65536 + 1024;
    cudaFuncSetAttribute(k_mma<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_mma<N, TS><<<sms, 128, smem>>>(d_cyc, 10);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_mma<N, TS><<<sms, 128, smem>>>(d_cyc, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[1024];
    cudaMemcpy(h, d_cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += h[i];
    avg /= sms;
    const double k_per_block = TS ? 64 : 128;
    const double macs = (double)iters * 128.0 * N * k_per_block;
    printf("{\"bench\":\"mma\",\"kind\":\"%s\",\"N\":%d,\"ms\":%.3f,\"mac_per_sm_clk\":%.1f,\"frac_of_4096\":%.3f,\"tflops\":%.1f,\"err\":\"%s\"}\n",
           name, N, ms, macs / avg, macs / avg / 4096.0, 2.0 * macs * sms / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d_cyc;
    cudaMalloc(&d_cyc, sizeof(long long) * 1024);
    run<64, false>("SS M128 K-major A,B", d_cyc, sms);
    run<128, false>("SS M128 K-major A,B", d_cyc, sms);
    run<256, false>("SS M128 K-major A,B", d_cyc, sms);
    run<64, true>("TS M128 A=TMEM, B MN-major", d_cyc, sms);
    run<128, true>("TS M128 A=TMEM, B MN-major", d_cyc, sms);
    run<256, true>("TS M128 A=TMEM, B MN-major", d_cyc, sms);
    return 0;
}
