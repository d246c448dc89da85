// Microbenchmark (profiling only, not the product): throughput of the softmax inner loop's
// instruction mix on one SM sub-partition, with 1 or 2 warps per SMSP (the tile pipeline
// runs one softmax warp per SMSP per query tile):
//   mufu   : ex2.approx.ftz.f32 only
//   f2fp   : cvt.rn.bf16x2.f32 only (does the bf16 pack share the MUFU/XU pipe?)
//   pair   : the per-pair body of the tile softmax: FFMA2, 2 x MUFU.EX2, FADD2, F2FP
//   pair_p4: the same with one pair in four on the FMA-pipe polynomial
// Prints element-exps per SM per clock.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2312_05516_b200/csrc -o xu_mix xu_mix.cu
#include "sm100_ptx.cuh"
#include <cstdio>
#include <cstdint>
using namespace pb::sm100;

template <int KIND>
__global__ void k_mix(float* out, long long* cyc, int iters) {
    float x[32];
    for (int i = 0; i < 32; ++i) x[i] = -(threadIdx.x + i) * 1e-3f;
    float2 acc = make_float2(0.f, 0.f);
    uint32_t pk = 0;
    const float2 sc = make_float2(0.9f, 0.9f), nm = make_float2(-0.5f, -0.5f);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
            if (KIND == 0) {
                x[c] = ex2(x[c]) - 1.f;
                x[c + 1] = ex2(x[c + 1]) - 1.f;
            } else if (KIND == 1) {
                uint32_t r = pack_bf16x2(x[c], x[c + 1]);
                pk ^= r;
                x[c] += 1e-7f;
            } else {
                const float2 a = fma2(make_float2(x[c], x[c + 1]), sc, nm);
                float2 e;
                if (KIND == 3 && ((c >> 1) & 3) == 3) {
                    e = exp2_neg_poly_x2(a);
                } else {
                    e.x = ex2(a.x);
                    e.y = ex2(a.y);
                }
                acc = add2(acc, e);
                pk ^= pack_bf16x2(e.x, e.y);
                x[c] = e.x;
                x[c + 1] = e.y;
            }
        }
    }
    const long long t1 = clock64();
    float s = acc.x + acc.y + __uint_as_float(pk);
    for (int i = 0; i < 32; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int KIND>
void run(const char* name, int threads, float* d_out, long long* d_cyc, int sms) {
    const int iters = 2000;
    k_mix<KIND><<<sms, threads>>>(d_out, d_cyc, 10);
    cudaDeviceSynchronize();
    k_mix<KIND><<<sms, threads>>>(d_out, d_cyc, iters);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, d_cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += h[i];
    avg /= sms;
    const double elems = (double)iters * 32.0 * threads;
    printf("{\"bench\":\"xu_mix\",\"kind\":\"%s\",\"warps_per_smsp\":%d,\"elem_per_sm_clk\":%.2f,\"err\":\"%s\"}\n", name,
           threads / 128, elems / avg, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* d_out;
    long long* d_cyc;
    cudaMalloc(&d_out, sizeof(float) * sms * 1024);
    cudaMalloc(&d_cyc, sizeof(long long) * 1024);
    for (int t : {128, 256, 512}) {
        run<0>("mufu", t, d_out, d_cyc, sms);
        run<1>("f2fp", t, d_out, d_cyc, sms);
        run<2>("pair", t, d_out, d_cyc, sms);
        run<3>("pair_p4", t, d_out, d_cyc, sms);
    }
    return 0;
}
