// FP64 pipe microbenchmark for the roofline of the active-flow path:
// DFMA throughput (many independent chains per thread, full GPU) and the
// dependent-chain latency (one warp, one chain).  nvcc -arch=sm_100a -O3 fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dfma_chains(double* out, int iters, double a, double b) {
    double x[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < CH; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < CH; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double a = 0.999999, b = 1e-7;
    // throughput: 8 chains per thread, 8 CTAs of 256 threads per SM
    const int iters = 20000, blocks = sms * 8, threads = 256;
    dfma_chains<8><<<blocks, threads>>>(out, 100, a, b);
    cudaEventRecord(e0);
    dfma_chains<8><<<blocks, threads>>>(out, iters, a, b);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fma_s = (double)blocks * threads * 8.0 * iters / (ms * 1e-3);
    printf("{\"dfma_per_s\": %.4g, \"fp64_tflops\": %.2f, \"dfma_per_clk_per_sm\": %.1f, ",
           fma_s, 2 * fma_s / 1e12, fma_s / sms / (clk * 1e3));
    // latency: one warp, one dependent chain
    const int it2 = 200000;
    dfma_chains<1><<<1, 32>>>(out, 100, a, b);
    cudaEventRecord(e0);
    dfma_chains<1><<<1, 32>>>(out, it2, a, b);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("\"dfma_latency_ns\": %.3f, \"dfma_latency_clk_at_max\": %.1f, \"sms\": %d, \"max_clk_mhz\": %d}\n",
           ms * 1e6 / it2, ms * 1e-3 / it2 * clk * 1e3, sms, clk / 1000);
    return 0;
}
