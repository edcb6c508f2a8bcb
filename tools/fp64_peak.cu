// fp64_peak.cu -- measured fp64 FMA throughput of this GPU (denominator of the "alu" roofline in
// bench.py): every thread runs 8 independent DFMA chains; grid = 148 SMs x 8 blocks of 256 threads.
// Prints one JSON line {"fp64_tflops": ..., "sm_mhz_during": ...}.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_dfma(double *out, int iters, double a, double b)
{
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[threadIdx.x] = s;   // never true; keeps the chains alive
}

int main()
{
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double *out;
    cudaMalloc(&out, 1024 * sizeof(double));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(a);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads * reps;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    printf("{\"fp64_tflops\": %.3f, \"sms\": %d, \"ms\": %.3f, \"max_clock_mhz\": %.0f, \"err\": \"%s\"}\n",
           flops / (ms * 1e-3) / 1e12, sms, ms, clk / 1e3, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
