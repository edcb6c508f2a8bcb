// fp64_latency.cu -- fp64 FMA throughput vs warps/SM and independent chains per thread (development
// aid: how much ILP x occupancy the DFMA pipe needs on this GPU).
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k_chain(double *out, int iters, double a, double b)
{
    double x[C];
#pragma unroll
    for (int k = 0; k < C; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 32; ++r)
#pragma unroll
            for (int k = 0; k < C; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < C; ++k) s += x[k];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <int C>
void run(double *out, int warps_per_sm, int sms)
{
    const int threads = 32 * (warps_per_sm < 32 ? warps_per_sm : 32);
    const int blocks = sms * (warps_per_sm * 32 / threads);
    const int iters = 2048 / C;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_chain<C><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(a);
    k_chain<C><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double fl = 2.0 * 32 * C * (double)iters * blocks * threads;
    printf("{\"warps_per_sm\": %d, \"chains\": %d, \"tflops\": %.2f}\n", warps_per_sm, C, fl / (ms * 1e-3) / 1e12);
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 4096 * sizeof(double));
    for (int w : {4, 8, 12, 16, 20, 24, 32, 48, 64}) {
        run<1>(out, w, sms);
        run<2>(out, w, sms);
        run<4>(out, w, sms);
    }
    return 0;
}
