// Microbenchmark: fp64 DFMA / DADD throughput and shared-memory LDS.128
// bandwidth per SM on the local GPU.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double *out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;
}
__global__ void dadd_kernel(double *out, int iters, double a) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = x[i] + a;
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;
}
__global__ void lds_kernel(double *out, int iters) {
    __shared__ double2 buf[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, i);
    __syncthreads();
    double2 acc = make_double2(0, 0);
    int idx = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            double2 v = buf[(idx + r * 256) & 2047];
            acc.x += v.x;
            acc.y += v.y;
        }
        idx += 1;
    }
    if (acc.x == 1.2345) out[0] = acc.y;
}
int main() {
    double *d;
    cudaMalloc(&d, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int threads : {256, 512, 1024}) {
        const int iters = 20000;
        dfma_kernel<<<sms * 2, threads>>>(d, 100, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        dfma_kernel<<<sms * 2, threads>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double ops = double(sms) * 2 * threads * iters * 8;
        printf("DFMA threads/CTA %d: %.2f TFLOP/s (%.1f DFMA/clk/SM at %d MHz)\n", threads, 2 * ops / ms / 1e9,
               ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
        dadd_kernel<<<sms * 2, threads>>>(d, iters, 1e-9);
        cudaEventRecord(e0);
        dadd_kernel<<<sms * 2, threads>>>(d, iters, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("DADD threads/CTA %d: %.1f DADD/clk/SM\n", threads, ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
    {
        const int iters = 20000, threads = 512;
        lds_kernel<<<sms * 2, threads>>>(d, 100);
        cudaEventRecord(e0);
        lds_kernel<<<sms * 2, threads>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double bytes = double(sms) * 2 * threads * iters * 8 * 16;
        printf("LDS.128: %.1f B/clk/SM\n", bytes / (ms * 1e-3) / sms / (clk * 1e3));
    }
    return 0;
}
