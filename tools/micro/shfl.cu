// Microbenchmark: do warp shuffles and shared-memory accesses share one data path?
// LDS.128 only, SHFL only, both interleaved (bytes per clock per SM).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double *out, int iters) {
    __shared__ double2 buf[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, i);
    __syncthreads();
    double2 acc = make_double2(threadIdx.x, 1.0);
    int idx = threadIdx.x;
    unsigned a = threadIdx.x, b = threadIdx.x * 3, c = threadIdx.x * 5, d = threadIdx.x * 7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            if (MODE & 1) {
                double2 v = buf[(idx + r * 256) & 2047];
                acc.x += v.x;
                acc.y += v.y;
            }
            if (MODE & 2) {   // 4 x 32-bit shuffles = 16 bytes per lane, like one LDS.128
                a = __shfl_xor_sync(0xffffffffu, a, 1 + (r & 15));
                b = __shfl_xor_sync(0xffffffffu, b, 2 + (r & 7));
                c = __shfl_xor_sync(0xffffffffu, c, 3 + (r & 3));
                d = __shfl_xor_sync(0xffffffffu, d, 5 + (r & 1));
            }
        }
        idx += 1;
    }
    if (acc.x == 1.2345 || a + b + c + d == 12345u) out[0] = acc.y;
}
int main() {
    double *d;
    cudaMalloc(&d, 8);
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](auto kern, const char *name, double bytes_per_iter_thread) {
        const int iters = 20000, threads = 512;
        kern<<<sms * 2, threads>>>(d, 100);
        cudaEventRecord(e0);
        kern<<<sms * 2, threads>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = double(sms) * 2 * threads * iters * bytes_per_iter_thread;
        printf("%-28s %.1f B/clk/SM   (%.2f ms)\n", name, bytes / (ms * 1e-3) / sms / (clk * 1e3), ms);
    };
    run(k<1>, "LDS.128 only", 8 * 16);
    run(k<2>, "SHFL only (4 x b32 = 16 B)", 8 * 16);
    run(k<3>, "LDS.128 + SHFL interleaved", 8 * 32);
    return 0;
}
