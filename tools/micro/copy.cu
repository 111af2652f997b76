// Microbenchmark: effective bandwidth of an 84 MB row copy (5120 rows of 1023
// doubles in, the same out; 8 rotating sets) for several launch structures.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int n = 1023, rows = 5120, pairs = rows / 2;
// one CTA per row pair
__global__ void __launch_bounds__(128, 8) per_pair(const double *in, double *out) {
    const double *A = in + size_t(2 * blockIdx.x) * n;
    double *O = out + size_t(2 * blockIdx.x) * n;
    for (int q = threadIdx.x; q < 2 * n; q += 128) O[q] = A[q] * 1.000001;
}
// persistent: CTAs loop over pairs
template <int NT>
__global__ void __launch_bounds__(NT) persistent(const double *in, double *out) {
    for (int p = blockIdx.x; p < pairs; p += gridDim.x) {
        const double *A = in + size_t(2 * p) * n;
        double *O = out + size_t(2 * p) * n;
#pragma unroll 4
        for (int q = threadIdx.x; q < 2 * n; q += NT) O[q] = A[q] * 1.000001;
    }
}
// persistent, 16-byte accesses (pair starts are 16-byte aligned: 2 n doubles per pair)
template <int NT>
__global__ void __launch_bounds__(NT) persistent16(const double2 *in, double2 *out) {
    for (int p = blockIdx.x; p < pairs; p += gridDim.x) {
        const double2 *A = in + size_t(p) * n;
        double2 *O = out + size_t(p) * n;
#pragma unroll 4
        for (int q = threadIdx.x; q < n; q += NT) {
            double2 v = A[q];
            v.x *= 1.000001;
            O[q] = v;
        }
    }
}
// flat grid-stride copy (the plain memcpy kernel)
__global__ void __launch_bounds__(256) flat(const double2 *in, double2 *out, size_t count) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x) {
        double2 v = in[i];
        v.x *= 1.000001;
        out[i] = v;
    }
}
int main() {
    const size_t elems = size_t(rows) * n;
    const int NB = 8;
    double *din, *dout;
    cudaMalloc(&din, elems * 8 * NB);
    cudaMalloc(&dout, elems * 8 * NB);
    cudaMemset(din, 0, elems * 8 * NB);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time = [&](auto launch, const char *name) {
        for (int i = 0; i < 5; ++i) launch(i % NB);
        cudaEventRecord(e0);
        const int R = 200;
        for (int i = 0; i < R; ++i) launch(i % NB);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-44s %.1f us  %.2f TB/s  (%s)\n", name, ms / R * 1e3, 2.0 * elems * 8 / (ms / R * 1e-3) / 1e12,
               cudaGetErrorString(cudaGetLastError()));
    };
    time([&](int b) { per_pair<<<pairs, 128>>>(din + b * elems, dout + b * elems); }, "one CTA of 128 per pair");
    for (int g : {148 * 4, 148 * 8, 148 * 16})
        time([&](int b) { persistent<128><<<g, 128>>>(din + b * elems, dout + b * elems); },
             g == 592 ? "persistent 128 thr, 4/SM" : g == 1184 ? "persistent 128 thr, 8/SM" : "persistent 128 thr, 16/SM");
    time([&](int b) { persistent<512><<<148 * 2, 512>>>(din + b * elems, dout + b * elems); }, "persistent 512 thr, 2/SM");
    time([&](int b) { persistent16<128><<<148 * 8, 128>>>((double2 *)(din + b * elems), (double2 *)(dout + b * elems)); },
         "persistent 128 thr, 8/SM, 16-byte");
    time([&](int b) { persistent16<512><<<148 * 2, 512>>>((double2 *)(din + b * elems), (double2 *)(dout + b * elems)); },
         "persistent 512 thr, 2/SM, 16-byte");
    time([&](int b) { flat<<<148 * 8, 256>>>((double2 *)(din + b * elems), (double2 *)(dout + b * elems), elems / 2); },
         "flat grid-stride, 16-byte");
    time([&](int b) { cudaMemcpyAsync(dout + b * elems, din + b * elems, elems * 8, cudaMemcpyDeviceToDevice); },
         "cudaMemcpyAsync D2D");
    return 0;
}
