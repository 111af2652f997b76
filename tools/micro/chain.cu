// Microbenchmark: one warp running a dependent DFMA chain with the results
// stored to / operands loaded from shared memory, as in the mode-sliced Thomas
// sweep.  Cycles per row for several instruction mixes.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/micro/chain.cu -o tools/micro/chain
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int W = 36, ROWS = 64, TILES = 64;
template <int MODE>
__global__ void k(double *out, long long *cyc, double a, int poll) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bar;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < ROWS * W * 2; i += blockDim.x) sm[i] = 1e-3 * i;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    __syncthreads();
    if (warp == 2) {   // polling warp
        if (lane == 0 && poll) {
            uint32_t done = 0;
            for (int it = 0; it < 20000 && !done; ++it)
                asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                             : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(0) : "memory");
        }
        return;
    }
    double y = lane * 1e-3;
    double *sl = sm + lane;
    long long c0 = clock64();
    for (int t = 0; t < TILES; ++t) {
        double *s = sl + (t & 1) * ROWS * W;
#pragma unroll
        for (int c = 0; c < ROWS / 16; ++c) {
            double d[16], o[16];
            if (MODE >= 2) {
#pragma unroll
                for (int r = 0; r < 16; ++r) d[r] = s[(c * 16 + r) * W];
            } else {
#pragma unroll
                for (int r = 0; r < 16; ++r) d[r] = 1e-3 * r;
            }
            if (MODE == 4) {   // all DFMAs, then all stores
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    y = fma(a, y, d[r]);
                    o[r] = y;
                }
                asm volatile("" ::: "memory");
#pragma unroll
                for (int r = 0; r < 16; ++r) s[(c * 16 + r) * W] = o[r];
            } else {
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    y = fma(a, y, d[r]);
                    if (MODE >= 1) s[(c * 16 + r) * W] = y;
                }
            }
        }
    }
    long long c1 = clock64();
    if (threadIdx.x == 0) cyc[0] = c1 - c0;
    out[threadIdx.x] = y;
}
int main() {
    double *out;
    long long *cyc, h;
    cudaMalloc(&out, 4096);
    cudaMalloc(&cyc, 64);
    const int smem = ROWS * W * 2 * 8;
    auto run = [&](auto kern, const char *name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int warps : {1, 2, 3})
            for (int poll : {0, 1}) {
                if (poll && warps < 3) continue;
                for (int rep = 0; rep < 2; ++rep) kern<<<1, 32 * warps, smem>>>(out, cyc, 0.999, poll);
                cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
                printf("%-40s warps %d poll %d: %.2f cycles/row\n", name, warps, poll, h / double(TILES * ROWS));
            }
    };
    run(k<0>, "DFMA chain only");
    run(k<1>, "DFMA + STS interleaved");
    run(k<2>, "LDS + DFMA + STS interleaved");
    run(k<4>, "LDS + DFMA chain, then STS");
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
