// Microbenchmark 2: the consumer loop of the mode-sliced Thomas sweep built up
// feature by feature (one warp; cycles per row).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int W = 36, ROWS = 64, TILES = 64, NG = 10;
__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
// F bits: 1 ping-pong prefetch, 2 predicated stores, 4 counter loads + compare, 8 fence + arrive, 16 runtime slot ring
template <int F>
__global__ void k(double *out, long long *cyc, double a, int wlim) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bar[NG];
    __shared__ uint32_t landed[2];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < ROWS * W * NG; i += blockDim.x) sm[i] = 1e-3 * i;
    if (threadIdx.x == 0) {
        for (int g = 0; g < NG; ++g) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[g])));
        landed[0] = landed[1] = 1000000;
    }
    __syncthreads();
    const bool inb = lane < wlim;
    double y = lane * 1e-3;
    uint32_t need = 0, seen = 0;
    int g = 0;
    long long c0 = clock64();
    double da[16], db[16];
    {
        const double *s = sm + lane;
#pragma unroll
        for (int r = 0; r < 16; ++r) da[r] = s[r * W];
    }
    for (int t = 0; t < TILES; ++t) {
        const int gn = (F & 16) ? (g + 1 == NG ? 0 : g + 1) : ((t + 1) % 2);
        double *s = sm + size_t((F & 16) ? g : (t % 2)) * ROWS * W + lane;
        const double *sn = sm + size_t(gn) * ROWS * W + lane;
        if (F & 4) seen = *(volatile uint32_t *)&landed[0];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            auto body = [&](double (&dc)[16], double (&dn)[16]) {
                if (F & 1) {
                    if (c < 3) {
#pragma unroll
                        for (int r = 0; r < 16; ++r) dn[r] = s[((c + 1) * 16 + r) * W];
                    } else {
                        if (F & 4) {
                            ++need;
                            while (seen < need) seen = *(volatile uint32_t *)&landed[0];
                        }
#pragma unroll
                        for (int r = 0; r < 16; ++r) dn[r] = sn[r * W];
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < 16; ++r) dc[r] = s[(c * 16 + r) * W];
                }
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    y = fma(a, y, dc[r]);
                    if (!(F & 2) || inb) s[(c * 16 + r) * W] = y;
                }
            };
            if (c & 1) body(db, da);
            else body(da, db);
        }
        if (F & 8) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&bar[g % NG])) : "memory");
        }
        g = gn;
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
    const int smem = ROWS * W * NG * 8;
    auto run = [&](auto kern, const char *name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int rep = 0; rep < 2; ++rep) kern<<<1, 32, smem>>>(out, cyc, 0.999, 32);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-60s %.2f cycles/row  %s\n", name, h / double(TILES * ROWS), cudaGetErrorString(cudaGetLastError()));
    };
    run(k<0>, "load, chain+store per chunk");
    run(k<1>, "+ ping-pong prefetch of the next chunk");
    run(k<3>, "+ predicated stores");
    run(k<7>, "+ counter load and compare per tile");
    run(k<15>, "+ fence.proxy.async + syncwarp + arrive per tile");
    run(k<31>, "+ runtime slot ring");
    run(k<25>, "prefetch + fence/arrive + ring (no counters, no pred)");
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
