// Microbenchmark: ways to gather 16-row tiles of 304-byte row segments (row
// pitch 8184 B) from L2 into shared memory, one CTA per SM: per-row
// cp.async.bulk issued by 1/2/4/8 warps, 8-byte cp.async (LDGSTS), LDG + STS.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/micro/gather.cu -o tools/micro/gather
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_bar(uint64_t *bar, uint32_t par) {
    uint32_t done = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(s32(bar)), "r"(par) : "memory");
    } while (!done);
}
constexpr int PITCH = 1023, SEG = 38, ROWS = 1024, TILE = 16;
// mode 0: bulk per row, one expect_tx per copy; 1: bulk per row, one expect_tx per tile; 2: cp.async 8 B; 3: LDG+STS
template <int MODE>
__global__ void gather(const double *src, long long *cyc, double *sink, int warps) {
    extern __shared__ __align__(128) unsigned char sm[];
    double *slots = reinterpret_cast<double *>(sm);   // [ROWS][SEG] (whole thing resident: 311 KB is too much -> ring of 512 rows)
    __shared__ __align__(8) uint64_t bar[64];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double *base = src + size_t(blockIdx.x) * 36;   // 16-byte aligned start for even rows only
    if (tid == 0) {
        for (int i = 0; i < 64; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(&bar[i])), "r"(MODE == 2 ? warps * 32 : (MODE == 3 ? warps : 1)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    long long c0 = clock64();
    const int ntiles = ROWS / TILE;
    if (warp < warps) {
        for (int t = warp; t < ntiles; t += warps) {
            uint64_t *b = &bar[t];
            double *dst = slots + size_t(t % 32) * TILE * SEG;
            if (MODE <= 1) {
                const int r = lane;
                const double *p = base + size_t(t * TILE + r) * PITCH;
                const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
                const uint32_t bytes = 304;
                if (MODE == 1) {
                    if (lane == 0)
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes * TILE) : "memory");
                    __syncwarp();
                }
                if (r < TILE) {
                    if (MODE == 0)
                        asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                     s32(dst + r * SEG)), "l"(a), "r"(bytes), "r"(s32(b)) : "memory");
                }
                if (MODE == 0) {
                    __syncwarp();
                    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
                }
            } else {
                for (int e = lane; e < TILE * 36; e += 32) {
                    const int r = e / 36, q = e - r * 36;
                    const double *p = base + size_t(t * TILE + r) * PITCH + q;
                    if (MODE == 2)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s32(dst + e)), "l"(p) : "memory");
                    else
                        dst[e] = __ldcg(p);
                }
                if (MODE == 2)
                    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(s32(b)) : "memory");
                else {
                    __syncwarp();
                    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
                }
            }
        }
    }
    long long c1 = clock64();
    if (MODE == 2) {
        // tiles are owned by one warp each: its 32 threads arrive -> count = 32 would be right; we set warps*32, so emulate: all
        // other warps arrive for the tiles they do not own
        for (int t = 0; t < ntiles; ++t)
            if (warp < warps && (t % warps) != warp) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&bar[t])) : "memory");
    } else if (MODE == 3) {
        for (int t = 0; t < ntiles; ++t)
            if (warp < warps && (t % warps) != warp && lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&bar[t])) : "memory");
    }
    for (int t = 0; t < ntiles; ++t) wait_bar(&bar[t], 0);
    long long c2 = clock64();
    if (tid == 0) {
        cyc[blockIdx.x * 2] = c1 - c0;
        cyc[blockIdx.x * 2 + 1] = c2 - c0;
    }
    sink[blockIdx.x * blockDim.x + tid] = slots[tid];
}
int main() {
    double *src, *sink;
    long long *cyc;
    const size_t elems = size_t(5) * 1023 * 1023 + 4096;
    cudaMalloc(&src, elems * 8);
    cudaMemset(src, 0, elems * 8);
    cudaMalloc(&sink, 1 << 20);
    cudaMalloc(&cyc, 148 * 16);
    const int smem = 32 * TILE * SEG * 8;
    auto run = [&](auto kern, const char *name, int warps) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        long long h[296];
        for (int rep = 0; rep < 3; ++rep) kern<<<148, 256, smem>>>(src, cyc, sink, warps);
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        long long mi = 0, mt = 0;
        for (int c = 0; c < 148; ++c) { mi = std::max(mi, h[2 * c]); mt = std::max(mt, h[2 * c + 1]); }
        printf("%-34s warps %d: issue %6lld cyc, landed %6lld cyc -> %.1f cyc/row (148 CTAs, %d rows each)  %s\n", name, warps, mi, mt,
               mt / double(ROWS), ROWS, cudaGetErrorString(cudaGetLastError()));
    };
    for (int w : {1, 2, 4, 8}) run(gather<0>, "bulk/row, expect_tx per copy", w);
    for (int w : {1, 2, 4, 8}) run(gather<1>, "bulk/row, expect_tx per tile", w);
    for (int w : {1, 2, 4, 8}) run(gather<2>, "cp.async 8 B", w);
    for (int w : {1, 2, 4, 8}) run(gather<3>, "LDG.cg + STS", w);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
