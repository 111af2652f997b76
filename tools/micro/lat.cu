// Microbenchmarks: dependent-chain latency of DFMA / DADD / DMUL (one warp),
// issue cost of small cp.async.bulk copies (one lane, 16 lanes), LDS latency.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/micro/lat.cu -o /tmp/lat
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void chain(double *out, long long *cyc, double a, double b, int n) {
    double x = threadIdx.x * 1e-3;
    long long c0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) x = fma(x, a, b);
    }
    long long c1 = clock64();
    double y = threadIdx.x * 1e-3;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) y = y + a;
    }
    long long c2 = clock64();
    double z = threadIdx.x * 1e-3 + 1;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) z = z * a;
    }
    long long c3 = clock64();
    // two independent chains
    double p = threadIdx.x * 1e-3, q = p + 1;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            p = fma(p, a, b);
            q = fma(q, a, b);
        }
    }
    long long c4 = clock64();
    double r4[4] = {p, q, x, y};
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int v = 0; v < 4; ++v) r4[v] = fma(r4[v], a, b);
        }
    }
    long long c5 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = c1 - c0;
        cyc[1] = c2 - c1;
        cyc[2] = c3 - c2;
        cyc[3] = c4 - c3;
        cyc[4] = c5 - c4;
    }
    out[threadIdx.x] = x + y + z + p + q + r4[0] + r4[1] + r4[2] + r4[3];
}
__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void bulk(const double *src, long long *cyc, int rows, int bytes, int lanes, double *sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    long long c0 = clock64();
    for (int r = threadIdx.x; r < rows; r += lanes) {
        if (threadIdx.x < lanes) {
            asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(s32(&bar)), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             s32(sm + size_t(r) * bytes)),
                         "l"(src + size_t(r) * 1024), "r"(bytes), "r"(s32(&bar))
                         : "memory");
        }
    }
    __syncwarp();
    long long c1 = clock64();
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&bar)) : "memory");
    uint32_t done = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(s32(&bar)), "r"(0) : "memory");
    } while (!done);
    long long c2 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = c1 - c0;
        cyc[1] = c2 - c0;
    }
    sink[threadIdx.x] = reinterpret_cast<double *>(sm)[threadIdx.x];
}
int main() {
    double *out;
    long long *cyc, h[8];
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 64);
    for (int rep = 0; rep < 2; ++rep) chain<<<1, 32>>>(out, cyc, 0.999, 0.001, 256);
    cudaMemcpy(h, cyc, 40, cudaMemcpyDeviceToHost);
    printf("dependent chain cycles/op: DFMA %.2f DADD %.2f DMUL %.2f | 2 chains: %.2f per pair | 4 chains: %.2f per quad\n",
           h[0] / 4096.0, h[1] / 4096.0, h[2] / 4096.0, h[3] / 4096.0, h[4] / 4096.0);
    double *src;
    cudaMalloc(&src, 64 << 20);
    cudaMemset(src, 0, 64 << 20);
    cudaFuncSetAttribute(bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int bytes : {304, 1024, 4096})
        for (int lanes : {1, 16, 32}) {
            int rows = 32;
            for (int rep = 0; rep < 2; ++rep) bulk<<<1, 32, 200 * 1024>>>(src, cyc, rows, bytes, lanes, out);
            cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
            printf("bulk %d B x %d rows, %d lanes issuing: issue %lld cyc (%.1f per copy), all landed %lld cyc\n", bytes, rows,
                   lanes, h[0], h[0] / double(rows), h[1]);
        }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
