// Back-to-back launch cost of an (almost) empty kernel shaped like the fused solve:
// 148 CTAs x 512 threads, 225 KB dynamic shared memory, normal vs cooperative launch,
// with and without a grid-wide barrier.   nvcc -arch=sm_100a -O3 -o launch launch.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void __launch_bounds__(512, 1) k_plain(int *p) {
    extern __shared__ unsigned char sm[];
    if (threadIdx.x == 0 && p) sm[0] = 1;
}
__global__ void __launch_bounds__(512, 1) k_coop(int *p, int syncs) {
    extern __shared__ unsigned char sm[];
    cg::grid_group g = cg::this_grid();
    if (threadIdx.x == 0 && p) sm[0] = 1;
    for (int i = 0; i < syncs; ++i) g.sync();
}
int main() {
    const int smem = 225 * 1024, steps = 2000;
    cudaFuncSetAttribute(k_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int *p = nullptr;
    auto run = [&](const char *name, int mode, int syncs) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            for (int i = 0; i < steps; ++i) {
                if (mode == 0) k_plain<<<148, 512, smem>>>(p);
                else {
                    void *args[] = {&p, &syncs};
                    cudaLaunchCooperativeKernel((void *)k_coop, dim3(148), dim3(512), args, smem, 0);
                }
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-40s %.2f us per launch (%s)\n", name, ms * 1e3 / steps, cudaGetErrorString(cudaGetLastError()));
    };
    run("normal launch, empty", 0, 0);
    run("cooperative launch, empty", 1, 0);
    run("cooperative launch, 2 grid syncs", 1, 2);
    run("cooperative launch, 10 grid syncs", 1, 10);
    return 0;
}
