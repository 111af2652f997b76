// Standalone timing of the warp-private N = 1024 row-pair DST-I (rsolve32.cu's
// transform): global rows -> registers -> FFT -> xslot region -> coalesced rows.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include tools/k3w32/fft_bench.cu -o /tmp/fftb
#include "../experimental/k3_warp_fft.cu"
#include <vector>
namespace fd { void *dmalloc(size_t b) { void *p; cudaMalloc(&p, b); return p; } void dfree(void *p) { cudaFree(p); } }
#include <cmath>
using namespace fd;
using namespace fd::r32;

// compute only: inputs synthesised from the lane index (no HBM loads)
__device__ __noinline__ void xform_synth(double h2, double2 *reg, int lane, LaneK lk, int pr) {
    double2 v[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) v[r] = make_double2(lk.alpha(r, h2) * (pr + r), lane * 1e-3 + r);
    transform(v, reg, lane, lk);
}
template <int CTAS, int MODE>
__global__ void __launch_bounds__(128, CTAS) dst_rows_m(const double *in, double *out, int pairs, double h2) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    double2 *reg = reinterpret_cast<double2 *>(smem_raw + size_t(wp) * REG);
    LaneK lk;
    lk.init(lane);
    double acc = 0;
    for (int pr = blockIdx.x * 4 + wp; pr < pairs; pr += gridDim.x * 4) {
        xform_synth(h2, reg, lane, lk, pr);
        if (MODE == 1) {
            double *oa = out + size_t(2 * pr) * 1023, *ob = oa + 1023;
#pragma unroll 8
            for (int q = lane; q < 1023; q += 32) {
                const double2 t = reg[phys(xslot(q))];
                oa[q] = t.x;
                ob[q] = t.y;
            }
        } else {
            acc += reg[lane].x;
        }
        __syncwarp();
    }
    if (acc == 1.2345) out[0] = acc;
}
template <int CTAS>
__global__ void __launch_bounds__(128, CTAS) dst_rows(const double *in, double *out, int pairs, double h2) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    double2 *reg = reinterpret_cast<double2 *>(smem_raw + size_t(wp) * REG);
    LaneK lk;
    lk.init(lane);
    for (int pr = blockIdx.x * 4 + wp; pr < pairs; pr += gridDim.x * 4) {
        const double *A = in + size_t(2 * pr) * 1023;
        xform_global(A, A + 1023, h2, reg, lane, lk);
        double *oa = out + size_t(2 * pr) * 1023, *ob = oa + 1023;
#pragma unroll 8
        for (int q = lane; q < 1023; q += 32) {
            const double2 t = reg[phys(xslot(q))];
            oa[q] = t.x;
            ob[q] = t.y;
        }
        __syncwarp();
    }
}

int main() {
    const int rows = 5120, n = 1023, pairs = rows / 2;
    std::vector<double> h(size_t(rows) * n);
    unsigned s = 1;
    for (auto &x : h) { s = s * 1664525u + 1013904223u; x = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
    double *d_in, *d_out;
    const int NB = 8;   // rotating buffers > L2
    cudaMalloc(&d_in, h.size() * 8 * NB);
    cudaMalloc(&d_out, h.size() * 8 * NB);
    for (int b = 0; b < NB; ++b) cudaMemcpy(d_in + b * h.size(), h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    const double h2 = 0.5 * sqrt(2.0 / 1024);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto run = [&](auto kern, int ctas, const char *name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, W * REG);
        const int grid = occ * sms;
        for (int i = 0; i < 3; ++i) kern<<<grid, 128, W * REG>>>(d_in, d_out, pairs, h2);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        const int it = 200;
        cudaEventRecord(e0);
        for (int i = 0; i < it; ++i)
            kern<<<grid, 128, W * REG>>>(d_in + (i % NB) * h.size(), d_out + (i % NB) * h.size(), pairs, h2);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / it;
        printf("%s: occ %d/SM grid %d: %.2f us per %d rows, %.0f GB/s (16 B/pt), err %s\n", name, occ, grid, us, rows,
               16.0 * rows * n / us * 1e-3, cudaGetErrorString(cudaGetLastError()));
    };
    run(dst_rows<2>, 2, "lb2");
    run(dst_rows<3>, 3, "lb3");
    run(dst_rows_m<2, 0>, 2, "compute-only lb2");
    run(dst_rows_m<2, 1>, 2, "compute+store lb2");
    run(dst_rows_m<3, 0>, 3, "compute-only lb3");
    // check two rows against the O(n^2) DST-I
    std::vector<double> o(size_t(4) * n);
    cudaMemcpy(o.data(), d_out + (199 % NB) * h.size(), o.size() * 8, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int r = 0; r < 4; ++r)
        for (int k = 1; k <= n; ++k) {
            long double acc = 0;
            for (int j = 1; j <= n; ++j) acc += h[size_t(r) * n + j - 1] * sinl(3.14159265358979323846264338327950288L * j * k / 1024);
            acc *= sqrtl(2.0L / 1024);
            err = fmax(err, fabs((double)acc - o[size_t(r) * n + k - 1]));
            mx = fmax(mx, fabs((double)acc));
        }
    printf("max abs err %.3e (max |X| %.3e)\n", err, mx);
    return 0;
}
