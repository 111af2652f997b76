// Element-wise and reduction kernels around the solve: the 5-point stencil
// (rectsolver.apply_rect_operator, rectsolver.py:264-289), interface coupling
// gather/scatter (ddm.CouplingMap.apply, ddm.py:44-51) and the Arnoldi
// building blocks of restarted GMRES (krylov.py:103-111,141).
//
// All HBM-bound: grids are multiples of the 148 SMs, loads are coalesced,
// reductions are deterministic (fixed grid, fixed combine order: per-block
// warp-shuffle trees, then the last block to finish combines the per-block
// partials in index order), so repeated runs give bitwise-equal results.
#include "fd_internal.h"

namespace fd {

// out = A v with the reference's accumulation order; every product is rounded
// before it is added, exactly as numpy's `out[...] += d * G[...]`.
__global__ void stencil_kernel(int m, int n, double c0, double dx, double dy, double mw, double me,
                               double ms, double mn, const double *__restrict__ v,
                               double *__restrict__ out) {
    const long long total = (long long)m * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
        const double g = v[idx];
        double a = __dmul_rn(c0, g);
        if (j > 0) a = __dadd_rn(a, __dmul_rn(dy, v[idx - 1]));
        if (j < n - 1) a = __dadd_rn(a, __dmul_rn(dy, v[idx + 1]));
        if (j == 0) a = __dadd_rn(a, __dmul_rn(ms, g));
        if (j == n - 1) a = __dadd_rn(a, __dmul_rn(mn, g));
        if (i > 0) a = __dadd_rn(a, __dmul_rn(dx, v[idx - n]));
        if (i < m - 1) a = __dadd_rn(a, __dmul_rn(dx, v[idx + n]));
        if (i == 0) a = __dadd_rn(a, __dmul_rn(mw, g));
        if (i == m - 1) a = __dadd_rn(a, __dmul_rn(me, g));
        out[idx] = a;
    }
}

static int grid_for(long long N, int threads) {
    long long g = (N + threads - 1) / threads;
    const long long cap = 148LL * 16;
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

void launch_stencil(int m, int n, double delta_x, double delta_y, double kappa, double mw,
                    double me, double ms, double mn, const double *v, double *out, cudaStream_t s) {
    const double c0 = -2.0 * (delta_x + delta_y) + kappa;   // rectsolver.py:270
    const long long N = (long long)m * n;
    stencil_kernel<<<grid_for(N, 256), 256, 0, s>>>(m, n, c0, delta_x, delta_y, mw, me, ms, mn, v,
                                                    out);
    FD_CUDA(cudaGetLastError());
}

// dst[to[t]] (+)= c * src[from[t]]
__global__ void scatter_kernel(int len, const int64_t *__restrict__ from, const int64_t *__restrict__ to,
                               double c, const double *__restrict__ src, double *dst, int acc) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < len; t += gridDim.x * blockDim.x) {
        const double v = __dmul_rn(c, src[from[t]]);
        const int64_t d = to[t];
        dst[d] = acc ? __dadd_rn(dst[d], v) : v;
    }
}

void launch_scatter(int len, const int64_t *from, const int64_t *to, double c, const double *src,
                    double *dst, int accumulate, cudaStream_t s) {
    if (len <= 0) return;
    scatter_kernel<<<(len + 255) / 256, 256, 0, s>>>(len, from, to, c, src, dst, accumulate);
    FD_CUDA(cudaGetLastError());
}

__global__ void axpby_kernel(long long N, double a, const double *__restrict__ x, double b,
                             const double *__restrict__ y, double *out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        double r = a * x[i];
        if (y) r = __dadd_rn(r, __dmul_rn(b, y[i]));
        out[i] = r;
    }
}

void launch_axpby(long long N, double a, const double *x, double b, const double *y, double *out,
                  cudaStream_t s) {
    axpby_kernel<<<grid_for(N, 256), 256, 0, s>>>(N, a, x, b, y, out);
    FD_CUDA(cudaGetLastError());
}

// out = x / (*s)   (reference: V[k+1] = w / h_next, a true division)
__global__ void scale_kernel(long long N, const double *__restrict__ x, const double *__restrict__ sp,
                             double *out) {
    const double s = *sp;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = x[i] / s;
}

void launch_scale(long long N, const double *x, const double *s_dev, double *out, cudaStream_t s) {
    scale_kernel<<<grid_for(N, 256), 256, 0, s>>>(N, x, s_dev, out);
    FD_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// deterministic reductions
constexpr int kRedThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double block_sum(double v, double *sh) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (wid == 0) {
        r = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;   // valid in thread 0
}

// Combine per-block partials in a fixed order; the last block to arrive does it.
__device__ void finish(double part, RedWork w, double *out) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        w.partials[blockIdx.x] = part;
        __threadfence();
        const unsigned int done = atomicAdd(w.counter, 1u);
        last = (done == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
        __shared__ double sh[32];
        __threadfence();
        double v = 0.0;
        for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
            v += ((volatile double *)w.partials)[i];
        v = block_sum(v, sh);
        if (threadIdx.x == 0) {
            *out = v;
            *w.counter = 0u;
        }
    }
}

__global__ void __launch_bounds__(kRedThreads) dot_kernel(long long N, const double *__restrict__ x,
                                                          const double *__restrict__ y, RedWork w,
                                                          double *out) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x)
        acc = fma(x[i], y[i], acc);
    acc = block_sum(acc, sh);
    finish(acc, w, out);
}

void launch_dot(long long N, const double *x, const double *y, double *out, RedWork w,
                cudaStream_t s) {
    dot_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(N, x, y, w, out);
    FD_CUDA(cudaGetLastError());
}

// Fused modified-Gram-Schmidt step (krylov.py:107-109):
//   w -= h_prev * vprev        (the previous projection, if vprev)
//   h_out = vi . w             (the next projection; vi == null -> w . w)
__global__ void __launch_bounds__(kRedThreads) mgs_kernel(long long N, double *__restrict__ w,
                                                          const double *__restrict__ vprev,
                                                          const double *__restrict__ h_prev,
                                                          const double *__restrict__ vi, RedWork wk,
                                                          double *h_out) {
    __shared__ double sh[32];
    const double h = vprev ? *h_prev : 0.0;
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        double wv = w[i];
        if (vprev) {
            wv = __dsub_rn(wv, __dmul_rn(h, vprev[i]));
            w[i] = wv;
        }
        acc = fma(vi ? vi[i] : wv, wv, acc);
    }
    acc = block_sum(acc, sh);
    finish(acc, wk, h_out);
}

void launch_mgs(long long N, double *w, const double *vprev, const double *h_prev, const double *vi,
                double *h_out, RedWork wk, cudaStream_t s) {
    mgs_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(N, w, vprev, h_prev, vi, wk, h_out);
    FD_CUDA(cudaGetLastError());
}

// x += sum_t y_t V_t  (krylov.py:141)
__global__ void basis_update_kernel(long long N, int k, const double *__restrict__ V,
                                    const double *__restrict__ y, double *x) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int t = 0; t < k; ++t) s = fma(V[(long long)t * N + i], __ldg(y + t), s);
        x[i] = x[i] + s;
    }
}

void launch_basis_update(long long N, int k, const double *V, const double *y_dev, double *x,
                         cudaStream_t s) {
    basis_update_kernel<<<grid_for(N, 256), 256, 0, s>>>(N, k, V, y_dev, x);
    FD_CUDA(cudaGetLastError());
}

}  // namespace fd
