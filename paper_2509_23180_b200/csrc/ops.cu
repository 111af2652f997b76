// Element-wise and reduction kernels around the solve: the 5-point stencil
// (rectsolver.apply_rect_operator, rectsolver.py:264-289), interface coupling
// gather/scatter (ddm.CouplingMap.apply, ddm.py:44-51) and the Arnoldi
// building blocks of restarted GMRES (krylov.py:103-111,141).
//
// All HBM-bound: grids are multiples of the 148 SMs, loads are coalesced,
// reductions are deterministic (fixed grid, fixed combine order: per-block
// warp-shuffle trees, then the last block to finish combines the per-block
// partials in index order), so repeated runs give bitwise-equal results.
#include <algorithm>

#include "fd_internal.h"

namespace fd {

// out = A v with the reference's accumulation order; every product is rounded
// before it is added, exactly as numpy's `out[...] += d * G[...]`.
__global__ void stencil_kernel(int m, int n, double c0, double dx, double dy, double mw, double me,
                               double ms, double mn, const double *__restrict__ v,
                               double *__restrict__ out, int ppx, int ppy) {
    const long long total = (long long)m * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
        const double g = v[idx];
        double a = __dmul_rn(c0, g);
        if (j > 0) a = __dadd_rn(a, __dmul_rn(dy, v[idx - 1]));
        if (j < n - 1) a = __dadd_rn(a, __dmul_rn(dy, v[idx + 1]));
        if (ppy) {   // periodic y: wrap-around neighbours (rectsolver.py:274-276)
            if (j == 0) a = __dadd_rn(a, __dmul_rn(dy, v[idx + n - 1]));
            if (j == n - 1) a = __dadd_rn(a, __dmul_rn(dy, v[idx - (n - 1)]));
        } else {
            if (j == 0) a = __dadd_rn(a, __dmul_rn(ms, g));
            if (j == n - 1) a = __dadd_rn(a, __dmul_rn(mn, g));
        }
        if (i > 0) a = __dadd_rn(a, __dmul_rn(dx, v[idx - n]));
        if (i < m - 1) a = __dadd_rn(a, __dmul_rn(dx, v[idx + n]));
        if (ppx) {   // periodic x (rectsolver.py:283-285)
            if (i == 0) a = __dadd_rn(a, __dmul_rn(dx, v[idx + (long long)(m - 1) * n]));
            if (i == m - 1) a = __dadd_rn(a, __dmul_rn(dx, v[idx - (long long)(m - 1) * n]));
        } else {
            if (i == 0) a = __dadd_rn(a, __dmul_rn(mw, g));
            if (i == m - 1) a = __dadd_rn(a, __dmul_rn(me, g));
        }
        out[idx] = a;
    }
}

static int grid_for(long long N, int threads) {
    long long g = (N + threads - 1) / threads;
    const long long cap = 148LL * 16;
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

void launch_stencil(int m, int n, double delta_x, double delta_y, double kappa, double mw,
                    double me, double ms, double mn, const double *v, double *out, cudaStream_t s,
                    int ppx, int ppy) {
    const double c0 = -2.0 * (delta_x + delta_y) + kappa;   // rectsolver.py:270
    const long long N = (long long)m * n;
    stencil_kernel<<<grid_for(N, 256), 256, 0, s>>>(m, n, c0, delta_x, delta_y, mw, me, ms, mn, v,
                                                    out, ppx, ppy);
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

__global__ void mul_kernel(long long N, const double *__restrict__ x, const double *__restrict__ y, double *out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x)
        out[i] = x[i] * y[i];
}

void launch_mul(long long N, const double *x, const double *y, double *out, cudaStream_t s) {
    if (N <= 0) return;
    mul_kernel<<<(int)std::min<long long>((N + 255) / 256, 148LL * 16), 256, 0, s>>>(N, x, y, out);
    FD_CUDA(cudaGetLastError());
}

__global__ void zero_at_kernel(int len, const int64_t *__restrict__ to, double *dst) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < len; t += gridDim.x * blockDim.x) dst[to[t]] = 0.0;
}

void launch_zero_at(int len, const int64_t *to, double *dst, cudaStream_t s) {
    if (len <= 0) return;
    zero_at_kernel<<<(len + 255) / 256, 256, 0, s>>>(len, to, dst);
    FD_CUDA(cudaGetLastError());
}

__global__ void scatter_batch_kernel(const __grid_constant__ ScatterBatch b, int mode) {
    const int i = blockIdx.y, len = b.len[i];
    const int64_t *__restrict__ to = b.to[i];
    double *dst = b.dst[i];
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < len; t += gridDim.x * blockDim.x) {
        const int64_t d = to[t];
        if (mode == 2) {
            dst[d] = 0.0;
            continue;
        }
        const double v = __dmul_rn(b.c[i], b.src[i][b.from[i][t]]);
        if (mode == 0)
            dst[d] = v;
        else
            atomicAdd(dst + d, v);
    }
}

void launch_scatter_batch(const ScatterBatch &b, int mode, cudaStream_t s) {
    int mx = 0;
    for (int i = 0; i < b.count; ++i) mx = std::max(mx, b.len[i]);
    if (b.count <= 0 || mx <= 0) return;
    scatter_batch_kernel<<<dim3((mx + 255) / 256, b.count), 256, 0, s>>>(b, mode);
    FD_CUDA(cudaGetLastError());
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

namespace fd {

// ---------------------------------------------------------------------------
// Low-synchronisation MGS Arnoldi step (restates krylov.py:105-111).
//
// MGS computes h_i = V_i . (w - sum_{j<i} h_j V_j) one projection at a time,
// i.e. k+1 dependent passes over the basis.  In exact arithmetic
//   h_i = s_i - sum_{j<i} G_ij h_j,   s_i = V_i . w,  G_ij = V_i . V_j  (i > j),
// so one pass computes every s_i plus the new Gram row G_k. = V_k . V_{j<k},
// a (k+1)-step forward substitution (the last block, subtraction order j
// ascending as in MGS) gives h, and a second pass forms
//   w' = w - h_0 V_0 - h_1 V_1 - ... - h_k V_k  (same order)   and ||w'||^2.
// Bytes per centre point: 8(k+2) + 8(k+1) + 16 instead of 32(k+1) + 8.
//
// dots pass: each CTA stages a chunk of w and V_k in shared memory; warp q
// owns the basis vectors j = q, q + 16, ... and keeps their two running sums
// in registers across all chunks, so no per-chunk block reductions are needed.
constexpr int kArnThreads = 512;
constexpr int kArnWarps = kArnThreads / 32;
constexpr int kArnChunk = 2048;

__device__ __forceinline__ void arn_finish(ArnWork a, int nd, const double *bacc, int k, int ldg,
                                           bool want_h) {
    __shared__ bool last;
    __syncthreads();
    // [d][block]: the last block's reduction reads each d coalesced over blocks
    for (int d = threadIdx.x; d < nd; d += blockDim.x) a.partials[size_t(d) * gridDim.x + blockIdx.x] = bacc[d];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int done = atomicAdd(a.counter, 1u);
        last = (done == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    __shared__ double tot[2 * kMaxArnoldi + 2];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double *pp = a.partials;   // read past L1 (__ldcg): other blocks' writes
    for (int d = wid; d < nd; d += int(blockDim.x >> 5)) {   // fixed order: lanes stride blocks, then a tree
        double v = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) v += __ldcg(pp + size_t(d) * gridDim.x + b);
        v = warp_sum(v);
        if (lane == 0) tot[d] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) *a.counter = 0u;
    if (!want_h) {
        if (threadIdx.x < nd) a.out[threadIdx.x] = tot[threadIdx.x];
        return;
    }
    // tot = [s_0..s_k | c_0..c_{k-1} | w.w]; Gram row k <- c; h by forward substitution
    if (wid == 0) {
        constexpr int RL = kMaxArnoldi / 32;   // rows per lane: i = lane + 32 r
        double *G = a.G;
        for (int j = lane; j < k; j += 32) G[size_t(k) * ldg + j] = tot[k + 1 + j];
        __syncwarp();
        double h[RL];
#pragma unroll
        for (int r = 0; r < RL; ++r) h[r] = lane + 32 * r <= k ? tot[lane + 32 * r] : 0.0;
        const int rows = k / 32 + 1;   // rows r in use (warp-uniform)
        auto hj_of = [&](int jj) {
            double v = h[0];
#pragma unroll
            for (int r = 1; r < RL; ++r)
                if ((jj >> 5) == r) v = h[r];
            return __shfl_sync(0xffffffffu, v, jj & 31);
        };
        int j = 0;
        // the Gram entries of 8 steps loaded ahead of their dependent chain (an
        // L2 round trip per step otherwise sits on this serial tail)
        for (; j + 8 <= k; j += 8) {
            double g[RL][8];
#pragma unroll
            for (int r = 0; r < RL; ++r) {
                const int i = lane + 32 * r;
#pragma unroll
                for (int q = 0; q < 8; ++q) g[r][q] = (r < rows && i > j + q && i <= k) ? G[size_t(i) * ldg + j + q] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int jj = j + q;
                const double hj = hj_of(jj);
#pragma unroll
                for (int r = 0; r < RL; ++r) {
                    const int i = lane + 32 * r;
                    if (i > jj && i <= k) h[r] = __dsub_rn(h[r], __dmul_rn(g[r][q], hj));
                }
            }
        }
        for (; j < k; ++j) {
            const double hj = hj_of(j);
#pragma unroll
            for (int r = 0; r < RL; ++r) {
                const int i = lane + 32 * r;
                if (i > j && i <= k) h[r] = __dsub_rn(h[r], __dmul_rn(G[size_t(i) * ldg + j], hj));
            }
        }
#pragma unroll
        for (int r = 0; r < RL; ++r)
            if (lane + 32 * r <= k) a.out[lane + 32 * r] = h[r];
        if (lane == 0) a.out[k + 1] = tot[2 * k + 1];   // ||w||^2 before orthogonalisation
    }
}

// JPW basis vectors per warp: 4 covers k + 1 <= 64 (the m = 50 configs), 8
// covers k + 1 <= 128 (the reference's default m = 80)
template <int JPW>
__global__ void __launch_bounds__(kArnThreads) arnoldi_dots_kernel(long long N, int k, const double *__restrict__ V,
                                                                    const double *__restrict__ w, ArnWork a, int ldg,
                                                                    int chunk) {
    __shared__ double sw[kArnChunk], sv[kArnChunk];
    __shared__ double bacc[2 * kMaxArnoldi + 2];
    __shared__ double wred[kArnWarps];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nd = 2 * k + 2;
    const double *vk = V + (long long)k * N;
    double as[JPW], ac[JPW];
#pragma unroll
    for (int q = 0; q < JPW; ++q) as[q] = ac[q] = 0.0;
    double ww = 0.0;
    for (long long c0 = (long long)blockIdx.x * chunk; c0 < N; c0 += (long long)gridDim.x * chunk) {
        const int len = (int)min((long long)chunk, N - c0);
        __syncthreads();
        for (int t = threadIdx.x; t < len; t += kArnThreads) {
            const double wv = w[c0 + t];
            sw[t] = wv;
            sv[t] = vk[c0 + t];
            ww = fma(wv, wv, ww);
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < JPW; ++q) {
            const int j = wid + q * kArnWarps;
            if (j > k) break;
            const double *vj = V + (long long)j * N + c0;
            double s = as[q], c = ac[q];
            const bool gram = j < k;
            int t = lane;
#pragma unroll 4
            for (; t + 96 < len; t += 128) {
                const double x0 = vj[t], x1 = vj[t + 32], x2 = vj[t + 64], x3 = vj[t + 96];
                s = fma(x0, sw[t], s);
                s = fma(x1, sw[t + 32], s);
                s = fma(x2, sw[t + 64], s);
                s = fma(x3, sw[t + 96], s);
                if (gram) {
                    c = fma(x0, sv[t], c);
                    c = fma(x1, sv[t + 32], c);
                    c = fma(x2, sv[t + 64], c);
                    c = fma(x3, sv[t + 96], c);
                }
            }
            for (; t < len; t += 32) {
                const double x = vj[t];
                s = fma(x, sw[t], s);
                if (gram) c = fma(x, sv[t], c);
            }
            as[q] = s;
            ac[q] = c;
        }
    }
#pragma unroll
    for (int q = 0; q < JPW; ++q) {
        const int j = wid + q * kArnWarps;
        const double s = warp_sum(as[q]), c = warp_sum(ac[q]);
        if (lane == 0 && j <= k) {
            bacc[j] = s;
            if (j < k) bacc[k + 1 + j] = c;
        }
    }
    ww = warp_sum(ww);
    if (lane == 0) wred[wid] = ww;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < kArnWarps; ++q) t += wred[q];
        bacc[2 * k + 1] = t;
    }
    arn_finish(a, nd, bacc, k, ldg, true);
}

// w <- w - h_0 V_0 - ... - h_k V_k (MGS subtraction order); out[0] = ||w||^2
__global__ void __launch_bounds__(256) arnoldi_update_kernel(long long N, int k, const double *__restrict__ V,
                                                             double *__restrict__ w, const double *__restrict__ h,
                                                             ArnWork a) {
    __shared__ double sh[kMaxArnoldi + 1];
    __shared__ double bacc[1];
    __shared__ double red[32];
    for (int j = threadIdx.x; j <= k; j += blockDim.x) sh[j] = h[j];
    __syncthreads();
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        double x = w[i];
        int j = 0;
        for (; j + 7 <= k; j += 8) {   // 8 basis loads in flight per thread
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = V[(long long)(j + q) * N + i];
#pragma unroll
            for (int q = 0; q < 8; ++q) x = __dsub_rn(x, __dmul_rn(sh[j + q], v[q]));
        }
        for (; j + 3 <= k; j += 4) {
            const double v0 = V[(long long)j * N + i], v1 = V[(long long)(j + 1) * N + i];
            const double v2 = V[(long long)(j + 2) * N + i], v3 = V[(long long)(j + 3) * N + i];
            x = __dsub_rn(x, __dmul_rn(sh[j], v0));
            x = __dsub_rn(x, __dmul_rn(sh[j + 1], v1));
            x = __dsub_rn(x, __dmul_rn(sh[j + 2], v2));
            x = __dsub_rn(x, __dmul_rn(sh[j + 3], v3));
        }
        for (; j <= k; ++j) x = __dsub_rn(x, __dmul_rn(sh[j], V[(long long)j * N + i]));
        w[i] = x;
        acc = fma(x, x, acc);
    }
    acc = block_sum(acc, red);
    if (threadIdx.x == 0) bacc[0] = acc;
    arn_finish(a, 1, bacc, k, 0, false);
}

// out = x / sqrt(*nrm2)  (reference: V[k+1] = w / h[k+1, k], h = ||w||)
__global__ void scale_sqrt_kernel(long long N, const double *__restrict__ x, const double *__restrict__ nrm2,
                                  double *out) {
    const double s = sqrt(*nrm2);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = x[i] / s;
}

// points per staged chunk: the full 2048 for large vectors, smaller for small
// ones so that at least ~2 CTAs per SM take part (c0: N_c = 19881)
static int arn_chunk(long long N) {
    long long c = N / (148 * 2);
    c = std::max<long long>(256, std::min<long long>(kArnChunk, (c + 31) / 32 * 32));
    return (int)c;
}
static int arn_grid(long long N) {
    const long long ch = arn_chunk(N);
    long long g = (N + ch - 1) / ch;
    return (int)std::min<long long>(std::max<long long>(g, 1), 148LL * 4);
}

void launch_arnoldi_dots(long long N, int k, const double *V, const double *w, ArnWork a, int ldg,
                         cudaStream_t s) {
    if (k + 1 > kMaxArnoldi) throw Error{FD_ERR_VALIDATION, "arnoldi: more basis vectors than kMaxArnoldi"};
    if (k + 1 <= 4 * kArnWarps)
        arnoldi_dots_kernel<4><<<arn_grid(N), kArnThreads, 0, s>>>(N, k, V, w, a, ldg, arn_chunk(N));
    else
        arnoldi_dots_kernel<kMaxArnoldi / kArnWarps><<<arn_grid(N), kArnThreads, 0, s>>>(N, k, V, w, a, ldg,
                                                                                        arn_chunk(N));
    FD_CUDA(cudaGetLastError());
}

void launch_arnoldi_update(long long N, int k, const double *V, double *w, const double *h, ArnWork a,
                           cudaStream_t s) {
    arnoldi_update_kernel<<<grid_for(N, 256), 256, 0, s>>>(N, k, V, w, h, a);
    FD_CUDA(cudaGetLastError());
}

void launch_scale_sqrt(long long N, const double *x, const double *nrm2, double *out, cudaStream_t s) {
    scale_sqrt_kernel<<<grid_for(N, 256), 256, 0, s>>>(N, x, nrm2, out);
    FD_CUDA(cudaGetLastError());
}

}  // namespace fd

namespace fd {

// out (C x R) = alpha * in^T + beta * other, in (R x C) row-major.  32 x 32
// tiles through padded shared memory: coalesced reads and writes, HBM-bound.
// Used for the transposed transform axis (reference transform_axis == "x",
// rectsolver.py:198-199,211-212): fields go to the plan's internal layout and
// back; the epilogue folds the back-substitution's p_i = q_i - A_i^{-1}(...).
__global__ void __launch_bounds__(256) transpose_kernel(int R, int C, const double *__restrict__ in,
                                                        double *out, double alpha, double beta,
                                                        const double *other) {
    __shared__ double tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    const long long r0 = (long long)blockIdx.y * 32, c0 = (long long)blockIdx.x * 32;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const long long r = r0 + ty + 8 * q, c = c0 + tx;
        if (r < R && c < C) tile[ty + 8 * q][tx] = in[r * C + c];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const long long c = c0 + ty + 8 * q, r = r0 + tx;
        if (r < R && c < C) {
            double v = alpha * tile[tx][ty + 8 * q];
            if (other) v = __dadd_rn(v, __dmul_rn(beta, other[c * R + r]));
            out[c * R + r] = v;
        }
    }
}

void launch_transpose(int R, int C, const double *in, double *out, double alpha, double beta,
                      const double *other, cudaStream_t s) {
    if (R <= 0 || C <= 0) return;
    dim3 grid((C + 31) / 32, (R + 31) / 32);
    transpose_kernel<<<grid, 256, 0, s>>>(R, C, in, out, alpha, beta, other);
    FD_CUDA(cudaGetLastError());
}

}  // namespace fd

namespace fd {

// ---------------------------------------------------------------------------
// Device-side problem assembly: the manufactured right-hand
// side f = lap p + kappa p at the cell-centred nodes of one rectangle, each
// Dirichlet edge lifted with p at its ghost points (rectsolver.lift_dirichlet,
// rectsolver.py:292-313: rhs -= factor * delta * g on the adjacent line, in
// edge order west, east, south, north), and optionally p itself.  Solutions:
// 0 = sin(pi x) sin(pi y) + e^(x+y)/e^2, 1 = sin(pi x) sin(pi y).
__device__ __forceinline__ double mf_p(int sol, double x, double y) {
    const double s = sin(M_PI * x) * sin(M_PI * y);
    return sol == 0 ? s + exp(x + y) / (M_E * M_E) : s;
}
__device__ __forceinline__ double mf_lap(int sol, double x, double y) {
    const double s = -2.0 * (M_PI * M_PI) * sin(M_PI * x) * sin(M_PI * y);
    return sol == 0 ? s + 2.0 * exp(x + y) / (M_E * M_E) : s;
}

__global__ void assemble_kernel(int m, int n, double x0, double y0, double dx, double dy, double kappa,
                                int sol, double lw, double le, double ls, double ln, double delta_x,
                                double delta_y, double *__restrict__ f, double *__restrict__ exact) {
    const long long total = (long long)m * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
        const double x = x0 + (double(i + 1) - 0.5) * dx, y = y0 + (double(j + 1) - 0.5) * dy;
        const double p = mf_p(sol, x, y);
        double v = mf_lap(sol, x, y) + kappa * p;
        if (lw != 0.0 && i == 0) v = v - lw * delta_x * mf_p(sol, x - dx, y);
        if (le != 0.0 && i == m - 1) v = v - le * delta_x * mf_p(sol, x + dx, y);
        if (ls != 0.0 && j == 0) v = v - ls * delta_y * mf_p(sol, x, y - dy);
        if (ln != 0.0 && j == n - 1) v = v - ln * delta_y * mf_p(sol, x, y + dy);
        f[idx] = v;
        if (exact) exact[idx] = p;
    }
}

void launch_assemble(int m, int n, double x0, double y0, double dx, double dy, double kappa, int sol,
                     const double lift[4], double *f, double *exact, cudaStream_t s) {
    const long long N = (long long)m * n;
    assemble_kernel<<<grid_for(N, 256), 256, 0, s>>>(m, n, x0, y0, dx, dy, kappa, sol, lift[0], lift[1], lift[2],
                                                     lift[3], 1.0 / (dx * dx), 1.0 / (dy * dy), f, exact);
    FD_CUDA(cudaGetLastError());
}

}  // namespace fd
