// Fused subdomain fast solve A^{-1} f on B200 (sm_100a), fp64 CUDA cores.
//
// Reference pipeline (fftddm/rectsolver.py:183-213): fhat = Q^T f along y
// (DST-I, transforms.py:74-80,112-113), per-mode tridiagonal solve along x
// (rectsolver.py:80-91), p = Q phat.
//
// B200 design: two streaming passes over the field plus a tiny carry pass.
//   pass 1 (row blocks of R rows, one CTA each): DST-I of every row (two rows
//          packed into one complex FFT of length L = 2(n+1), Stockham radix-16
//          in shared memory), then the *local* forward elimination of the
//          block (zero carry-in), written back as yhat; per mode the block-end
//          value yhat_e and the block-start value of the local backward sweep
//          F_s = sum_i yhat_i * pi_i / beta_i are kept for the carries.
//   carry   per mode, sequential over blocks: true y at block ends
//          Y_b = yhat_e + P_e Y_{b-1} and true x at block starts
//          X_b = F_s + Y_{b-1} xi_s + Q X_{b+1}  (tables from plan.cpp).
//   pass 2 (row blocks, rows descending): y_i = yhat_i + P_i Y_{b-1}, the
//          reference back-substitution x_i = (y_i - delta x_{i+1}) / beta_i
//          with x_{e+1} = X_{b+1}, then the inverse DST-I (same transform) and
//          an optional epilogue out = alpha x + beta other.
// HBM traffic: 8 B/pt read + 8 B/pt write per pass = the 32 B/pt algorithmic
// minimum of a separable transform solve; the yhat intermediate lives in the
// caller's output buffer, so the solve is in-place capable and needs no
// field-sized scratch.  The forward/backward recurrences run in the
// reference's row order; only the block carries are re-associated (measured
// <= 4e-14 relative to the sequential Thomas at m = 16383).

#include <math.h>
#include <stdio.h>

#include <mutex>
#include <set>

#include "fd_internal.h"
#include "dst_device.cuh"

namespace fd {

// Forward-transform `rows` rows starting at `in` (global) into rowbuf (shared).
template <class P>
struct FwdT;
template <class P>
struct InvT;

template <int LG>
struct FwdT<FftDst<LG>> {
    __device__ static void run(const double *in, int rows, int n, double *rowbuf, double2 *smem,
                               const PlanDev &p) {
        using F = FftDst<LG>;
        const int pr = threadIdx.x / F::T, t = threadIdx.x % F::T;
        const int ra = 2 * pr, rb = 2 * pr + 1;
        GRow A{ra < rows ? in + size_t(ra) * n : nullptr};
        GRow B{rb < rows ? in + size_t(rb) * n : nullptr};
        double2 *buf = smem + pr * F::PADL;
        F::first_pass(buf, A, B, t);
        F::template mids<F::NMID, 16>(buf, TwGlobal{p.tw}, t);
        SmemRow oa{ra < rows ? rowbuf + ra * n : nullptr};
        SmemRow ob{rb < rows ? rowbuf + rb * n : nullptr};
        F::last_pass(buf, TwGlobal{p.tw}, t, oa, ob, p.scale);
        __syncthreads();
    }
};

template <int LG>
struct InvT<FftDst<LG>> {
    // rowbuf rows -> global rows out (row stride n) with epilogue
    __device__ static void run(const double *rowbuf, int rows, int n, double *out, const double *other,
                               double alpha, double beta, double2 *smem, const PlanDev &p) {
        using F = FftDst<LG>;
        const int pr = threadIdx.x / F::T, t = threadIdx.x % F::T;
        const int ra = 2 * pr, rb = 2 * pr + 1;
        SRow A{ra < rows ? rowbuf + ra * n : nullptr};
        SRow B{rb < rows ? rowbuf + rb * n : nullptr};
        double2 *buf = smem + pr * F::PADL;
        F::first_pass(buf, A, B, t);
        F::template mids<F::NMID, 16>(buf, TwGlobal{p.tw}, t);
        OutRow oa{ra < rows ? out + size_t(ra) * n : nullptr,
                  other ? other + size_t(ra) * n : nullptr, alpha, beta};
        OutRow ob{rb < rows ? out + size_t(rb) * n : nullptr,
                  other ? other + size_t(rb) * n : nullptr, alpha, beta};
        F::last_pass(buf, TwGlobal{p.tw}, t, oa, ob, p.scale);
        __syncthreads();
    }
};

// Dense transform of the G-row group in rowbuf (shared) into acc (registers):
// acc[g][o] = sum_i T(q_io) x_g[i], T a periodic table, q_io = idx0(o) + i step(o)
// (mod the period).  DD (both directions): T = sin(pi q/(n+1)), q = (i+1)(o+1).
// NN forward (Q^T, transforms.py:83-90,129-134): T = cos(pi q/2n), q = o(2i+1);
// NN inverse (Q, transforms.py:92-98,106-109): q = i(2o+1), input 0 scaled by
// 1/sqrt(2) (the basis' sqrt(1/n) vs sqrt(2/n)).  PP (real Fourier basis,
// transforms.py:114-126,139-148): T = cos(2 pi q/n) for basis index <= n/2,
// sin(2 pi q/n) above (table halves), q = o i mod n; basis 0 and n/2 carry
// sqrt(1/n) (a 1/sqrt(2) on the output forward, on the input inverse).
template <int M, int NT_, int S_>
__device__ __forceinline__ void dense_rows(const double *rowbuf, int n, const double *tab,
                                           double (&acc)[DenseDstT<M, NT_, S_>::G][M], int pair, bool inverse) {
    using D = DenseDstT<M, NT_, S_>;
    constexpr int G = D::G, S = D::S, NM = D::NMODE;
    const bool nn = pair == kPairNN, pp = pair == kPairPP;
    const int period = nn ? 4 * n : pp ? n : 2 * (n + 1);
    const int half = n >> 1;
    const int q = threadIdx.x % S;                     // this thread's share of the input sum
    const int chunk = (n + S - 1) / S, jb = min(n, q * chunk), je = min(n, jb + chunk);
    int idx[M], step[M], toff[M];
#pragma unroll
    for (int u = 0; u < M; ++u) {
        const int o = threadIdx.x / S + u * NM;
        toff[u] = 0;
        long long i0;
        if (pp) {
            i0 = (long long)o * jb;            // o i mod n
            step[u] = o;
            if (!inverse && o > half) toff[u] = n;   // sine half of the table
        } else if (!nn) {
            i0 = (long long)(jb + 1) * (o + 1);  // (i + 1)(o + 1)
            step[u] = o + 1;
        } else if (!inverse) {
            i0 = (long long)o * (2 * jb + 1);  // o (2i + 1)
            step[u] = 2 * o;
        } else {
            i0 = (long long)jb * (2 * o + 1);  // i (2o + 1)
            step[u] = 2 * o + 1;
        }
        idx[u] = int(i0 % period);
        if (step[u] >= period) step[u] -= period;
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g][u] = 0.0;
    }
#pragma unroll 2
    for (int j = jb; j < je; ++j) {
        double x[G];
        const double xs = ((nn || pp) && inverse && (j == 0 || (pp && j == half))) ? 0.70710678118654752440 : 1.0;
        const int joff = (pp && inverse && j > half) ? n : 0;   // inverse: the input's basis picks the half
#pragma unroll
        for (int g = 0; g < G; ++g) x[g] = rowbuf[g * n + j] * xs;
#pragma unroll
        for (int u = 0; u < M; ++u) {
            const int o = threadIdx.x / S + u * NM;
            if (o < n) {
                const double sv = tab[idx[u] + toff[u] + joff];
#pragma unroll
                for (int g = 0; g < G; ++g) acc[g][u] = fma(sv, x[g], acc[g][u]);
                idx[u] += step[u];
                if (idx[u] >= period) idx[u] -= period;
            }
        }
    }
    if constexpr (S > 1) {   // combine the S partial sums (adjacent lanes)
#pragma unroll
        for (int off = 1; off < S; off <<= 1)
#pragma unroll
            for (int u = 0; u < M; ++u)
#pragma unroll
                for (int g = 0; g < G; ++g) acc[g][u] += __shfl_xor_sync(0xffffffffu, acc[g][u], off);
    }
    if ((nn || pp) && !inverse) {   // output 0 (and n/2 for PP) carries sqrt(1/n) instead of sqrt(2/n)
#pragma unroll
        for (int u = 0; u < M; ++u) {
            const int o = threadIdx.x / S + u * NM;
            if (o == 0 || (pp && o == half))
#pragma unroll
                for (int g = 0; g < G; ++g) acc[g][u] *= 0.70710678118654752440;
        }
    }
}

template <int M, int NT_, int S_>
__device__ __forceinline__ double *dense_tab(double2 *smem) {
    return reinterpret_cast<double *>(smem) + DenseDstT<M, NT_, S_>::G * DenseDstT<M, NT_, S_>::NMAX;
}

template <int M, int NT_, int S_>
__device__ __forceinline__ void stage_tab(double *tab, int n, const PlanDev &p) {
    const int period = p.tpair == kPairNN ? 4 * n : p.tpair == kPairPP ? 2 * n : 2 * (n + 1);
    for (int q = threadIdx.x; q < period; q += DenseDstT<M, NT_, S_>::NT) tab[q] = __ldg(p.dense + q);
}

template <int M, int NT_, int S_>
struct FwdT<DenseDstT<M, NT_, S_>> {
    __device__ static void run(const double *in, int rows, int n, double *rowbuf, double2 *smem,
                               const PlanDev &p) {
        constexpr int NT = DenseDstT<M, NT_, S_>::NT, G = DenseDstT<M, NT_, S_>::G;
        double *tab = dense_tab<M, NT_, S_>(smem);
        stage_tab<M, NT_, S_>(tab, n, p);
#pragma unroll 8
        for (int idx = threadIdx.x; idx < G * n; idx += NT)
            rowbuf[idx] = idx < rows * n ? __ldg(in + idx) : 0.0;
        __syncthreads();
        double acc[G][M];
        dense_rows<M, NT_, S_>(rowbuf, n, tab, acc, p.tpair, false);
        __syncthreads();
        constexpr int S = DenseDstT<M, NT_, S_>::S, NM = DenseDstT<M, NT_, S_>::NMODE;
#pragma unroll
        for (int u = 0; u < M; ++u) {
            const int k = threadIdx.x / S + u * NM;
            if (k < n && threadIdx.x % S == 0)
#pragma unroll
                for (int g = 0; g < G; ++g)
                    if (g < rows) rowbuf[g * n + k] = p.scale * acc[g][u];
        }
        __syncthreads();
    }
};

template <int M, int NT_, int S_>
struct InvT<DenseDstT<M, NT_, S_>> {
    __device__ static void run(double *rowbuf, int rows, int n, double *out, const double *other,
                               double alpha, double beta, double2 *smem, const PlanDev &p) {
        constexpr int NT = DenseDstT<M, NT_, S_>::NT, G = DenseDstT<M, NT_, S_>::G;
        double *tab = dense_tab<M, NT_, S_>(smem);
        stage_tab<M, NT_, S_>(tab, n, p);
        for (int idx = rows * n + threadIdx.x; idx < G * n; idx += NT) rowbuf[idx] = 0.0;
        __syncthreads();
        double acc[G][M];
        dense_rows<M, NT_, S_>(rowbuf, n, tab, acc, p.tpair, true);
        constexpr int S = DenseDstT<M, NT_, S_>::S, NM = DenseDstT<M, NT_, S_>::NMODE;
#pragma unroll
        for (int u = 0; u < M; ++u) {
            const int k = threadIdx.x / S + u * NM;
            if (k < n && threadIdx.x % S == 0)
#pragma unroll
                for (int g = 0; g < G; ++g)
                    if (g < rows) {
                        OutRow o{out + size_t(g) * n, other ? other + size_t(g) * n : nullptr, alpha,
                                 beta};
                        o.put(k, p.scale * acc[g][u]);
                    }
        }
        __syncthreads();
    }
};

template <class P>
struct Cfg;
template <int LG>
struct Cfg<FftDst<LG>> {
    static constexpr int MPT = ((1 << (LG - 1)) - 1 + FftDst<LG>::NT - 1) / FftDst<LG>::NT;
};
template <int M, int NT_, int S_>
struct Cfg<DenseDstT<M, NT_, S_>> {
    static constexpr int MPT = M;
};

// ---------------------------------------------------------------------------
// pass 1: DST rows + local forward elimination per block
template <class P>
__global__ void __launch_bounds__(P::NT, P::MINB) pass1_kernel(const __grid_constant__ JobList jl) {
    extern __shared__ __align__(16) double2 smem[];
    constexpr int MPT = Cfg<P>::MPT;
    const int job = find_job(jl, blockIdx.x);
    const SolveJob &J = jl.job[job];
    const PlanDev &p = J.p;
    const int b = blockIdx.x - jl.block_start[job];
    const int n = p.n, m = p.m;
    const int s = b * p.R, e = min(m, s + p.R) - 1;
    double *rowbuf = reinterpret_cast<double *>(smem);
    double yh[MPT], pi[MPT], fs[MPT];
#pragma unroll
    for (int u = 0; u < MPT; ++u) yh[u] = pi[u] = fs[u] = 0.0;

#pragma unroll 1
    for (int g0 = s; g0 <= e; g0 += P::G) {
        const int rows = min(P::G, e - g0 + 1);
        FwdT<P>::run(J.in + size_t(g0) * n, rows, n, rowbuf, smem, p);
#pragma unroll
        for (int u = 0; u < MPT; ++u) {
            const int k = threadIdx.x + u * P::NT;
            if (k >= n) continue;
            ModeView mv;
            mv.load(p, k);
            const int si = p.nsing ? __ldg(p.sidx + k) : -1;
            double y = yh[u], w = pi[u], f = fs[u];
            double lv[P::G], ibv[P::G];   // the group's factors, loaded ahead of the chain
#pragma unroll
            for (int rr = 0; rr < P::G; ++rr) {
                const int i = g0 + rr;
                const bool ex = rr < rows && i < mv.len;
                const double *er = p.ex + 4 * size_t(mv.off + i);
                lv[rr] = ex ? __ldg(er) : mv.l_inf;
                ibv[rr] = (i == m - 1) ? mv.ib_last : (ex ? __ldg(er + 1) : mv.ib_inf);
            }
#pragma unroll
            for (int rr = 0; rr < P::G; ++rr) {
                if (rr >= rows) break;
                const int i = g0 + rr;
                const double r = rowbuf[rr * n + k];
                if (si >= 0) p.sf[size_t(si) * m + i] = r;   // fhat column of a pinned mode
                if (i == s) {
                    y = r;
                    w = 1.0;
                } else {
                    const double l = lv[rr];
                    y = __dsub_rn(r, __dmul_rn(l, y));   // rectsolver.py:86
                    w = -l * w;
                }
                const double ib = ibv[rr];
                f = fma(y, w * ib, f);
                J.out[size_t(i) * n + k] = y;
            }
            yh[u] = y;
            pi[u] = w;
            fs[u] = f;
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < MPT; ++u) {
        const int k = threadIdx.x + u * P::NT;
        if (k < n) {
            p.ye[size_t(b) * n + k] = yh[u];
            p.fs[size_t(b) * n + k] = fs[u];
        }
    }
}

// ---------------------------------------------------------------------------
// carries: one thread per mode, chunks of blocks staged through shared memory
constexpr int kCarryModes = 32;
constexpr int kCarryChunk = 40;
constexpr int kCarryThreads = 256;

// Jobs of at most kCarryFast blocks (the small dense problems, where this kernel
// is a visible part of a GMRES iteration): all five block scalars of the chain
// are fetched at once into dynamic shared memory, one thread per mode walks
// the chain forward and back, and Y, X are stored -- one memory round trip
// instead of one per pass and chunk.
constexpr int kCarryFast = 96;
constexpr size_t kCarrySmem = size_t(5) * kCarryFast * kCarryModes * sizeof(double);

__global__ void __launch_bounds__(kCarryThreads) carry_kernel(const __grid_constant__ JobList jl) {
    // one dynamic buffer: [5][nb][kCarryModes] on the fast path, four chunk
    // arrays on the chunked path (no static arrays on top: a kernel whose
    // shared-memory footprint differs a lot from its neighbours' makes the SM
    // re-partition L1 / shared memory at every switch)
    extern __shared__ __align__(16) double dyn[];
    typedef double (*ChunkArr)[kCarryModes];
    ChunkArr sa = reinterpret_cast<ChunkArr>(dyn);
    ChunkArr sb = sa + kCarryChunk, sc = sb + kCarryChunk, sd = sc + kCarryChunk;
    const int job = find_job(jl, blockIdx.x);
    const PlanDev &p = jl.job[job].p;
    const int k0 = (blockIdx.x - jl.block_start[job]) * kCarryModes;
    const int n = p.n, nb = p.nb;
    const int lane = threadIdx.x % kCarryModes, slot = threadIdx.x / kCarryModes;
    constexpr int SLOTS = kCarryThreads / kCarryModes;
    const int k = k0 + lane;
    const bool ok = k < n;
    const double *Pe = p.blk;  // [nb][3][n]
    if (nb <= kCarryFast) {
        double *ye = dyn, *pe = ye + nb * kCarryModes, *fs = pe + nb * kCarryModes, *xi = fs + nb * kCarryModes,
               *qq = xi + nb * kCarryModes;
        for (int b = slot; b < nb; b += SLOTS) {
            const int o = b * kCarryModes + lane;
            ye[o] = ok ? p.ye[size_t(b) * n + k] : 0.0;
            fs[o] = ok ? p.fs[size_t(b) * n + k] : 0.0;
            pe[o] = ok ? __ldg(Pe + (size_t(b) * 3 + 0) * n + k) : 0.0;
            xi[o] = ok ? __ldg(Pe + (size_t(b) * 3 + 1) * n + k) : 0.0;
            qq[o] = ok ? __ldg(Pe + (size_t(b) * 3 + 2) * n + k) : 0.0;
        }
        __syncthreads();
        if (slot == 0) {
            double y = 0.0;
#pragma unroll 4
            for (int b = 0; b < nb; ++b) {   // Y_b = ye_b + Pe_b Y_{b-1}
                const int o = b * kCarryModes + lane;
                double v = ye[o];
                if (b > 0) v = fma(pe[o], y, v);
                ye[o] = v;
                y = v;
            }
            double x = 0.0;
#pragma unroll 4
            for (int b = nb - 1; b >= 0; --b) {   // X_b = fs_b + Y_{b-1} xi_b + Q_b X_{b+1}
                const int o = b * kCarryModes + lane;
                double v = fs[o];
                if (b > 0) v = fma(ye[o - kCarryModes], xi[o], v);
                if (b < nb - 1) v = fma(qq[o], x, v);
                fs[o] = v;
                x = v;
            }
        }
        __syncthreads();
        if (ok)
            for (int b = slot; b < nb; b += SLOTS) {
                const int o = b * kCarryModes + lane;
                p.ye[size_t(b) * n + k] = ye[o];
                p.fs[size_t(b) * n + k] = fs[o];
            }
        return;
    }
    // forward: Y_b = ye_b + Pe_b Y_{b-1}
    double yprev = 0.0;
#pragma unroll 1
    for (int c0 = 0; c0 < nb; c0 += kCarryChunk) {
        const int cn = min(kCarryChunk, nb - c0);
        for (int bb = slot; bb < cn; bb += SLOTS) {
            const int b = c0 + bb;
            sa[bb][lane] = ok ? p.ye[size_t(b) * n + k] : 0.0;
            sb[bb][lane] = ok ? __ldg(Pe + (size_t(b) * 3 + 0) * n + k) : 0.0;
        }
        __syncthreads();
        if (slot == 0) {
            for (int bb = 0; bb < cn; ++bb) {
                const int b = c0 + bb;
                double y = sa[bb][lane];
                if (b > 0) y = fma(sb[bb][lane], yprev, y);
                sa[bb][lane] = y;
                yprev = y;
            }
        }
        __syncthreads();
        for (int bb = slot; bb < cn; bb += SLOTS)
            if (ok) p.ye[size_t(c0 + bb) * n + k] = sa[bb][lane];
        __syncthreads();
    }
    // backward: X_b = fs_b + Y_{b-1} xi_b + Q_b X_{b+1}
    double xnext = 0.0;
#pragma unroll 1
    for (int c1 = nb; c1 > 0; c1 -= kCarryChunk) {
        const int c0 = max(0, c1 - kCarryChunk);
        const int cn = c1 - c0;
        for (int bb = slot; bb < cn; bb += SLOTS) {
            const int b = c0 + bb;
            sa[bb][lane] = ok ? p.fs[size_t(b) * n + k] : 0.0;
            sb[bb][lane] = ok ? __ldg(Pe + (size_t(b) * 3 + 1) * n + k) : 0.0;
            sc[bb][lane] = ok ? __ldg(Pe + (size_t(b) * 3 + 2) * n + k) : 0.0;
            sd[bb][lane] = (ok && b > 0) ? p.ye[size_t(b - 1) * n + k] : 0.0;
        }
        __syncthreads();
        if (slot == 0) {
            for (int bb = cn - 1; bb >= 0; --bb) {
                const int b = c0 + bb;
                double x = sa[bb][lane];
                if (b > 0) x = fma(sd[bb][lane], sb[bb][lane], x);
                if (b < nb - 1) x = fma(sc[bb][lane], xnext, x);
                sa[bb][lane] = x;
                xnext = x;
            }
        }
        __syncthreads();
        for (int bb = slot; bb < cn; bb += SLOTS)
            if (ok) p.fs[size_t(c0 + bb) * n + k] = sa[bb][lane];
        __syncthreads();
    }
}

// dynamic shared memory of the carry kernel's fast path (0: chunked path only)
static size_t carry_smem(const JobList &jc) {
    {   // once per device
        static std::mutex mu;
        static std::set<int> done;
        int dev = 0;
        FD_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> g(mu);
        if (done.insert(dev).second)
            FD_CUDA(cudaFuncSetAttribute((const void *)carry_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kCarrySmem));
    }
    int nbmax = 0;
    bool chunked = false;
    for (int j = 0; j < jc.count; ++j) {
        if (jc.job[j].p.nb <= kCarryFast) nbmax = std::max(nbmax, jc.job[j].p.nb);
        else chunked = true;
    }
    const size_t fast = size_t(5) * nbmax * kCarryModes * sizeof(double);
    const size_t chunk = chunked ? size_t(4) * kCarryChunk * kCarryModes * sizeof(double) : 0;
    return std::max(fast, chunk);
}

// ---------------------------------------------------------------------------
// pinned (singular) modes: sph = M_k^+ fhat_k, pinv stored transposed [j][i]
__global__ void __launch_bounds__(256) pinv_kernel(int m, int nsing, const double *pinvT,
                                                   const double *sf, double *sph) {
    const int i = blockIdx.x * 256 + threadIdx.x, si = blockIdx.y;
    if (i >= m) return;
    const double *P = pinvT + size_t(si) * m * m;
    const double *f = sf + size_t(si) * m;
    double acc = 0.0;
    for (int j = 0; j < m; ++j) acc = fma(__ldg(P + size_t(j) * m + i), f[j], acc);
    sph[size_t(si) * m + i] = acc;
}

// ---------------------------------------------------------------------------
// pass 2: carry fix-up + back-substitution (rows descending) + inverse DST
template <class P>
__global__ void __launch_bounds__(P::NT, P::MINB) pass2_kernel(const __grid_constant__ JobList jl) {
    extern __shared__ __align__(16) double2 smem[];
    constexpr int MPT = Cfg<P>::MPT;
    const int job = find_job(jl, blockIdx.x);
    const SolveJob &J = jl.job[job];
    const PlanDev &p = J.p;
    const int b = blockIdx.x - jl.block_start[job];
    const int n = p.n, m = p.m;
    const int s = b * p.R, e = min(m, s + p.R) - 1;
    const double off = p.off;
    double *rowbuf = reinterpret_cast<double *>(smem);
    double yin[MPT], xn[MPT], pc[MPT], cc[MPT];
#pragma unroll
    for (int u = 0; u < MPT; ++u) {
        const int k = threadIdx.x + u * P::NT;
        yin[u] = xn[u] = pc[u] = cc[u] = 0.0;
        if (k < n) {
            if (b > 0) yin[u] = p.ye[size_t(b - 1) * n + k];
            if (b < p.nb - 1) xn[u] = p.fs[size_t(b + 1) * n + k];
            pc[u] = __ldg(p.blk + (size_t(b) * 3 + 0) * n + k);   // P at row e
            if (p.cyclic) {
                // Sherman-Morrison factor from the carried ends: x_0 = X_0,
                // x_{m-1} = Y_{m-1} / beta_{m-1}   (rectsolver.py:203-205)
                const double x0 = p.fs[k];
                const double xl = __ddiv_rn(p.ye[size_t(p.nb - 1) * n + k], __ldg(p.last + 2 * k));
                const double vy = __dadd_rn(x0, __dmul_rn(__ldg(p.cyc + 2 * k), xl));
                cc[u] = __ddiv_rn(vy, __ldg(p.cyc + 2 * k + 1));
            }
        }
    }
    const int glast = s + ((e - s) / P::G) * P::G;
#pragma unroll 1
    for (int g0 = glast; g0 >= s; g0 -= P::G) {
        const int rows = min(P::G, e - g0 + 1);
#pragma unroll
        for (int u = 0; u < MPT; ++u) {
            const int k = threadIdx.x + u * P::NT;
            if (k >= n) continue;
            ModeView mv;
            mv.load(p, k);
            double yv[P::G];
#pragma unroll
            for (int rr = 0; rr < P::G; ++rr)
                yv[rr] = rr < rows ? J.out[size_t(g0 + rr) * n + k] : 0.0;
            double x = xn[u], pcur = pc[u];
            double Pv[P::G], bv[P::G];   // the group's factors, loaded ahead of the chain
#pragma unroll
            for (int rr = 0; rr < P::G; ++rr) {
                const int i = g0 + rr;
                const bool ex = rr < rows && i < mv.len;
                const double *er = p.ex + 4 * size_t(mv.off + i);
                Pv[rr] = ex ? __ldg(er + 3) : 0.0;
                bv[rr] = (i == m - 1) ? mv.b_last : (ex ? __ldg(er + 2) : mv.b_inf);
            }
#pragma unroll
            for (int rr = P::G - 1; rr >= 0; --rr) {
                if (rr >= rows) continue;
                const int i = g0 + rr;
                const bool ex = i < mv.len;
                double y = yv[rr];
                if (b > 0) {
                    const double Pi = ex ? Pv[rr] : pcur;
                    y = fma(Pi, yin[u], y);
                    pcur *= mv.inv_nl;
                }
                const double bi = bv[rr];
                x = __ddiv_rn(__dsub_rn(y, __dmul_rn(off, x)), bi);   // rectsolver.py:90
                double xo = x;
                if (p.cyclic) xo = __dsub_rn(x, __dmul_rn(__ldg(p.smq + size_t(i) * n + k), cc[u]));
                if (p.nsing) {
                    const int si = __ldg(p.sidx + k);
                    if (si >= 0) xo = p.sph[size_t(si) * m + i];   // rectsolver.py:206-207
                }
                rowbuf[rr * n + k] = xo;
            }
            xn[u] = x;
            pc[u] = pcur;
        }
        __syncthreads();
        InvT<P>::run(rowbuf, rows, n, J.out + size_t(g0) * n,
                     J.other ? J.other + size_t(g0) * n : nullptr, J.alpha, J.beta, smem, p);
    }
}

// ---------------------------------------------------------------------------
// Separate-transform solve (kSep: transform lengths without a fused kernel):
// the rows are transformed by the any-length passes of fft_any.cu; the two
// sweeps below are pass1/pass2 without the transform, every CTA handling one
// carry block for a slice of kSepModes modes (coalesced over modes), so any n
// fits.  Same recurrences and carries as the dense path.
constexpr int kSepThreads = 256, kSepMPT = 4, kSepModes = kSepThreads * kSepMPT, kSepG = 8;
__device__ __forceinline__ void sep_block(const JobList &jl, int &job, int &b, int &k0) {
    job = find_job(jl, blockIdx.x);
    const int local = blockIdx.x - jl.block_start[job];
    const int slices = (jl.job[job].p.n + kSepModes - 1) / kSepModes;
    b = local / slices;
    k0 = (local % slices) * kSepModes;
}

// pass 1: local forward elimination of the transformed rows (in) -> yhat (out)
__global__ void __launch_bounds__(kSepThreads) sep_pass1_kernel(const __grid_constant__ JobList jl) {
    int job, b, k0;
    sep_block(jl, job, b, k0);
    const SolveJob &J = jl.job[job];
    const PlanDev &p = J.p;
    const int n = p.n, m = p.m;
    const int s = b * p.R, e = min(m, s + p.R) - 1;
#pragma unroll 1
    for (int u = 0; u < kSepMPT; ++u) {
        const int k = k0 + threadIdx.x + u * kSepThreads;
        if (k >= n) continue;
        ModeView mv;
        mv.load(p, k);
        const int si = p.nsing ? __ldg(p.sidx + k) : -1;
        double y = 0.0, w = 0.0, f = 0.0;
#pragma unroll 1
        for (int g0 = s; g0 <= e; g0 += kSepG) {
            const int rows = min(kSepG, e - g0 + 1);
            double rv[kSepG], lv[kSepG], ibv[kSepG];   // the group's rows and factors ahead of the chain
#pragma unroll
            for (int rr = 0; rr < kSepG; ++rr) {
                const int i = g0 + rr;
                const bool in = rr < rows;
                const bool ex = in && i < mv.len;
                const double *er = p.ex + 4 * size_t(mv.off + i);
                rv[rr] = in ? J.in[size_t(i) * n + k] : 0.0;
                lv[rr] = ex ? __ldg(er) : mv.l_inf;
                ibv[rr] = (i == m - 1) ? mv.ib_last : (ex ? __ldg(er + 1) : mv.ib_inf);
            }
#pragma unroll
            for (int rr = 0; rr < kSepG; ++rr) {
                if (rr >= rows) break;
                const int i = g0 + rr;
                const double r = rv[rr];
                if (si >= 0) p.sf[size_t(si) * m + i] = r;   // fhat column of a pinned mode
                if (i == s) {
                    y = r;
                    w = 1.0;
                } else {
                    const double l = lv[rr];
                    y = __dsub_rn(r, __dmul_rn(l, y));   // rectsolver.py:86
                    w = -l * w;
                }
                f = fma(y, w * ibv[rr], f);
                J.out[size_t(i) * n + k] = y;
            }
        }
        p.ye[size_t(b) * n + k] = y;
        p.fs[size_t(b) * n + k] = f;
    }
}

// pass 2: carry fix-up + back-substitution of yhat (out) -> xhat (out, in place)
__global__ void __launch_bounds__(kSepThreads) sep_pass2_kernel(const __grid_constant__ JobList jl) {
    int job, b, k0;
    sep_block(jl, job, b, k0);
    const SolveJob &J = jl.job[job];
    const PlanDev &p = J.p;
    const int n = p.n, m = p.m;
    const int s = b * p.R, e = min(m, s + p.R) - 1;
    const double off = p.off;
#pragma unroll 1
    for (int u = 0; u < kSepMPT; ++u) {
        const int k = k0 + threadIdx.x + u * kSepThreads;
        if (k >= n) continue;
        ModeView mv;
        mv.load(p, k);
        const double yin = b > 0 ? p.ye[size_t(b - 1) * n + k] : 0.0;
        double x = b < p.nb - 1 ? p.fs[size_t(b + 1) * n + k] : 0.0;
        double pcur = __ldg(p.blk + (size_t(b) * 3 + 0) * n + k);   // P at row e
        double cc = 0.0;
        if (p.cyclic) {   // Sherman-Morrison factor from the carried ends (rectsolver.py:203-205)
            const double x0 = p.fs[k];
            const double xl = __ddiv_rn(p.ye[size_t(p.nb - 1) * n + k], __ldg(p.last + 2 * k));
            const double vy = __dadd_rn(x0, __dmul_rn(__ldg(p.cyc + 2 * k), xl));
            cc = __ddiv_rn(vy, __ldg(p.cyc + 2 * k + 1));
        }
        const int si = p.nsing ? __ldg(p.sidx + k) : -1;
        const int glast = s + ((e - s) / kSepG) * kSepG;
#pragma unroll 1
        for (int g0 = glast; g0 >= s; g0 -= kSepG) {
            const int rows = min(kSepG, e - g0 + 1);
            double yv[kSepG], Pv[kSepG], bv[kSepG];
#pragma unroll
            for (int rr = 0; rr < kSepG; ++rr) {
                const int i = g0 + rr;
                const bool in = rr < rows;
                const bool ex = in && i < mv.len;
                const double *er = p.ex + 4 * size_t(mv.off + i);
                yv[rr] = in ? J.out[size_t(i) * n + k] : 0.0;
                Pv[rr] = ex ? __ldg(er + 3) : 0.0;
                bv[rr] = (i == m - 1) ? mv.b_last : (ex ? __ldg(er + 2) : mv.b_inf);
            }
#pragma unroll
            for (int rr = kSepG - 1; rr >= 0; --rr) {
                if (rr >= rows) continue;
                const int i = g0 + rr;
                double y = yv[rr];
                if (b > 0) {
                    const double Pi = i < mv.len ? Pv[rr] : pcur;
                    y = fma(Pi, yin, y);
                    pcur *= mv.inv_nl;
                }
                x = __ddiv_rn(__dsub_rn(y, __dmul_rn(off, x)), bv[rr]);   // rectsolver.py:90
                double xo = x;
                if (p.cyclic) xo = __dsub_rn(x, __dmul_rn(__ldg(p.smq + size_t(i) * n + k), cc));
                if (si >= 0) xo = p.sph[size_t(si) * m + i];   // rectsolver.py:206-207
                J.out[size_t(i) * n + k] = xo;
            }
        }
    }
}

// jobs of one (n, pair): Q^T of every rectangle into its plan scratch, the two
// sweeps with the carries in between, Q back into out with the epilogue
static void run_sep(const std::vector<SolveJob> &jobs, cudaStream_t s) {
    for (size_t j0 = 0; j0 < jobs.size(); j0 += kMaxJobs) {
        JobList jl{}, jc{};
        jl.count = jc.count = (int)std::min<size_t>(kMaxJobs, jobs.size() - j0);
        int tot = 0, totc = 0;
        for (int j = 0; j < jl.count; ++j) {
            SolveJob sj = jobs[j0 + j];
            const PlanDev &p = sj.p;
            double *T = sj.ws->get(size_t(p.m) * p.n);   // transformed right-hand side
            transform_rows_any(p.m, p.n, p.tpair, 0, sj.in, T, 1.0, 0.0, nullptr, s);
            sj.in = T;
            jl.job[j] = sj;
            jc.job[j] = sj;
            jl.block_start[j] = tot;
            jc.block_start[j] = totc;
            tot += p.nb * ((p.n + kSepModes - 1) / kSepModes);
            totc += (p.n + kCarryModes - 1) / kCarryModes;
        }
        jl.block_start[jl.count] = tot;
        jc.block_start[jc.count] = totc;
        sep_pass1_kernel<<<tot, kSepThreads, 0, s>>>(jl);
        FD_CUDA(cudaGetLastError());
        carry_kernel<<<totc, kCarryThreads, carry_smem(jc), s>>>(jc);
        FD_CUDA(cudaGetLastError());
        for (int j = 0; j < jl.count; ++j) {
            const PlanDev &p = jl.job[j].p;
            if (!p.nsing) continue;
            if (!p.pinv) FD_FAIL(FD_ERR_SINGULAR, "plan is singular (pin_mean plan without pseudo-inverses)");
            pinv_kernel<<<dim3((p.m + 255) / 256, p.nsing), 256, 0, s>>>(p.m, p.nsing, p.pinv, p.sf, p.sph);
            FD_CUDA(cudaGetLastError());
        }
        sep_pass2_kernel<<<tot, kSepThreads, 0, s>>>(jl);
        FD_CUDA(cudaGetLastError());
        for (int j = 0; j < jl.count; ++j) {
            const SolveJob &sj = jl.job[j];
            transform_rows_any(sj.p.m, sj.p.n, sj.p.tpair, 1, sj.out, sj.out, sj.alpha, sj.beta, sj.other, s);
        }
    }
}

// plain row transform (apply_Q): rows of `in` -> `out`
template <class P>
__global__ void __launch_bounds__(P::NT) dst_rows_kernel(int rows_total, int n, const double *in,
                                                         double *out, PlanDev p) {
    extern __shared__ __align__(16) double2 smem[];
    double *rowbuf = reinterpret_cast<double *>(smem);
    const int g0 = blockIdx.x * P::G;
    const int rows = min(P::G, rows_total - g0);
    for (int idx = threadIdx.x; idx < rows * n; idx += P::NT) rowbuf[idx] = in[size_t(g0) * n + idx];
    __syncthreads();
    InvT<P>::run(rowbuf, rows, n, out + size_t(g0) * n, nullptr, 1.0, 0.0, smem, p);
}

// dense basis transform of rows (any pair): forward = Q^T, inverse = Q
template <class P>
__global__ void __launch_bounds__(P::NT) dense_rows_kernel(int rows_total, int n, const double *in,
                                                           double *out, PlanDev p, int inverse) {
    extern __shared__ __align__(16) double2 smem[];
    double *rowbuf = reinterpret_cast<double *>(smem);
    const int g0 = blockIdx.x * P::G;
    const int rows = min(P::G, rows_total - g0);
    if (inverse) {
        for (int idx = threadIdx.x; idx < rows * n; idx += P::NT) rowbuf[idx] = in[size_t(g0) * n + idx];
        __syncthreads();
        InvT<P>::run(rowbuf, rows, n, out + size_t(g0) * n, nullptr, 1.0, 0.0, smem, p);
    } else {
        FwdT<P>::run(in + size_t(g0) * n, rows, n, rowbuf, smem, p);
        for (int idx = threadIdx.x; idx < rows * n; idx += P::NT) out[size_t(g0) * n + idx] = rowbuf[idx];
    }
}

// ---------------------------------------------------------------------------
// host side
int transform_kind(int n, int pair) {
    const int N = n + 1;
    if (n < 1) return -1;
    if (pair == kPairDD && (N & (N - 1)) == 0 && N >= 256 && N <= 4096) return kFFT;
    if (pair == kPairPP && (n & 1)) return -1;   // periodic transforms need an even length
    if (n <= kDenseMax) return kDense;   // any pair: periodic-table dense transform
    if (n <= kSepMax) return kSep;       // any length: Stockham / Bluestein passes + sweeps
    return -1;
}

int rows_per_block(int n, int pair) {
    const int N = n + 1;
    if (transform_kind(n, pair) == kFFT) return N >= 4096 ? 8 : 16;
    if (transform_kind(n, pair) == kSep) return 32;
    // one group per carry block: more CTAs for the small dense solves
    return n <= 160 ? DenseDstT<1, 160, 4>::G : DenseDstT<1, 256>::G;
}

template <class P>
static void setup_smem(const void *fn) {
    // once per (kernel, device)
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    FD_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    if (done.insert({fn, dev}).second)
        FD_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM));
}

template <class P>
static void run_solve(const std::vector<SolveJob> &jobs, cudaStream_t s) {
    for (size_t j0 = 0; j0 < jobs.size(); j0 += kMaxJobs) {
        JobList jl{}, jc{};
        jl.count = jc.count = (int)std::min<size_t>(kMaxJobs, jobs.size() - j0);
        int tot = 0, totc = 0;
        for (int j = 0; j < jl.count; ++j) {
            jl.job[j] = jobs[j0 + j];
            jc.job[j] = jobs[j0 + j];
            jl.block_start[j] = tot;
            jc.block_start[j] = totc;
            tot += jobs[j0 + j].p.nb;
            totc += (jobs[j0 + j].p.n + kCarryModes - 1) / kCarryModes;
        }
        jl.block_start[jl.count] = tot;
        jc.block_start[jc.count] = totc;
        setup_smem<P>((const void *)pass1_kernel<P>);
        setup_smem<P>((const void *)pass2_kernel<P>);
        pass1_kernel<P><<<tot, P::NT, P::SMEM, s>>>(jl);
        FD_CUDA(cudaGetLastError());
        carry_kernel<<<totc, kCarryThreads, carry_smem(jc), s>>>(jc);
        FD_CUDA(cudaGetLastError());
        for (int j = 0; j < jl.count; ++j) {
            const PlanDev &p = jl.job[j].p;
            if (!p.nsing) continue;
            if (!p.pinv) FD_FAIL(FD_ERR_SINGULAR, "plan is singular (pin_mean plan without pseudo-inverses)");
            pinv_kernel<<<dim3((p.m + 255) / 256, p.nsing), 256, 0, s>>>(p.m, p.nsing, p.pinv, p.sf, p.sph);
            FD_CUDA(cudaGetLastError());
        }
        pass2_kernel<P><<<tot, P::NT, P::SMEM, s>>>(jl);
        FD_CUDA(cudaGetLastError());
    }
}

template <class P>
static void run_dst(int rows, int n, const double *in, double *out, const double2 *tw,
                    const double *dense, cudaStream_t s) {
    PlanDev p{};
    p.n = n;
    p.scale = sqrt(2.0 / (n + 1));
    p.tw = tw;
    p.dense = dense;
    setup_smem<P>((const void *)dst_rows_kernel<P>);
    const int grid = (rows + P::G - 1) / P::G;
    dst_rows_kernel<P><<<grid, P::NT, P::SMEM, s>>>(rows, n, in, out, p);
    FD_CUDA(cudaGetLastError());
}

#define FD_FFT_DISPATCH(LGV, CALL) \
    case LGV: {                    \
        using P = FftDst<LGV>;     \
        CALL;                      \
    } break;

static int lg_of(int n) {
    int lg = 0;
    while ((1 << lg) < 2 * (n + 1)) ++lg;
    return lg;
}

void launch_solve(const std::vector<SolveJob> &jobs, cudaStream_t s) {
    if (jobs.empty()) return;
    const int n = jobs[0].p.n;
    for (auto &j : jobs)
        if (j.p.n != n) FD_FAIL(FD_ERR_VALIDATION, "launch_solve: mixed transform lengths in one batch");
    for (auto &j : jobs)
        if (j.p.tpair != jobs[0].p.tpair) FD_FAIL(FD_ERR_VALIDATION, "launch_solve: mixed transform pairs in one batch");
    if (jobs[0].p.tkind == kSep) {
        if (!jobs[0].ws) FD_FAIL(FD_ERR_VALIDATION, "launch_solve: separate-transform solve needs plan scratch");
        run_sep(jobs, s);
        return;
    }
    if (jobs[0].p.dense) {
        if (n <= 128) run_solve<DenseDstT<1, 128, 4>>(jobs, s);
        else if (n <= 160) run_solve<DenseDstT<1, 160, 4>>(jobs, s);
        else if (n <= 256) run_solve<DenseDstT<1, 256>>(jobs, s);
        else if (n <= 512) run_solve<DenseDstT<2, 256>>(jobs, s);
        else if (n <= 1024) run_solve<DenseDstT<4, 256>>(jobs, s);
        else run_solve<DenseDstT<8, 256>>(jobs, s);
        return;
    }
    if (jobs[0].ws && launch_persist(jobs, s, *jobs[0].ws)) return;
    switch (lg_of(n)) {
        FD_FFT_DISPATCH(9, run_solve<P>(jobs, s))
        FD_FFT_DISPATCH(10, run_solve<P>(jobs, s))
        FD_FFT_DISPATCH(11, run_solve<P>(jobs, s))
        FD_FFT_DISPATCH(12, run_solve<P>(jobs, s))
        FD_FFT_DISPATCH(13, run_solve<P>(jobs, s))
        default:
            FD_FAIL(FD_ERR_UNSUPPORTED, "no transform for this length");
    }
}

template <class P>
static void run_dense_rows(int rows, int n, int pair, int inverse, const double *in, double *out,
                           const double *dense, cudaStream_t s) {
    PlanDev p{};
    p.n = n;
    p.tpair = pair;
    p.scale = (pair == kPairNN || pair == kPairPP) ? sqrt(2.0 / n) : sqrt(2.0 / (n + 1));
    p.dense = dense;
    setup_smem<P>((const void *)dense_rows_kernel<P>);
    const int grid = (rows + P::G - 1) / P::G;
    dense_rows_kernel<P><<<grid, P::NT, P::SMEM, s>>>(rows, n, in, out, p, inverse);
    FD_CUDA(cudaGetLastError());
}

void launch_transform_rows(int rows, int n, int pair, int inverse, const double *in, double *out,
                           const double *dense, cudaStream_t s) {
    if (rows <= 0) return;
    if (transform_kind(n, pair) == kSep) {
        transform_rows_any(rows, n, pair, inverse, in, out, 1.0, 0.0, nullptr, s);
        return;
    }
    if (!dense) FD_FAIL(FD_ERR_UNSUPPORTED, "no dense table for this transform");
    if (n <= 128) run_dense_rows<DenseDstT<1, 128>>(rows, n, pair, inverse, in, out, dense, s);
    else if (n <= 160) run_dense_rows<DenseDstT<1, 160>>(rows, n, pair, inverse, in, out, dense, s);
    else if (n <= 256) run_dense_rows<DenseDstT<1, 256>>(rows, n, pair, inverse, in, out, dense, s);
    else if (n <= 512) run_dense_rows<DenseDstT<2, 256>>(rows, n, pair, inverse, in, out, dense, s);
    else if (n <= 1024) run_dense_rows<DenseDstT<4, 256>>(rows, n, pair, inverse, in, out, dense, s);
    else run_dense_rows<DenseDstT<8, 256>>(rows, n, pair, inverse, in, out, dense, s);
}

void launch_dst_rows(int rows, int n, const double *in, double *out, const double2 *tw,
                     const double *dense, cudaStream_t s) {
    if (rows <= 0) return;
    if (transform_kind(n) == kSep) {
        transform_rows_any(rows, n, kPairDD, 0, in, out, 1.0, 0.0, nullptr, s);
        return;
    }
    if (transform_kind(n) == kDense) {
        if (n <= 128) run_dst<DenseDstT<1, 128>>(rows, n, in, out, tw, dense, s);
        else if (n <= 160) run_dst<DenseDstT<1, 160>>(rows, n, in, out, tw, dense, s);
        else if (n <= 256) run_dst<DenseDstT<1, 256>>(rows, n, in, out, tw, dense, s);
        else if (n <= 512) run_dst<DenseDstT<2, 256>>(rows, n, in, out, tw, dense, s);
        else if (n <= 1024) run_dst<DenseDstT<4, 256>>(rows, n, in, out, tw, dense, s);
        else run_dst<DenseDstT<8, 256>>(rows, n, in, out, tw, dense, s);
        return;
    }
    switch (lg_of(n)) {
        FD_FFT_DISPATCH(9, run_dst<P>(rows, n, in, out, tw, dense, s))
        FD_FFT_DISPATCH(10, run_dst<P>(rows, n, in, out, tw, dense, s))
        FD_FFT_DISPATCH(11, run_dst<P>(rows, n, in, out, tw, dense, s))
        FD_FFT_DISPATCH(12, run_dst<P>(rows, n, in, out, tw, dense, s))
        FD_FFT_DISPATCH(13, run_dst<P>(rows, n, in, out, tw, dense, s))
        default:
            FD_FAIL(FD_ERR_UNSUPPORTED, "no transform for this length");
    }
}

}  // namespace fd
