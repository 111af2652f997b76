// Device building blocks of the DST-I transforms (shared by solve.cu and
// persist.cu): complex helpers, in-register radix-2/4/8/16 DFTs, the
// Stockham radix-16 FFT of a packed row pair, the dense fallback, per-mode
// factor-table views.
#pragma once
#include "fd_internal.h"

namespace fd {

// ---------------------------------------------------------------------------
// complex helpers
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 w) {
    return make_double2(fma(a.x, w.x, -a.y * w.y), fma(a.x, w.y, a.y * w.x));
}
// multiply by -i
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }

#define C16_1 0.92387953251128675613  // cos(pi/8)
#define S16_1 0.38268343236508977173  // sin(pi/8)
#define R2 0.70710678118654752440

// a * e^{-2 pi i p / 16}, p known at compile time
template <int P>
__device__ __forceinline__ double2 tw16(double2 a) {
    constexpr int p = P & 15;
    if constexpr (p == 0) return a;
    else if constexpr (p == 4) return mul_mi(a);
    else if constexpr (p == 8) return make_double2(-a.x, -a.y);
    else if constexpr (p == 12) return make_double2(-a.y, a.x);
    else if constexpr (p == 2) return make_double2(R2 * (a.x + a.y), R2 * (a.y - a.x));
    else if constexpr (p == 6) return make_double2(R2 * (a.y - a.x), -R2 * (a.x + a.y));
    else {
        constexpr double c[16] = {1, C16_1, R2, S16_1, 0, -S16_1, -R2, -C16_1,
                                  -1, -C16_1, -R2, -S16_1, 0, S16_1, R2, C16_1};
        constexpr double s[16] = {0, S16_1, R2, C16_1, 1, C16_1, R2, S16_1,
                                  0, -S16_1, -R2, -C16_1, -1, -C16_1, -R2, -S16_1};
        return cmul(a, make_double2(c[p], -s[p]));
    }
}

__device__ __forceinline__ void dft2(double2 &a, double2 &b) {
    double2 t = a;
    a = cadd(t, b);
    b = csub(t, b);
}
// forward 4-point DFT in place, natural order
__device__ __forceinline__ void dft4(double2 &a0, double2 &a1, double2 &a2, double2 &a3) {
    double2 s02 = cadd(a0, a2), d02 = csub(a0, a2), s13 = cadd(a1, a3), d13 = csub(a1, a3);
    a0 = cadd(s02, s13);
    a2 = csub(s02, s13);
    a1 = make_double2(d02.x + d13.y, d02.y - d13.x);
    a3 = make_double2(d02.x - d13.y, d02.y + d13.x);
}

template <int R>
__device__ __forceinline__ void dft(double2 (&v)[R]);

template <>
__device__ __forceinline__ void dft<2>(double2 (&v)[2]) { dft2(v[0], v[1]); }
template <>
__device__ __forceinline__ void dft<4>(double2 (&v)[4]) { dft4(v[0], v[1], v[2], v[3]); }
template <>
__device__ __forceinline__ void dft<8>(double2 (&v)[8]) {
    // n = 2 n1 + n2, k = k1 + 4 k2
    dft4(v[0], v[2], v[4], v[6]);
    dft4(v[1], v[3], v[5], v[7]);
    v[3] = tw16<2>(v[3]);
    v[5] = tw16<4>(v[5]);
    v[7] = tw16<6>(v[7]);
    dft2(v[0], v[1]);
    dft2(v[2], v[3]);
    dft2(v[4], v[5]);
    dft2(v[6], v[7]);
    // X[k1 + 4 k2] sits at v[2 k1 + k2]
    double2 t[8];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
        for (int k2 = 0; k2 < 2; ++k2) t[k1 + 4 * k2] = v[2 * k1 + k2];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = t[i];
}
template <>
__device__ __forceinline__ void dft<16>(double2 (&v)[16]) {
    // n = 4 n1 + n2, k = k1 + 4 k2
    dft4(v[0], v[4], v[8], v[12]);
    dft4(v[1], v[5], v[9], v[13]);
    dft4(v[2], v[6], v[10], v[14]);
    dft4(v[3], v[7], v[11], v[15]);
    // v[4 k1 + n2] *= W16^{n2 k1}
    v[5] = tw16<1>(v[5]);
    v[6] = tw16<2>(v[6]);
    v[7] = tw16<3>(v[7]);
    v[9] = tw16<2>(v[9]);
    v[10] = tw16<4>(v[10]);
    v[11] = tw16<6>(v[11]);
    v[13] = tw16<3>(v[13]);
    v[14] = tw16<6>(v[14]);
    v[15] = tw16<9>(v[15]);
    dft4(v[0], v[1], v[2], v[3]);
    dft4(v[4], v[5], v[6], v[7]);
    dft4(v[8], v[9], v[10], v[11]);
    dft4(v[12], v[13], v[14], v[15]);
    double2 t[16];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) t[k1 + 4 * k2] = v[4 * k1 + k2];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = t[i];
}

__device__ __forceinline__ int pad16(int q) { return q + (q >> 4); }

// ---------------------------------------------------------------------------
// Row sources / sinks.  A "row" is n contiguous doubles.
struct GRow {   // global memory
    const double *p;
    __device__ double get(int j) const { return p ? __ldg(p + j) : 0.0; }
};
struct SRow {   // shared memory
    const double *p;
    __device__ double get(int j) const { return p ? p[j] : 0.0; }
};

// Sink for the transform output k in [0, n): out[k] = alpha*val + beta*other[k]
struct OutRow {
    double *p;
    const double *other;
    double alpha, beta;
    __device__ void put(int k, double v) const {
        if (!p) return;
        double r = alpha * v;
        if (other) r = fma(beta, __ldg(other + k), r);
        p[k] = r;
    }
};
struct SmemRow {
    double *p;
    __device__ void put(int k, double v) const {
        if (p) p[k] = v;
    }
};

// ---------------------------------------------------------------------------
// DST-I of row pairs via one complex FFT of length L = 2N (N = n + 1 = 2^(LG-1)):
// c = a + i b odd-extended, C = FFT(c) = 2 DST(b) - 2i DST(a).
// Twiddle sources: e^{-2 pi i q / L}.
struct TwGlobal {   // full table in global memory (L1/L2 cached)
    const double2 *tw;
    template <int STEP>
    __device__ double2 at(int m) const { return __ldg(tw + m * STEP); }
};
// Two-level shared-memory table: A[a] = e^{-2 pi i a/256}, B[b] = e^{-2 pi i b/L},
// q = (L/256) a + b.  4.6 KB instead of the L-entry table, so the twiddles stay
// on chip next to ~200 KB of exchange/staging buffers per SM.
template <int LG>
struct TwSmem {
    const double2 *A, *B;
    static constexpr int SH = LG - 8;
    template <int STEP>
    __device__ double2 at(int m) const {
        if constexpr ((STEP & ((1 << SH) - 1)) == 0) {
            return A[m * (STEP >> SH)];
        } else {
            const int q = m * STEP;
            const int b = q & ((1 << SH) - 1);
            const double2 w = A[q >> SH];
            return b ? cmul(w, B[b]) : w;
        }
    }
};

template <int LG, int CTA_THREADS = 256>
struct FftDst {
    static constexpr int L = 1 << LG;
    static constexpr int N = L / 2;
    static constexpr int T = L / 16;                       // threads per pair
    static constexpr int PAIRS = (T >= CTA_THREADS) ? 1 : CTA_THREADS / T;
    static constexpr int NT = PAIRS * T;
    static constexpr int G = 2 * PAIRS;                    // rows per group
    static constexpr int MINB = NT <= 256 ? 2 : 1;         // CTAs per SM (register cap)
    static constexpr int PADL = L + L / 16;
    static constexpr int NMID = (LG - 1) / 4 - 1;
    static constexpr int RL = 1 << (LG - 4 * ((LG - 1) / 4));
    static constexpr int NS_LAST = L / RL;
    static constexpr size_t SMEM = size_t(PAIRS) * PADL * sizeof(double2);

    template <class Src>
    __device__ static void first_pass(double2 *buf, const Src &A, const Src &B, int t) {
        double2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            int q = t + r * (L / 16);
            double2 c;
            if (r < 8) {
                c = (q == 0) ? make_double2(0.0, 0.0) : make_double2(A.get(q - 1), B.get(q - 1));
            } else {
                int qq = 2 * N - q;
                c = (qq == N) ? make_double2(0.0, 0.0) : make_double2(-A.get(qq - 1), -B.get(qq - 1));
            }
            v[r] = c;
        }
        __syncthreads();   // the source rows may alias the exchange buffer
        dft<16>(v);
#pragma unroll
        for (int r = 0; r < 16; ++r) buf[pad16(16 * t + r)] = v[r];
        __syncthreads();
    }

    template <int NS, class TW>
    __device__ static void mid_pass(double2 *buf, const TW &tw, int t) {
        constexpr int NB = L / 16;
        double2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = buf[pad16(t + r * NB)];
        __syncthreads();
        const int jm = t % NS;
        constexpr int TS = L / (NS * 16);
#pragma unroll
        for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], tw.template at<TS>(jm * r));
        dft<16>(v);
        const int idx = (t / NS) * NS * 16 + jm;
#pragma unroll
        for (int r = 0; r < 16; ++r) buf[pad16(idx + r * NS)] = v[r];
        __syncthreads();
    }

    template <int K, int NS, class TW>
    __device__ static void mids(double2 *buf, const TW &tw, int t) {
        if constexpr (K > 0) {
            mid_pass<NS>(buf, tw, t);
            mids<K - 1, NS * 16>(buf, tw, t);
        }
    }

    template <class Sink, class TW>
    __device__ static void last_pass(double2 *buf, const TW &tw, int t,
                                     const Sink &outA, const Sink &outB, double scale) {
        constexpr int NB = L / RL;
        constexpr int PER = NB / T;
        double2 v[PER][RL];
#pragma unroll
        for (int u = 0; u < PER; ++u)
#pragma unroll
            for (int r = 0; r < RL; ++r) v[u][r] = buf[pad16(t + u * T + r * NB)];
        __syncthreads();   // the sink may alias the exchange buffer
        const double sa = -0.5 * scale, sb = 0.5 * scale;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int j = t + u * T;
#pragma unroll
            for (int r = 1; r < RL; ++r) v[u][r] = cmul(v[u][r], tw.template at<1>(j * r));
            dft<RL>(v[u]);
#pragma unroll
            for (int r = 0; r < RL; ++r) {
                int o = j + r * NB;
                if (o >= 1 && o < N) {
                    outA.put(o - 1, sa * v[u][r].y);
                    outB.put(o - 1, sb * v[u][r].x);
                }
            }
        }
    }

};

// Power-based twiddles for Fft2: one conflict-free shared-memory load of the
// pass's base root w = e^{-2 pi i j / span} per radix group, then w^r by two
// interleaved multiplication chains (odd and even powers, step w^2): at most 8
// rounding steps (< 2e-15 relative), and ~15x less shared-memory traffic than
// loading every twiddle.  Tables (exact, from the host-built L-point table):
//   m16[q]  = e^{-2 pi i q / 256}    (first mid pass, NS = 16)
//   m256[q] = e^{-2 pi i q / 4096}   (second mid pass, NS = 256, LG = 13)
//   la/lb   : last pass, e^{-2 pi i j / L} = la[j] (L/RL <= 256) or
//             la[j >> 4] * lb[j & 15] with la[a] = e^{-2 pi i 16 a / L}.
struct TwPow {
    const double2 *m16, *m256, *la, *lb;
};
template <int R>
__device__ __forceinline__ void apply_powers(double2 (&v)[R], double2 w) {
    if constexpr (R == 2) {
        v[1] = cmul(v[1], w);
    } else {
        const double2 w2 = cmul(w, w);
        double2 po = w, pe = w2;
        v[1] = cmul(v[1], po);
        v[2] = cmul(v[2], pe);
#pragma unroll
        for (int r = 3; r < R; r += 2) {
            po = cmul(po, w2);
            v[r] = cmul(v[r], po);
            if (r + 1 < R) {
                pe = cmul(pe, w2);
                v[r + 1] = cmul(v[r + 1], pe);
            }
        }
    }
}

// Barrier over the T threads of one row pair: a warp sync for a single-warp
// pair, else a named barrier (ids 1..15; id 0 is __syncthreads).
template <int T>
__device__ __forceinline__ void pair_sync(int pr) {
    if constexpr (T <= 32) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + pr), "r"(T) : "memory");
    }
}

// ---------------------------------------------------------------------------
// Lean variant for the persistent kernel: identical arithmetic to FftDst, with
// the padded addresses hoisted out of the radix loops (every stride is a
// multiple of 16 points), the odd-extension mirror resolved per thread, and
// only the outputs o < N of the last pass produced (o = j + r L/RL < N  <=>
// r < RL/2), so no per-element bounds tests remain.
template <int LG, int CTA_THREADS>
struct Fft2 {
    using Base = FftDst<LG, CTA_THREADS>;
    static constexpr int L = Base::L, N = Base::N, T = Base::T, PAIRS = Base::PAIRS;
    static constexpr int NT = Base::NT, G = Base::G, PADL = Base::PADL, NMID = Base::NMID;
    static constexpr int RL = Base::RL;

    // first pass, split so the caller can act between the source reads and the
    // exchange-buffer writes: load() reads rows A, B (shared memory; either may
    // be null = zero row) into registers, store() transforms and writes.
    __device__ static void load(double2 (&v)[16], const double *A, const double *B, int t) {
        constexpr int S = N / 8;          // = L/16, distance between radix inputs
        const int b1 = t - 1, b2 = N - 1 - t;
        const bool t0 = (t == 0);
        if (A && B) {
            v[0] = t0 ? make_double2(0.0, 0.0) : make_double2(A[b1], B[b1]);
            v[8] = t0 ? make_double2(0.0, 0.0) : make_double2(-A[b2], -B[b2]);
#pragma unroll
            for (int r = 1; r < 8; ++r) {
                v[r] = make_double2(A[b1 + r * S], B[b1 + r * S]);
                v[8 + r] = make_double2(-A[b2 - r * S], -B[b2 - r * S]);
            }
        } else if (A) {
            v[0] = t0 ? make_double2(0.0, 0.0) : make_double2(A[b1], 0.0);
            v[8] = t0 ? make_double2(0.0, 0.0) : make_double2(-A[b2], 0.0);
#pragma unroll
            for (int r = 1; r < 8; ++r) {
                v[r] = make_double2(A[b1 + r * S], 0.0);
                v[8 + r] = make_double2(-A[b2 - r * S], 0.0);
            }
        } else {
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = make_double2(0.0, 0.0);
        }
    }
    __device__ static void store(double2 *buf, double2 (&v)[16], int t, int pr) {
        dft<16>(v);
        double2 *w = buf + 17 * t;   // pad16(16 t + r) = 17 t + r
#pragma unroll
        for (int r = 0; r < 16; ++r) w[r] = v[r];
        pair_sync<T>(pr);
    }
    // source rows (shared memory) may alias this pair's exchange buffer only
    __device__ static void first(double2 *buf, const double *A, const double *B, int t, int pr) {
        double2 v[16];
        load(v, A, B, t);
        pair_sync<T>(pr);
        store(buf, v, t, pr);
    }

    template <int NS>
    __device__ static void mid(double2 *buf, const TwPow &tw, int t, int pr) {
        constexpr int NB = L / 16, RS = NB + NB / 16;
        static_assert(NS == 16 || NS == 256, "mid pass strides");
        double2 v[16];
        const double2 *rd = buf + pad16(t);
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = rd[r * RS];
        const int jm = t % NS;
        const double2 w = (NS == 16) ? tw.m16[jm] : tw.m256[jm];
        pair_sync<T>(pr);
        apply_powers<16>(v, w);
        dft<16>(v);
        double2 *wr = buf + pad16((t / NS) * NS * 16 + jm);
        constexpr int WS = NS + NS / 16;
#pragma unroll
        for (int r = 0; r < 16; ++r) wr[r * WS] = v[r];
        pair_sync<T>(pr);
    }

    template <int K, int NS>
    __device__ static void mids(double2 *buf, const TwPow &tw, int t, int pr) {
        if constexpr (K > 0) {
            mid<NS>(buf, tw, t, pr);
            mids<K - 1, NS * 16>(buf, tw, t, pr);
        }
    }

    // last pass; sink(k, a_val, b_val) receives output k in [0, n) of rows A and B
    // the sink may alias the exchange buffer of this pair only
    template <class Sink>
    __device__ static void last(double2 *buf, const TwPow &tw, int t, int pr, double scale, const Sink &sink) {
        constexpr int NB = L / RL, PER = NB / T, RS = NB + NB / 16, US = T + T / 16;
        double2 v[PER][RL];
        const double2 *rd = buf + pad16(t);
#pragma unroll
        for (int u = 0; u < PER; ++u)
#pragma unroll
            for (int r = 0; r < RL; ++r) v[u][r] = rd[u * US + r * RS];
        pair_sync<T>(pr);
        const double sa = -0.5 * scale, sb = 0.5 * scale;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int j = t + u * T;
            double2 w;
            if constexpr (NB <= 256) w = tw.la[j];
            else w = cmul(tw.la[j >> 4], tw.lb[j & 15]);
            apply_powers<RL>(v[u], w);
            dft<RL>(v[u]);
#pragma unroll
            for (int r = 0; r < RL / 2; ++r) {
                if (r == 0 && u == 0 && j == 0) continue;   // o = 0 is not an output
                sink(j - 1 + r * NB, sa * v[u][r].y, sb * v[u][r].x);
            }
        }
    }
};

// ---------------------------------------------------------------------------
// Dense DST-I (any n <= kDenseMax): out_k = scale * sum_j sin(pi (j+1)(k+1)/N) in_j,
// N = n + 1.  The sine is periodic in (j+1)(k+1) mod 2N, so a 2N-entry table
// (host-built, exact argument reduction) staged in shared memory serves every
// (j, k); each thread walks its index by k + 1 per j.  MPT modes per thread
// (n <= 256 MPT), G rows per group share every table load.
template <int MPT_, int NT_ = 128, int S_ = 1>
struct DenseDstT {
    // NT_ mode columns x S_ threads each: the S_ threads of a mode split the
    // transform's input sum (small n: more threads, shorter dependent loops)
    static constexpr int S = S_;
    static constexpr int NMODE = NT_;
    static constexpr int NT = NT_ * S_;
    static constexpr int G = NT_ <= 160 ? 4 : 8;   // small n: fewer rows per CTA, more CTAs
    static constexpr int MINB = (S_ > 1 || MPT_ >= 8) ? 1 : 2;   // n > 1024: one CTA per SM (shared memory)
    static constexpr int MPT = MPT_;
    static constexpr int NMAX = NT_ * MPT_;
    // rows + the periodic basis table: 2(n+1) entries (DD sine), 4n (NN cosine) or 2n (PP)
    static constexpr size_t SMEM = size_t(G) * NMAX * sizeof(double) + size_t(4) * (NMAX + 1) * sizeof(double);
    static_assert(S_ == 1 || MPT_ == 1, "split transforms own one mode per thread group");
};

// ---------------------------------------------------------------------------
// per-mode table access (see PlanDev)
struct ModeView {
    int off, len;
    double l_inf, ib_inf, b_inf, inv_nl;
    double b_last, ib_last;
    __device__ void load(const PlanDev &p, int k) {
        off = __ldg(p.ex_off + k);
        len = __ldg(p.ex_len + k);
        const double4 c = *reinterpret_cast<const double4 *>(p.cv + 4 * k);
        l_inf = c.x;
        ib_inf = c.y;
        b_inf = c.z;
        inv_nl = c.w;
        b_last = __ldg(p.last + 2 * k);
        ib_last = __ldg(p.last + 2 * k + 1);
    }
};

__device__ __forceinline__ int find_job(const JobList &jl, int bid) {
    int j = 0;
#pragma unroll 1
    while (j + 1 < jl.count && bid >= jl.block_start[j + 1]) ++j;
    return j;
}


}  // namespace fd
