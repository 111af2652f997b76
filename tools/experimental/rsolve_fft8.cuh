// Real-symmetric row-pair DST-I with EIGHT points per thread (N/8 threads per
// pair) -- the same transform as RFft (rsolve_common.cuh: 16 points per thread,
// N/16 threads per pair), traded for occupancy: half the registers per thread,
// twice the warps per pair, one more shared-memory exchange.
//
//   N = 1024 = 8 x 8 x 8 x 2, input index j = 128 n1 + 16 n2 + 2 n3 + n4,
//   output index k = k1 + 8 k2 + 64 k3 + 512 k4.  Pass p transforms the input
//   digit n_p after the twiddle W_{M_p}^{K_{p-1} n_p} (M_p = R_1 .. R_p, K_{p-1}
//   the output digits so far) -- the scheme of RFft with other radices.
//   Positions in the exchange buffer are padded pad8(p) = p + p/8 (one complex
//   of 16 bytes per 8), which makes the stride-8 writes of the first pass
//   conflict-free; every other access walks consecutive positions.
#pragma once
#include "rsolve_common.cuh"

namespace fd {

__device__ __forceinline__ int pad8(int p) { return p + (p >> 3); }

template <int NL>
struct RFft8 {
    static_assert(NL == 10, "radix 8 x 8 x 8 x 2");
    static constexpr int N = 1 << NL;
    static constexpr int T = N / 8;                       // threads per row pair
    static constexpr int PADN = N + N / 8;                // complex entries per pair region
    static constexpr size_t REG = size_t(PADN) * 16;
    static constexpr int XR = (N - 1) + ((N - 2) >> 4);   // row b of the padded X layout (as RS<NL>)
    static constexpr int NTW = 8 + 64 + N / 2;            // W_64^a (a < 8), W_512^a (a < 64), W_N^a (a < N/2)
    static_assert(size_t(2) * (XR + 1) * 8 <= REG, "transformed rows fit the pair region");

    static void host_twiddles(double2 *tw) {
        const long double PI = 3.141592653589793238462643383279502884L;
        auto W = [&](long double num, long double den) {
            const long double a = 2.0L * PI * num / den;
            return make_double2((double)cosl(a), (double)(-sinl(a)));
        };
        for (int a = 0; a < 8; ++a) tw[a] = W(a, 64);
        for (int a = 0; a < 64; ++a) tw[8 + a] = W(a, 512);
        for (int a = 0; a < N / 2; ++a) tw[72 + a] = W(a, N);
    }

    // pre-weighted input of the first pass: v[r] = y_a(j) + i y_b(j), j = t + r T
    __device__ static void load(double2 (&v)[8], const double *A, const double *B, const double *al, double h2,
                                int t) {
        if (!B) B = A;   // a single row is paired with itself, the second output is not stored
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int j = t + r * T;
            if (r == 0 && t == 0) {
                v[0] = make_double2(0.0, 0.0);   // x_0 = x_N = 0
                continue;
            }
            const double a = al[j], b = a - h2;
            const int i1 = j - 1, i2 = N - 1 - j;
            v[r].x = fma(a, A[i1], b * A[i2]);
            v[r].y = fma(a, B[i1], b * B[i2]);
        }
    }
    // C = FFT_N(c) in natural order at buf[pad8(k)]
    __device__ static void passes(double2 *buf, double2 (&v)[8], const double2 *tw, int t, int pr) {
        // pass 1: n1 -> k1, element (t, k1) to position 8 t + k1
        dft<8>(v);
        {
            double2 *w = buf + 9 * t;   // pad8(8 t + r)
#pragma unroll
            for (int r = 0; r < 8; ++r) w[r] = v[r];
        }
        rsync<T>(pr);
        // pass 2: thread (k1, tl) = (t & 7, t >> 3), n2 -> k2; reads 128 r + t, writes k1 + 8 k2 + 64 tl
        {
            const double2 *rd = buf + pad8(t);
#pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = rd[144 * r];
            const double2 w = tw[t & 7];
            rsync<T>(pr);
            apply_powers<8>(v, w);
            dft<8>(v);
            double2 *wr = buf + (t & 7) + 72 * (t >> 3);   // pad8(k1 + 64 tl); pad8 adds 9 per k2
#pragma unroll
            for (int r = 0; r < 8; ++r) wr[9 * r] = v[r];
            rsync<T>(pr);
        }
        // pass 3: thread (K2, n4) = (t & 63, t >> 6), n3 -> k3; reads t + 128 r, writes K2 + 64 k3 + 512 n4
        {
            const double2 *rd = buf + pad8(t);
#pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = rd[144 * r];
            const double2 w = tw[8 + (t & 63)];
            rsync<T>(pr);
            apply_powers<8>(v, w);
            dft<8>(v);
            double2 *wr = buf + pad8(t & 63) + 576 * (t >> 6);   // pad8(K2 + 512 n4); pad8 adds 72 per k3
#pragma unroll
            for (int r = 0; r < 8; ++r) wr[72 * r] = v[r];
            rsync<T>(pr);
        }
        // pass 4, in place: K3 = t + 128 u, n4 -> k4 at K3 + 512 k4
        {
            double2 *p = buf + pad8(t);
            double2 a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a[u] = p[144 * u];
                b[u] = p[144 * u + 576];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                b[u] = cmul(b[u], tw[72 + t + 128 * u]);
                dft2(a[u], b[u]);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                p[144 * u] = a[u];
                p[144 * u + 576] = b[u];
            }
            rsync<T>(pr);
        }
    }
    // C -> transformed rows (padded X layout xi) of A (and B when XB)
    __device__ static void post(double2 *buf, double *scr, int t, int pr, int lane, double *XA, double *XB) {
        const bool HB = XB != nullptr;
        double ea[4], eb[4], da[4], db[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int k = 4 * t + i;
            const double2 c = buf[pad8(k)];
            double2 c2 = make_double2(0.0, 0.0);
            if (i > 0 || t > 0) c2 = buf[pad8(N - k)];
            ea[i] = c2.y - c.y;
            eb[i] = c.x - c2.x;
            da[i] = c.x + c2.x;
            db[i] = c.y + c2.y;
        }
#pragma unroll
        for (int i = 1; i < 4; ++i) {
            da[i] += da[i - 1];
            db[i] += db[i - 1];
        }
        double ia = da[3], ib = db[3];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double xa = __shfl_up_sync(0xffffffffu, ia, o), xb = __shfl_up_sync(0xffffffffu, ib, o);
            if (lane >= o) {
                ia += xa;
                ib += xb;
            }
        }
        double pa = __shfl_up_sync(0xffffffffu, ia, 1), pb = __shfl_up_sync(0xffffffffu, ib, 1);
        if (lane == 0) {
            pa = 0.0;
            pb = 0.0;
        }
        const int w = t >> 5;
        if (lane == 31) {
            scr[(pr * 8 + w) * 2] = ia;
            scr[(pr * 8 + w) * 2 + 1] = ib;
        }
        rsync<T>(pr);   // every C value read, the warp totals visible
#pragma unroll
        for (int q = 0; q < T / 32 - 1; ++q)
            if (q < w) {
                pa += scr[(pr * 8 + q) * 2];
                pb += scr[(pr * 8 + q) * 2 + 1];
            }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int k = 4 * t + i;
            if (i > 0 || t > 0) XA[xi(2 * k - 1)] = ea[i];
            XA[xi(2 * k)] = da[i] + pa;
            if (HB) {
                if (i > 0 || t > 0) XB[xi(2 * k - 1)] = eb[i];
                XB[xi(2 * k)] = db[i] + pb;
            }
        }
    }
    // full transform of rows A (, B) -> padded X rows in the pair region; `staged`:
    // the rows sit in the region themselves (their loads must finish before pass 1 writes)
    __device__ __forceinline__ static void run(double2 *buf, const double *A, const double *B, const double *al,
                                               double h2, const double2 *tw, double *scr, int t, int pr, int lane,
                                               double *XA, double *XB, bool staged = false) {
        double2 v[8];
        load(v, A, B, al, h2, t);
        if (staged) rsync<T>(pr);
        passes(buf, v, tw, t, pr);
        post(buf, scr, t, pr, lane, XA, XB);
    }
};

}  // namespace fd
