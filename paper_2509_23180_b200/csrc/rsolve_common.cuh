// Device pieces shared by the real-symmetric persistent solves (rsolve.cu:
// lockstep CTA; rsws.cu: warp-specialised FFT and sweep teams): geometry
// RS<NL>, the real-symmetric row-pair DST-I RFft<NL>, and the per-mode
// factor fall-backs.  See rsolve.cu for the algorithm.
#pragma once
#include "persist_common.cuh"

namespace fd {

__device__ __forceinline__ int xi(int q) { return q + (q >> 4); }

template <int NL>
struct RS {
    static constexpr int N = 1 << NL;
    static constexpr int NT = rs_threads(1 << NL);
    static constexpr int T = N / 16;                  // threads per row pair
    static constexpr int P = NT / T;                  // pairs per CTA
    static constexpr int G = 2 * P;                   // rows per group
    static constexpr int PADN = N + N / 16;           // complex entries per pair region
    static constexpr int NMID = (NL - 1) / 4 - 1;
    static constexpr int RL = 1 << (NL - 4 * ((NL - 1) / 4));
    static constexpr int NB = N / RL;                 // last-pass butterflies
    static constexpr int PER = NB / T;                // ... per thread
    static constexpr int MPT = (N - 1 + NT - 1) / NT; // modes per thread in the sweeps
    static constexpr int XR = (N - 1) + ((N - 2) >> 4);   // row b of the padded X layout
    static constexpr size_t REG = size_t(PADN) * 16;
    static constexpr size_t OFF_TW = size_t(P) * REG;     // m16[16], la[256]
    static constexpr size_t OFF_AL = OFF_TW + 272 * 16;   // alpha[N]
    static constexpr size_t OFF_SC = OFF_AL + size_t(N) * 8;
    static constexpr size_t OFF_LT = OFF_SC + size_t(P) * 16 * 8;
    static constexpr size_t SMEM = rs_smem(1 << NL);
    static_assert(OFF_LT == rs_fixed_smem(N), "layout shared with the plan builder");
    static_assert(PER * RL == 16, "16 points per thread in the last pass");
    static_assert(XR * 2 <= PADN * 2, "transformed rows fit the pair region");
    static_assert(NMID <= 1, "N <= 4096");
};

// barrier over the T threads of one pair (T = 16: half warp)
template <int T>
__device__ __forceinline__ unsigned pair_mask(int pr) {
    if constexpr (T >= 32) return 0xffffffffu;
    else return 0xffffu << (16 * (pr & 1));
}
template <int T>
__device__ __forceinline__ void rsync(int pr) {
    if constexpr (T <= 32) __syncwarp(pair_mask<T>(pr));
    else asm volatile("bar.sync %0, %1;" ::"r"(1 + pr), "r"(T) : "memory");
}

template <int NL>
struct RFft {
    using C = RS<NL>;
    static constexpr int N = C::N, T = C::T, RL = C::RL, NB = C::NB, PER = C::PER;

    // pre-weighted input of the first pass: v[r] = y_a(j) + i y_b(j), j = t + r T
    __device__ static void load(double2 (&v)[16], const double *A, const double *B, const double *al,
                                double h2, int t) {
        const bool HB = B != nullptr;
        if (!HB) B = A;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int j = t + r * T;
            if (r == 0 && t == 0) {
                v[0] = make_double2(0.0, 0.0);   // x_0 = x_N = 0
                continue;
            }
            const double a = al[j], b = a - h2;
            const int i1 = j - 1, i2 = N - 1 - j;
            // a single row is paired with itself (B = A): the two outputs separate
            // exactly, the second is simply not stored
            v[r].x = fma(a, A[i1], b * A[i2]);
            v[r].y = fma(a, B[i1], b * B[i2]);
        }
    }
    __device__ static void first(double2 *buf, double2 (&v)[16], int t, int pr) {
        dft<16>(v);
        double2 *w = buf + 17 * t;   // pad16(16 t + r)
#pragma unroll
        for (int r = 0; r < 16; ++r) w[r] = v[r];
        rsync<T>(pr);
    }
    __device__ static void mid(double2 *buf, const double2 *m16, int t, int pr) {
        constexpr int RS_ = T + T / 16;
        double2 v[16];
        const double2 *rd = buf + xi(t);
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = rd[r * RS_];
        const int jm = t & 15;
        const double2 w = m16[jm];
        rsync<T>(pr);
        apply_powers<16>(v, w);
        dft<16>(v);
        double2 *wr = buf + xi((t >> 4) * 256 + jm);
#pragma unroll
        for (int r = 0; r < 16; ++r) wr[r * 17] = v[r];
        rsync<T>(pr);
    }
    // last pass, in place: output o = j + r NB lands where its input was read
    __device__ static void last(double2 *buf, const double2 *la, int t, int pr) {
        constexpr int RS_ = NB + NB / 16, US = T + T / 16;
        double2 v[PER][RL];
        double2 *rd = buf + xi(t);
#pragma unroll
        for (int u = 0; u < PER; ++u)
#pragma unroll
            for (int r = 0; r < RL; ++r) v[u][r] = rd[u * US + r * RS_];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            apply_powers<RL>(v[u], la[t + u * T]);
            dft<RL>(v[u]);
        }
#pragma unroll
        for (int u = 0; u < PER; ++u)
#pragma unroll
            for (int r = 0; r < RL; ++r) rd[u * US + r * RS_] = v[u][r];
        rsync<T>(pr);
    }
    // C -> transformed rows (padded X layout) of A (and B when HB)
    __device__ static void post(double2 *buf, double *scr, int t, int pr, int lane, double *XA, double *XB) {
        const bool HB = XB != nullptr;
        double ea[8], eb[8], da[8], db[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = 8 * t + i;
            const double2 c = buf[xi(k)];
            double2 c2 = make_double2(0.0, 0.0);
            if (i > 0 || t > 0) c2 = buf[xi(N - k)];
            ea[i] = c2.y - c.y;
            eb[i] = c.x - c2.x;
            da[i] = c.x + c2.x;
            db[i] = c.y + c2.y;
        }
#pragma unroll
        for (int i = 1; i < 8; ++i) {
            da[i] += da[i - 1];
            db[i] += db[i - 1];
        }
        constexpr int W = T < 32 ? T : 32;
        const unsigned mask = pair_mask<T>(pr);
        double ia = da[7], ib = db[7];
#pragma unroll
        for (int o = 1; o < W; o <<= 1) {
            const double xa = __shfl_up_sync(mask, ia, o, W), xb = __shfl_up_sync(mask, ib, o, W);
            if ((lane & (W - 1)) >= o) {
                ia += xa;
                ib += xb;
            }
        }
        double pa = __shfl_up_sync(mask, ia, 1, W), pb = __shfl_up_sync(mask, ib, 1, W);
        if ((lane & (W - 1)) == 0) {
            pa = 0.0;
            pb = 0.0;
        }
        if constexpr (T > 32) {
            const int w = t >> 5;
            if (lane == 31) {
                scr[(pr * 8 + w) * 2] = ia;
                scr[(pr * 8 + w) * 2 + 1] = ib;
            }
            rsync<T>(pr);
            double sa = 0.0, sb = 0.0;
#pragma unroll
            for (int q = 0; q < T / 32 - 1; ++q)
                if (q < w) {
                    sa += scr[(pr * 8 + q) * 2];
                    sb += scr[(pr * 8 + q) * 2 + 1];
                }
            pa += sa;
            pb += sb;
        } else {
            rsync<T>(pr);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = 8 * t + i;
            if (i > 0 || t > 0) XA[xi(2 * k - 1)] = ea[i];
            XA[xi(2 * k)] = da[i] + pa;
            if (HB) {
                if (i > 0 || t > 0) XB[xi(2 * k - 1)] = eb[i];
                XB[xi(2 * k)] = db[i] + pb;
            }
        }
    }
    // full transform of the staged rows A (, B) -> padded X rows in the same region
#ifndef FD_FFT_INLINE
#define FD_FFT_INLINE __forceinline__
#endif
    __device__ FD_FFT_INLINE static void run(double2 *buf, const double *A, const double *B, const double *al,
                                            double h2, const double2 *m16, const double2 *la, double *scr, int t,
                                            int pr, int lane, double *XA, double *XB,
                                            long long *dbgp = nullptr) {
        double2 v[16];
        auto ck = [&](int s) {   // FD_DBG & 4: per-pass cycle stamps of pair 0 (timing studies)
            if (dbgp && t == 0 && pr == 0) {
                long long c;
                asm volatile("mov.u64 %0, %clock64;" : "=l"(c)::"memory");
                dbgp[s] = c;
            }
        };
        ck(0);
        load(v, A, B, al, h2, t);
        ck(1);
        rsync<T>(pr);   // the staged rows alias the exchange buffer
        first(buf, v, t, pr);
        ck(2);
        if constexpr (C::NMID > 0) mid(buf, m16, t, pr);
        ck(3);
        last(buf, la, t, pr);
        ck(4);
        post(buf, scr, t, pr, lane, XA, XB);
        ck(5);
    }
};

// Transient factors of mode k (modes >= kt, rows i < len): the row-major
// tables hold rows < ecap; beyond them (only when the long-transient table was
// capped) beta is rebuilt bitwise from the last table row with the reference
// recurrence (rectsolver.py:72-73).
static __device__ __noinline__ double beta_rebuild(const PlanDev &p, int k, int i) {
    const double lam = mode_lam(p, k);
    double b = __ldg(p.db + size_t(p.ecap - 1) * p.n + k);
    for (int q = p.ecap; q <= i; ++q) {
        const double d = diag_at(p, lam, q);
        b = __dsub_rn(d, __dmul_rn(p.off, __ddiv_rn(p.off, b)));
    }
    return b;
}
// beta_i for a row of a transient group (0 <= i < m)
__device__ __forceinline__ double beta_tr(const PlanDev &p, int k, int i, int len, double blast, double binf) {
    if (i == p.m - 1) return blast;
    if (i >= len) return binf;
    if (i < p.ecap) return __ldg(p.db + size_t(i) * p.n + k);
    return beta_rebuild(p, k, i);
}
// Factors of row i of mode k (k >= kt) for rows beyond the row-major tables
// (only when the long-transient table was capped): l_i, 1/beta_i, beta_{i-1}.
static __device__ __noinline__ void factors_slow(const PlanDev &p, int k, int i, int len, double l_inf, double ib_inf,
                                          double ib_last, double b_inf, double *l, double *ib, double *bm1) {
    if (i >= len) {
        *l = l_inf;
        *ib = (i == p.m - 1) ? ib_last : ib_inf;
        *bm1 = (i - 1 < len) ? beta_tr(p, k, i - 1, len, 0.0, b_inf) : b_inf;
        return;
    }
    const double bp = (i == 0) ? 0.0 : beta_tr(p, k, i - 1, len, 0.0, b_inf);
    const double d = diag_at(p, mode_lam(p, k), i);
    const double li = (i == 0) ? 0.0 : __ddiv_rn(p.off, bp);
    *l = li;
    *ib = 1.0 / ((i == 0) ? d : __dsub_rn(d, __dmul_rn(p.off, li)));
    *bm1 = bp;
}


// --- tensor memory (TMEM) as per-thread row storage ------------------------------
// 512 columns x 128 lanes x 32 bit per SM.  A warp may only touch the 32 lanes
// of its quarter (warp % 4); tcgen05.ld/st of shape 32x32b move N consecutive
// 32-bit columns of the thread's own lane.  The solve uses it as private
// storage for the phase-1 yhat values a thread needs again in phase 3.
__device__ __forceinline__ void tmem_alloc512(uint32_t *dst) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(dst))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc512(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// two doubles -> 4 columns of this thread's lane (warp-collective)
__device__ __forceinline__ void tmem_st2(uint32_t taddr, double a, double b) {
    const unsigned long long ua = __double_as_longlong(a), ub = __double_as_longlong(b);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
                 "r"(uint32_t(ua)), "r"(uint32_t(ua >> 32)), "r"(uint32_t(ub)), "r"(uint32_t(ub >> 32))
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, double &a, double &b) {
    uint32_t r0, r1, r2, r3;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    a = __longlong_as_double((long long)(((unsigned long long)r1 << 32) | r0));
    b = __longlong_as_double((long long)(((unsigned long long)r3 << 32) | r2));
}

// eight doubles <-> 16 consecutive columns of this thread's lane (warp-collective).
// The sweeps of the long transforms (>= 4 modes per thread) keep each mode's
// recurrence state and fixed-point factors in one such slot, so nothing of it
// occupies registers (or spills) across the transforms.
__device__ __forceinline__ void tmem_ld8d(uint32_t taddr, double (&d)[8]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
    // the registers are valid only after the wait: tie them to it
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
                 :
                 : "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = __hiloint2double(int(r[2 * i + 1]), int(r[2 * i]));
}
__device__ __forceinline__ void tmem_st8d(uint32_t taddr, const double (&d)[8]) {
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        r[2 * i] = uint32_t(__double2loint(d[i]));
        r[2 * i + 1] = uint32_t(__double2hiint(d[i]));
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

// Phase 2 of the persistent solves: block carries (see rsolve.cu).  All NT
// threads of the CTA; the first cap_bytes of shared memory are scratch.
template <int NT>
__device__ __forceinline__ void carries_phase(const PList &pl, unsigned char *smem_raw, size_t cap_bytes, int tid,
                                              int lane) {
    const int n = pl.n;
    // ===================== phase 2: block carries =====================================
    // Per (job, mode) chain over the job's blocks b:
    //   Y_b = yhat_b + P_b Y_{b-1}                  (forward)
    //   X_b = F_b + Y_{b-1} xi_b + Q_b X_{b+1}      (backward)
    // Items of (job, W modes), W ~ chains / grid so every CTA takes about one: the
    // item's block scalars are staged in shared memory (coalesced over modes), then
    // every warp evaluates chains as inclusive scans of the composed affine maps
    // y -> A y + B over 32 blocks at a time (lane = block), and Y, X go back.
    {
        const int warp = tid >> 5;
        constexpr int NW = NT / 32;
        const size_t bs = size_t(kCarryVals) * n;
        int nbmax = 1;
        for (int j = 0; j < pl.count; ++j) nbmax = max(nbmax, pl.job[j].nblk);
        const int cap = int(cap_bytes / (7 * 8)) / nbmax;   // modes per item that fit the regions
        const int cpj = max(1, int(gridDim.x) / pl.count);   // CTAs per job
        int W = (n + cpj - 1) / cpj;
        W = max(1, min(min(W, 64), cap - 1));
        const int WP = W | 1;                               // odd stride: lane-per-block reads conflict-free
        const int per_job = (n + W - 1) / W;
        double *sv = reinterpret_cast<double *>(smem_raw);   // [nb][7][WP]
        auto scan = [&](double &A, double &B) {   // lane l ends with f_l o ... o f_0
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double Ao = __shfl_up_sync(0xffffffffu, A, o), Bo = __shfl_up_sync(0xffffffffu, B, o);
                if (lane >= o) {
                    B = fma(A, Bo, B);
                    A *= Ao;
                }
            }
        };
            for (int item = blockIdx.x; item < pl.count * per_job; item += gridDim.x) {
            const PJob &J = pl.job[item / per_job];
            const int k0 = (item % per_job) * W, w = min(W, n - k0);
            double *cb = pl.carry + size_t(J.blk_base) * bs + k0;
            const int nb = J.nblk;
            // async copies global -> shared (no register round trip): every load of
            // the item in flight at once from a small loop
#pragma unroll 1
            for (int bv = warp; bv < nb * 5; bv += NW) {
                const int b = bv / 5, v = bv - 5 * b;
                const double *src = cb + b * bs + v * n;
                double *dst = sv + (b * 7 + v) * WP;
#pragma unroll 1
                for (int m = lane; m < w; m += 32)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst + m)), "l"(src + m)
                                 : "memory");
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads();
#pragma unroll 1
            for (int m = warp; m < w; m += NW) {
                double carry = 0.0;
#pragma unroll 1
                for (int b0 = 0; b0 < nb; b0 += 32) {
                    const int b = b0 + lane;
                    double A = 1.0, B = 0.0;
                    if (b < nb) {
                        B = sv[(b * 7 + 0) * WP + m];
                        A = (b == 0) ? 0.0 : sv[(b * 7 + 2) * WP + m];
                    }
                    scan(A, B);
                    const double Y = fma(A, carry, B);
                    if (b < nb) sv[(b * 7 + 5) * WP + m] = Y;
                    carry = __shfl_sync(0xffffffffu, Y, 31);
                }
                __syncwarp();
                carry = 0.0;
#pragma unroll 1
                for (int b1 = nb; b1 > 0; b1 -= 32) {
                    const int b = b1 - 1 - lane;   // lane 0 = highest block of the chunk
                    double A = 1.0, B = 0.0;
                    if (b >= 0) {
                        B = sv[(b * 7 + 1) * WP + m];
                        if (b > 0) B = fma(sv[((b - 1) * 7 + 5) * WP + m], sv[(b * 7 + 3) * WP + m], B);
                        A = (b < nb - 1) ? sv[(b * 7 + 4) * WP + m] : 0.0;
                    }
                    scan(A, B);
                    const double X = fma(A, carry, B);
                    if (b >= 0) sv[(b * 7 + 6) * WP + m] = X;
                    carry = __shfl_sync(0xffffffffu, X, 31);
                }
            }
            __syncthreads();
#pragma unroll 1
            for (int bv = warp; bv < nb * 2; bv += NW) {
                const int b = bv >> 1, v = 5 + (bv & 1);
#pragma unroll 1
                for (int m = lane; m < w; m += 32) __stcg(cb + b * bs + v * n + m, sv[(b * 7 + v) * WP + m]);
            }
            __syncthreads();
        }
    }
}

}  // namespace fd
