// Warp-specialised persistent fused rectangle solve, real-symmetric DST-I
// (N = n + 1 = 1024: the BASELINE config-1 shape n = 1023).  OPT-IN
// (FD_RSWS=1); the lockstep kernel (rsolve.cu) is the default because it is
// faster on B200 -- this file records the measured alternative.
//
// Same three phases and arithmetic as rsolve.cu (DST + local forward
// elimination | block carries | back-substitution + inverse DST), but the CTA
// is split into two teams that work on different row pairs at the same time
// instead of in lockstep over row groups:
//
//   FFT team   (NF threads = PF pair teams of T = N/16 threads): pair team q
//              takes row pairs j = q, q + PF, ... of the CTA's sequence and
//              transforms them in place in shared-memory region j mod R.
//   sweep team (NS threads, MPT modes each, state in registers): walks the
//              pairs strictly in row order (phase 1 ascending: local forward
//              elimination, yhat to HBM; phase 3 descending: carry fix-up +
//              back-substitution in place before the inverse DST).
//
// R regions of (N + N/16) complex (+ the pair's slice of the long-transient
// factor table) cycle through TMA load -> FFT -> sweep (phase 1) or TMA load
// -> sweep -> FFT + store (phase 3), handed over with one mbarrier per region
// and stage.
//
// Measured on B200 at c1 (5 x 1023^2, apply time): lockstep 101 us (89 us
// after this round's register work); teams of 256 + 256 threads 136 us with
// the long-transient factors read from L2 per row, 122 us with them staged per
// region by TMA (this file's configuration): the FFT team finishes phase 1 at
// 44 us, the sweep team at 60 us, and the kernel executes 50 M warp
// instructions against the lockstep kernel's 34 M (per-pair bookkeeping, two
// copies of the row loop); 384 + 128 threads 367 us (8 modes per sweep thread
// spill).  The lockstep
// kernel's components add up (load 11 + FFT 15 + sweep 13 us in phase 1) but
// each runs on all 16 warps; with 16 warps per SM (128 registers per thread)
// there is no spare team to overlap them with.
#include "rsolve_common.cuh"

namespace fd {

template <int NL>
struct WS {
    static constexpr int N = 1 << NL;
    static constexpr int T = N / 16;       // FFT threads per pair team
    static constexpr int NF = 256;         // FFT team (8 warps)
    static constexpr int PF = NF / T;      // pair teams
    static constexpr int NS = 256;         // sweep team (8 warps)
    static constexpr int NT = NF + NS;
    static constexpr int R = 2 * (256 / T);   // shared-memory regions (row pairs in flight)
    static constexpr int MPT = (N - 1 + NS - 1) / NS;
    static constexpr int PADN = N + N / 16;
    static constexpr int XR = (N - 1) + ((N - 2) >> 4);
    static constexpr int KTS = 128;        // long-transient modes staged per pair (kt <= KTS)
    static constexpr size_t REG = size_t(PADN) * 16;
    static constexpr size_t LSLOT = size_t(2) * 3 * KTS * 8;
    static constexpr size_t OFF_LT = size_t(R) * REG;     // per-region slice of the lt table
    static constexpr size_t OFF_TW = OFF_LT + size_t(R) * LSLOT;   // m16[16], la[256]
    static constexpr size_t OFF_AL = OFF_TW + 272 * 16;   // alpha[N]
    static constexpr size_t OFF_SC = OFF_AL + size_t(N) * 8;
    static constexpr size_t SMEM = OFF_SC + size_t(PF) * 16 * 8;
    static constexpr int SWEEP_BAR = 15;
    static_assert(PF <= 14 || T <= 32, "named barriers 1..PF for the pair teams");
    static_assert(SMEM <= 225 * 1024, "shared memory");
};

__device__ __forceinline__ void mbar_arrive1(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int NL>
__global__ void __launch_bounds__(WS<NL>::NT, 1) rsws_kernel(const __grid_constant__ PList pl) {
    using C = WS<NL>;
    using F = RFft<NL>;
    constexpr int T = C::T, PF = C::PF, R = C::R, MPT = C::MPT, XR = C::XR, NS = C::NS, NF = C::NF;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    auto regd = [&](int q) { return reinterpret_cast<double *>(smem_raw + size_t(q) * C::REG); };
    auto regc = [&](int q) { return reinterpret_cast<double2 *>(smem_raw + size_t(q) * C::REG); };
    double2 *m16 = reinterpret_cast<double2 *>(smem_raw + C::OFF_TW);
    double2 *la = m16 + 16;
    double *al = reinterpret_cast<double *>(smem_raw + C::OFF_AL);
    double *scr = reinterpret_cast<double *>(smem_raw + C::OFF_SC);
    auto lslot = [&](int q) { return reinterpret_cast<double *>(smem_raw + C::OFF_LT + size_t(q) * C::LSLOT); };
    __shared__ __align__(8) uint64_t bload[R], bfft[R], bsw[R];
    __shared__ Seg segs[kMaxSegs];
    __shared__ int pstart[kMaxSegs + 1];
    __shared__ int nseg_s;

    const int tid = threadIdx.x, lane = tid & 31;
    const int n = pl.n;
    cg::grid_group grid = cg::this_grid();
    auto stamp = [&](int slot) {
        if (pl.tstamp && tid == 0) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
            pl.tstamp[blockIdx.x * 8 + slot] = g;
        }
    };
    stamp(0);
    if (tid == 0) {
        int ns = 0, pairs = 0;
        for (int v = blockIdx.x; v < pl.V; v += gridDim.x) {
            const long long lo = pl.vstart[v], hi = pl.vstart[v + 1];
            for (int j = 0; j < pl.count; ++j) {
                const long long r0 = pl.job[j].row0, r1 = r0 + pl.job[j].p.m;
                if (r0 < hi && r1 > lo && ns < kMaxSegs) {
                    Seg sg;
                    sg.job = j;
                    sg.s = int(max(lo, r0) - r0);
                    sg.e = int(min(hi, r1) - r0) - 1;
                    sg.blk = pl.job[j].blk_base + (v - pl.job[j].c_first);
                    sg.ngroups = (sg.e - sg.s + 2) / 2;   // row pairs
                    sg.item0 = pairs;
                    pstart[ns] = pairs;
                    pairs += sg.ngroups;
                    segs[ns++] = sg;
                }
            }
        }
        pstart[ns] = pairs;
        nseg_s = ns;
        for (int q = 0; q < R; ++q) {
            mbar_init(&bload[q], 1);
            mbar_init(&bfft[q], T);
            mbar_init(&bsw[q], NS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    {
        constexpr int N = C::N;
        const double2 *tw = pl.job[0].p.tw;   // e^{-2 pi i q / 2N}
        const double *ra = pl.job[0].p.ralpha;
        for (int q = tid; q < 16; q += C::NT) m16[q] = __ldg(tw + q * (N / 128));
        for (int q = tid; q < F::NB; q += C::NT) la[q] = __ldg(tw + 2 * q);
        for (int q = tid; q < N; q += C::NT) al[q] = __ldg(ra + q);
    }
    __syncthreads();
    const int nseg = nseg_s, npairs = pstart[nseg_s];

    // pair ja (ascending order) -> segment, first row, rows (1 or 2)
    auto pair_of = [&](int ja, int &si, int &i0, int &rp) {
        si = 0;
        while (si + 1 < nseg && ja >= pstart[si + 1]) ++si;
        i0 = segs[si].s + 2 * (ja - pstart[si]);
        rp = min(2, segs[si].e - i0 + 1);
    };
    // rows [i0, i0 + rp) of base -> region q (lands at offset stg_off); a copy
    // ending at the end of the array leaves an 8-byte tail (see fix_tail)
    // plus the pair's rows of the long-transient factor table (modes < kt)
    auto issue = [&](int q, const double *base, int i0, int rp, const PlanDev &p) {
        const uintptr_t start = reinterpret_cast<uintptr_t>(base + size_t(i0) * n);
        const uintptr_t end = start + uintptr_t(rp) * n * sizeof(double);
        const uintptr_t a = start & ~uintptr_t(15);
        const uintptr_t e = (i0 + rp >= p.m) ? (end & ~uintptr_t(15)) : ((end + 15) & ~uintptr_t(15));
        const uint32_t lb = p.lt ? uint32_t(rp) * 3u * uint32_t(p.ktp) * 8u : 0u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bload[q], uint32_t(e - a) + lb);
        tma_load_1d(regd(q), reinterpret_cast<const void *>(a), uint32_t(e - a), &bload[q]);
        if (lb) tma_load_1d(lslot(q), p.lt + size_t(i0) * 3 * p.ktp, lb, &bload[q]);
    };
    auto tail_of = [&](const double *base, int i0, int rp, int m, int &idx) {   // -> address or null
        const uintptr_t start = reinterpret_cast<uintptr_t>(base + size_t(i0) * n);
        const uintptr_t end = start + uintptr_t(rp) * n * sizeof(double);
        if (i0 + rp < m || !(end & 15)) return (const double *)nullptr;
        idx = int(((end - 8) - (start & ~uintptr_t(15))) / 8);
        return reinterpret_cast<const double *>(end - 8);
    };

    // ===================== phase 1: DST + local forward elimination ===================
    if (tid == 0) {
        for (int ja = 0; ja < min(R, npairs); ++ja) {
            int si, i0, rp;
            pair_of(ja, si, i0, rp);
            const PJob &J = pl.job[segs[si].job];
            issue(ja % R, J.in, i0, rp, J.p);
        }
    }
    if (tid < NF) {
        const int q = tid / T, t = tid % T;
#pragma unroll 1
        for (int ja = q; ja < npairs; ja += PF) {
            const int r = ja % R;
            int si, i0, rp;
            pair_of(ja, si, i0, rp);
            const PJob &J = pl.job[segs[si].job];
            mbar_wait(&bload[r], (ja / R) & 1);
            int tix;
            const double *tp = tail_of(J.in, i0, rp, J.p.m, tix);
            if (tp) {
                if (t == 0) regd(r)[tix] = __ldcg(tp);
                rsync<T>(q);
            }
            double *base = regd(r) + stg_off(J.in, i0, n);
            F::run(regc(r), base, rp > 1 ? base + n : nullptr, al, 0.5 * J.p.scale, m16, la, scr, t, q, lane,
                   regd(r), rp > 1 ? regd(r) + XR : nullptr);
            mbar_arrive1(&bfft[r]);
        }
    } else {
        const int st = tid - NF;
        double ys[MPT], pis[MPT], fss[MPT], s2s[MPT], ccs[MPT];
        double cl[MPT], cib[MPT], cibl[MPT];
        int clen[MPT];
#pragma unroll
        for (int u = 0; u < MPT; ++u) {
            ys[u] = pis[u] = fss[u] = s2s[u] = ccs[u] = cl[u] = cib[u] = cibl[u] = 0.0;
            clen[u] = 0;
        }
#pragma unroll 1
        for (int ja = 0; ja < npairs; ++ja) {
            const int r = ja % R;
            int si, i0, rp;
            pair_of(ja, si, i0, rp);
            const Seg sg = segs[si];
            const PJob &J = pl.job[sg.job];
            const PlanDev &p = J.p;
            const int mlast = p.m - 1, ktp = p.ktp;
            mbar_wait(&bfft[r], (ja / R) & 1);
#pragma unroll 1
            for (int rr = 0; rr < rp; ++rr) {
                const int i = i0 + rr;
                const double *X = regd(r) + (rr ? XR : 0);
                const double *lt_r = lslot(r) + rr * 3 * ktp;
                const bool start = (i == sg.s), endb = (i == sg.e);
                double *og = J.out + size_t(i) * n;
#pragma unroll
                for (int u = 0; u < MPT; ++u) {
                    const int k = st + u * NS;
                    if (k >= n) continue;
                    if (start) {
                        ModeRec c;
                        c.load(p, k);
                        cl[u] = c.l_inf;
                        cib[u] = c.ib_inf;
                        cibl[u] = 1.0 / c.b_last;
                        clen[u] = c.len;
                    }
                    const int len = clen[u];
                    double l = cl[u], ib = (i == mlast) ? cibl[u] : cib[u];
                    if (k < p.kt) {
                        l = lt_r[k];
                        ib = lt_r[ktp + k];
                    } else if (i < len) {
                        if (i < p.ecap) {
                            l = __ldg(p.dl + size_t(i) * n + k);
                            ib = __ldg(p.dib + size_t(i) * n + k);
                        } else {
                            double bm1;
                            factors_slow(p, k, i, len, cl[u], cib[u], cibl[u], 0.0, &l, &ib, &bm1);
                        }
                    }
                    const double xv = X[xi(k)];
                    double y, w, f, s2;
                    if (start) {   // block start: y = r, pi = 1 (rectsolver.py:86 with zero carry-in)
                        y = xv;
                        w = 1.0;
                        f = y * ib;
                        s2 = ib;
                        ccs[u] = (i == 0) ? 0.0 : -l;
                    } else {       // rectsolver.py:86, accumulating the block scalars
                        y = __dsub_rn(xv, __dmul_rn(l, ys[u]));
                        w = -l * pis[u];
                        const double W = w * ib;
                        f = fma(y, W, fss[u]);
                        s2 = fma(w, W, s2s[u]);
                    }
                    og[k] = y;
                    ys[u] = y;
                    pis[u] = w;
                    fss[u] = f;
                    s2s[u] = s2;
                    if (endb) {
                        const int e = i;
                        double lnext = cl[u];
                        if (k < p.kt) lnext = (e + 1 < p.m) ? __ldg(p.lt + size_t(e + 1) * 3 * ktp + k) : 0.0;
                        else if (e + 1 < len && e + 1 < p.ecap) lnext = __ldg(p.dl + size_t(e + 1) * n + k);
                        else if (e + 1 < len) {
                            double ib_, bm1_;
                            factors_slow(p, k, e + 1, len, cl[u], cib[u], cibl[u], 0.0, &lnext, &ib_, &bm1_);
                        }
                        const double Q = (e < p.m - 1) ? w * (-lnext) : 0.0;
                        const double cc = ccs[u];
                        double *cb = pl.carry + size_t(sg.blk) * kCarryVals * n + k;
                        __stcg(cb + 0 * n, y);
                        __stcg(cb + 1 * n, f);
                        __stcg(cb + 2 * n, cc * w);
                        __stcg(cb + 3 * n, cc * s2);
                        __stcg(cb + 4 * n, Q);
                    }
                }
            }
            asm volatile("bar.sync %0, %1;" ::"n"(C::SWEEP_BAR), "n"(NS) : "memory");   // region r consumed
            if (st == 0 && ja + R < npairs) {
                int si2, i2, rp2;
                pair_of(ja + R, si2, i2, rp2);
                const PJob &J2 = pl.job[segs[si2].job];
                issue(r, J2.in, i2, rp2, J2.p);
            }
        }
    }
    stamp(1);
    grid.sync();
    stamp(2);
    carries_phase<C::NT>(pl, smem_raw, C::OFF_TW, tid, lane);
    stamp(3);
    grid.sync();
    stamp(4);

    // ===================== phase 3: back-substitution + inverse DST ===================
    // pairs in descending row order: jd = 0 is the CTA's highest pair
    auto pair_desc = [&](int jd, int &si, int &i0, int &rp) { pair_of(npairs - 1 - jd, si, i0, rp); };
    auto base_par = [&](int r) { return npairs > r ? ((npairs - 1 - r) / R + 1) & 1 : 0; };   // phase-1 loads of r
    if (tid == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        for (int jd = 0; jd < min(R, npairs); ++jd) {
            int si, i0, rp;
            pair_desc(jd, si, i0, rp);
            const PJob &J = pl.job[segs[si].job];
            issue(jd % R, J.out, i0, rp, J.p);
        }
    }
    if (tid >= NF) {
        const int st = tid - NF;
        double xs[MPT], yins[MPT], pcs[MPT];
        double cib_inf[MPT], cinv[MPT], cibl[MPT];
        int clen[MPT];
#pragma unroll
        for (int u = 0; u < MPT; ++u) {
            xs[u] = yins[u] = pcs[u] = cib_inf[u] = cinv[u] = cibl[u] = 0.0;
            clen[u] = 0;
        }
#pragma unroll 1
        for (int jd = 0; jd < npairs; ++jd) {
            const int r = jd % R;
            int si, i0, rp;
            pair_desc(jd, si, i0, rp);
            const Seg sg = segs[si];
            const PJob &J = pl.job[sg.job];
            const PlanDev &p = J.p;
            const double off = p.off, nio = -1.0 / off;
            const int mlast = p.m - 1, ktp = p.ktp;
            const bool has_in = sg.blk > J.blk_base;                 // block does not start at row 0
            const bool has_next = sg.blk < J.blk_base + J.nblk - 1;  // a block below carries X
            mbar_wait(&bload[r], (base_par(r) + jd / R) & 1);
            int tix;
            const double *tp = tail_of(J.out, i0, rp, J.p.m, tix);
            if (tp) {
                if (st == 0) regd(r)[tix] = __ldcg(tp);
                asm volatile("bar.sync %0, %1;" ::"n"(C::SWEEP_BAR), "n"(NS) : "memory");
            }
            double *rows = regd(r) + stg_off(J.out, i0, n);
#pragma unroll 1
            for (int rr = rp - 1; rr >= 0; --rr) {
                const int i = i0 + rr;
                const bool top = (i == sg.e);
                double *yr = rows + rr * n;
                const double *lt_r = lslot(r) + rr * 3 * ktp;
#pragma unroll
                for (int u = 0; u < MPT; ++u) {
                    const int k = st + u * NS;
                    if (k >= n) continue;
                    if (top) {
                        ModeRec c;
                        c.load(p, k);
                        cib_inf[u] = c.ib_inf;
                        cinv[u] = c.inv_nl;
                        cibl[u] = 1.0 / c.b_last;
                        clen[u] = c.len;
                        const double *cb = pl.carry + size_t(sg.blk) * kCarryVals * n + k;
                        const size_t bs = size_t(kCarryVals) * n;
                        xs[u] = has_next ? __ldcg(cb + bs + 6 * n) : 0.0;
                        yins[u] = has_in ? __ldcg(cb - bs + 5 * n) : 0.0;
                        pcs[u] = __ldcg(cb + 2 * n);
                    }
                    const int len = clen[u];
                    double ib = (i == mlast) ? cibl[u] : cib_inf[u], pm = cinv[u];
                    if (k < p.kt) {
                        ib = lt_r[ktp + k];
                        pm = lt_r[2 * ktp + k];   // -beta_{i-1} / delta
                    } else if (i < len) {
                        if (i < p.ecap) {
                            ib = __ldg(p.dib + size_t(i) * n + k);
                            pm = (i >= 1) ? __ldg(p.db + size_t(i - 1) * n + k) * nio : cinv[u];
                        } else {
                            double l, bm1;
                            factors_slow(p, k, i, len, 0.0, cib_inf[u], cibl[u], mode_binf(p, k), &l, &ib, &bm1);
                            pm = bm1 * nio;
                        }
                    }
                    double y = yr[k], Pc = pcs[u];
                    if (has_in) {
                        y = fma(Pc, yins[u], y);
                        pcs[u] = Pc * pm;   // P_{i-1} = P_i / (-l_i)
                    }
                    const double x = __dsub_rn(y, __dmul_rn(off, xs[u])) * ib;   // rectsolver.py:90
                    yr[k] = x;
                    xs[u] = x;
                }
            }
            mbar_arrive1(&bsw[r]);
        }
    } else {
        const int q = tid / T, t = tid % T;
#pragma unroll 1
        for (int jd = q; jd < npairs; jd += PF) {
            const int r = jd % R;
            int si, i0, rp;
            pair_desc(jd, si, i0, rp);
            const PJob &J = pl.job[segs[si].job];
            const PlanDev &p = J.p;
            mbar_wait(&bsw[r], (jd / R) & 1);
            double *base = regd(r) + stg_off(J.out, i0, n);
            double *XA = regd(r), *XB = regd(r) + XR;
            F::run(regc(r), base, rp > 1 ? base + n : nullptr, al, 0.5 * p.scale, m16, la, scr, t, q, lane, XA,
                   rp > 1 ? XB : nullptr);
            rsync<T>(q);
            // epilogue out = alpha x + beta other over the pair's rows (adjacent in HBM)
            const double al_ = J.alpha, be_ = J.beta;
            double *o0 = J.out + size_t(i0) * n;
            const double *q0p = J.other ? J.other + size_t(i0) * n : nullptr;
            const int tot = rp * n;
#pragma unroll 1
            for (int q0 = t; q0 < tot; q0 += 8 * T) {
                double v[8], w8[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int qq = q0 + u * T, h = qq >= n;
                    v[u] = (qq < tot) ? XA[h * XR + xi(qq - h * n)] : 0.0;
                    w8[u] = (qq < tot && q0p) ? __ldg(q0p + qq) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int qq = q0 + u * T;
                    if (qq < tot) o0[qq] = q0p ? fma(be_, w8[u], al_ * v[u]) : al_ * v[u];
                }
            }
            rsync<T>(q);   // region free
            if (t == 0 && jd + R < npairs) {
                int si2, i2, rp2;
                pair_desc(jd + R, si2, i2, rp2);
                const PJob &J2 = pl.job[segs[si2].job];
                issue(r, J2.out, i2, rp2, J2.p);
            }
        }
    }
    stamp(5);
}

template <int NL>
struct RwsK {
    static constexpr int NT = WS<NL>::NT, G = 2;
    static constexpr size_t SMEM = WS<NL>::SMEM;
    static const void *fn() { return (const void *)rsws_kernel<NL>; }
};

bool launch_rsws(const std::vector<SolveJob> &jobs, cudaStream_t s, Workspace &ws) {
    static const int mode = getenv("FD_RSWS") ? atoi(getenv("FD_RSWS")) : 0;   // opt-in (see header)
    const int n = jobs[0].p.n;
    if (!mode || !rs_supported(n) || !jobs[0].p.ralpha) return false;
    for (const auto &j : jobs)
        if (j.p.kt > 128) return false;   // long-transient slice must fit the per-region slot
    switch (n + 1) {
        case 1024: run_persist<RwsK<10>>(jobs, s, ws); return true;
        default: return false;
    }
}

}  // namespace fd
