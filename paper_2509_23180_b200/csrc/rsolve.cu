// Persistent fused rectangle solve with a real-symmetric DST-I
// (n + 1 = N = 2^NL, 256 <= N <= 4096).
//
// Three phases in one cooperative launch (DST + local forward elimination |
// block carries | back-substitution + inverse DST); the transform of a row pair
// is ONE N-point complex FFT instead of a 2N-point FFT of the odd extension:
//
//   y_j = alpha_j x_j + (alpha_j - s/2) x_{N-j},  alpha_j = s/2 sin(pi j/N) + s/4
//   c   = y_a + i y_b,  C = FFT_N(c)
//   X_{2k}   = -(Im C_k - Im C_{N-k})      (row a),   Re C_k - Re C_{N-k}   (row b)
//   X_{2k+1} = X_{2k-1} + Re C_k + Re C_{N-k} (row a), ... Im (row b),  X_1 = Re C_0
//
// (s = sqrt(2/N) the orthonormal factor; the odd outputs are a prefix sum over
// k, done per pair with a serial/warp-shuffle/cross-warp scan).  This halves the
// fp64 work of the transform, which bounds the complex-FFT kernel.
//
// One CTA per SM (512 threads; 576 = nine row pairs at N = 1024, see fd_internal.h).
// Shared memory:
//   P pair regions of (N + N/16) complex: a row pair is TMA-copied into its
//   region (unpadded, at offset so in {0,1}), transformed in place (padded
//   Stockham radix-16 passes, pad16(q) = q + q/16), and the transformed rows
//   are written back padded (xi(q) = q + q/16) for the mode-parallel Thomas
//   sweep; phase 3 runs the sweep in place on the staged yhat rows first.
//   Every pair has its own mbarrier, so a pair starts transforming as soon as
//   its rows have landed.  The rest holds the transform tables and one group's
//   slice of the slow-mode factor tables (wide before PlanDev::lt_need, one
//   warp's 32 modes after it).
// Tensor memory (N >= 1024): the CTA owns the SM's 512 columns; every thread
//   keeps the recurrence state and fixed-point factors of each of its modes in a
//   16-column slot of its lane (tcgen05.ld/st), so the sweeps hold nothing in
//   registers across the transforms and their body exists once per kernel.
#include "rsolve_common.cuh"

// FD_DIAG=1 (build flag) compiles in the per-item trace and the FD_DBG
// component-skip bits used by the timing studies in DESIGN.md; off by default
// so the production kernel carries no diagnostic code.
// unroll factor of the per-mode loops of the tensor-memory sweeps (>= 4 modes per
// thread): 1 keeps one copy of the sweep body in the instruction stream
#ifndef FD_TM_MIN_MPT
#define FD_TM_MIN_MPT 2
#endif
#ifndef FD_TM_UNROLL
#define FD_TM_UNROLL 1
#endif
#ifndef FD_DIAG
#define FD_DIAG 0
#endif

namespace fd {

template <int NL>
__global__ void __launch_bounds__(RS<NL>::NT, RS<NL>::NT <= 256 ? 2 : 1) rsolve_kernel(const __grid_constant__ PList pl) {
    using C = RS<NL>;
    using F = RFft<NL>;
    constexpr int NT = C::NT, G = C::G, P = C::P, T = C::T, MPT = C::MPT, XR = C::XR;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    auto regd = [&](int q) { return reinterpret_cast<double *>(smem_raw + size_t(q) * C::REG); };
    auto regc = [&](int q) { return reinterpret_cast<double2 *>(smem_raw + size_t(q) * C::REG); };
    double2 *m16 = reinterpret_cast<double2 *>(smem_raw + C::OFF_TW);
    double2 *la = m16 + 16;
    double *al = reinterpret_cast<double *>(smem_raw + C::OFF_AL);
    double *scr = reinterpret_cast<double *>(smem_raw + C::OFF_SC);
    double *lts = reinterpret_cast<double *>(smem_raw + C::OFF_LT);   // [G][3][ktp]
    __shared__ __align__(8) uint64_t pbar[P];
    __shared__ __align__(8) uint64_t ltbar;
    __shared__ Seg segs[kMaxSegs];
    __shared__ int nseg_s, nitems_s;
    // >= 4 modes per thread (N >= 2048): the sweeps' per-mode state and factors live
    // in tensor memory between the row groups (one CTA per SM owns all 512 columns)
    constexpr bool kTm = MPT >= FD_TM_MIN_MPT;
    constexpr int kTmUnroll = FD_TM_UNROLL;
    __shared__ uint32_t tmem_base_s;

    const int tid = threadIdx.x, lane = tid & 31;
    const int n = pl.n;
    const int pr = tid / T, t = tid % T;
    cg::grid_group grid = cg::this_grid();
    auto stamp = [&](int slot) {
        if (pl.tstamp && tid == 0) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
            pl.tstamp[blockIdx.x * 8 + slot] = g;
        }
    };
    auto trace = [&](int role, int item, int which) {   // FD_TRACE=<cta>
        if (FD_DIAG && pl.trace && (role >= 8 ? t == 0 : tid == 0) && blockIdx.x == pl.trace_cta && item < 64 &&
            role < 16) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g)::"memory");
            pl.trace[(role * 64 + item) * 2 + which] = g;
        }
    };
    stamp(0);
    if (pl.tstamp && tid == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        pl.tstamp[blockIdx.x * 8 + 6] = smid;
    }

    if (tid == 0) {
        int ns = 0, items = 0;
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
                    sg.ngroups = (sg.e - sg.s + G) / G;
                    sg.item0 = items;
                    items += sg.ngroups;
                    segs[ns++] = sg;
                }
            }
        }
        nseg_s = ns;
        nitems_s = items;
        for (int q = 0; q < P; ++q) mbar_init(&pbar[q], 1);
        mbar_init(&ltbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    {
        constexpr int N = C::N;
        const double2 *tw = pl.job[0].p.tw;   // e^{-2 pi i q / 2N}
        const double *ra = pl.job[0].p.ralpha;
        for (int q = tid; q < 16; q += NT) m16[q] = __ldg(tw + q * (N / 128));
        for (int q = tid; q < C::NB; q += NT) la[q] = __ldg(tw + 2 * q);
        for (int q = tid; q < N; q += NT) al[q] = __ldg(ra + q);
    }
    if constexpr (kTm) {
        if (tid < 32) tmem_alloc512(&tmem_base_s);
        tmem_fence_before();
    }
    __syncthreads();
    uint32_t tm = 0;   // this thread's slots: lane quarter of its warp, 128 columns per warp
    if constexpr (kTm) {
        tmem_fence_after();
        tm = tmem_base_s + ((uint32_t(tid >> 5) & 3u) << 21) + uint32_t(tid >> 7) * uint32_t(16 * MPT);
    }
    const int nseg = nseg_s, nitems = nitems_s;
    uint32_t ppar = 0, ltpar = 0;

    auto item_of = [&](int it, int &si, int &g0, int &rows, bool desc) {
        si = 0;
        while (si + 1 < nseg && it >= segs[si + 1].item0) ++si;
        const Seg &sg = segs[si];
        const int gi = it - sg.item0;
        const int gg = desc ? (sg.ngroups - 1 - gi) : gi;
        g0 = sg.s + gg * G;
        rows = min(G, sg.e - g0 + 1);
    };
    auto group_mask = [&](int rows) {   // pairs holding rows of the group
        const int np = (rows + 1) >> 1;
        return np >= 32 ? 0xffffffffu : ((1u << np) - 1u);
    };
    // this pair's rows [g0 + 2 pr, +rp) of base -> its region (lands at offset so)
    auto issue_pair = [&](const double *base, int g0, int rows, int m) {
        Tail tl{0.0, -1};
        const int r0 = 2 * pr, rp = min(2, rows - r0);
        if (rp <= 0) return tl;
        const uintptr_t start = reinterpret_cast<uintptr_t>(base + size_t(g0 + r0) * n);
        const uintptr_t end = start + uintptr_t(rp) * n * sizeof(double);
        const uintptr_t a = start & ~uintptr_t(15);
        const uintptr_t e = (g0 + r0 + rp >= m) ? (end & ~uintptr_t(15)) : ((end + 15) & ~uintptr_t(15));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&pbar[pr], uint32_t(e - a));
        tma_load_1d(regd(pr), reinterpret_cast<const void *>(a), uint32_t(e - a), &pbar[pr]);
        if (end != e) {
            tl.v = __ldcg(reinterpret_cast<const double *>(e));
            tl.idx = int((e - a) / 8);
        }
        return tl;
    };
    // slow-mode factor slice of a group: all kt modes before row lt_need, the
    // first kta (one warp's) after it, where every other mode is on its fixed point
    auto issue_lts = [&](const PlanDev &p, int g0, int rows) {
        const bool wide = g0 < p.lt_need;
        const int pitch = wide ? p.ktp : p.ktpa;
        const uint32_t bytes = uint32_t(rows) * 3u * uint32_t(pitch) * 8u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&ltbar, bytes);
        tma_load_1d(lts, (wide ? p.lt : p.lta) + size_t(g0) * 3 * pitch, bytes, &ltbar);
    };
    auto pair_tail = [&](const double *base, int g0, int rows, int m) {
        const int r0 = 2 * pr, rp = min(2, rows - r0);
        if (rp <= 0) return false;
        const uintptr_t end = reinterpret_cast<uintptr_t>(base + size_t(g0 + r0 + rp) * n);
        return (g0 + r0 + rp >= m) && (end & 15);
    };

    // ===================== phase 1: DST + local forward elimination ===================
    {
        constexpr int SR = kTm ? 1 : MPT;   // per-mode state in registers (short transforms)
        double ys[SR], pis[SR], fss[SR], s2s[SR], ccs[SR];
        double cl[SR], cib[SR], cibl[SR];
        int clen[SR];
        Tail tail{0.0, -1};
        if (nitems > 0) {
            int si, g0, rows;
            item_of(0, si, g0, rows, false);
            const PJob &J = pl.job[segs[si].job];
            if (t == 0) tail = issue_pair(J.in, g0, rows, J.p.m);
            if (tid == 0 && J.p.lt) issue_lts(J.p, g0, rows);
        }
#pragma unroll 1
        for (int it = 0; it < nitems; ++it) {
            int si, g0, rows;
            item_of(it, si, g0, rows, false);
            const Seg sg = segs[si];
            const PJob &J = pl.job[sg.job];
            const PlanDev &p = J.p;
            const int so = stg_off(J.in, g0, n);
            const int rp = min(2, rows - 2 * pr);
            // modes read from the staged table slice in this group, and its pitch
            const int ktg = g0 < p.lt_need ? p.kt : p.kta, ktpg = g0 < p.lt_need ? p.ktp : p.ktpa;
            trace(0, it, 0);
            if (rp > 0) {
                mbar_wait(&pbar[pr], (ppar >> pr) & 1u);
                if (pair_tail(J.in, g0, rows, p.m)) {
                    if (t == 0) regd(pr)[tail.idx] = tail.v;
                    rsync<T>(pr);
                }
                double *base = regd(pr) + so;
                if (!(FD_DIAG && (pl.dbg & 8)))
                F::run(regc(pr), base, rp > 1 ? base + n : nullptr, al, 0.5 * p.scale, m16, la, scr, t, pr, lane,
                       regd(pr), rp > 1 ? regd(pr) + XR : nullptr,
                       (FD_DIAG && pl.trace && (pl.dbg & 4) && blockIdx.x == pl.trace_cta && it < 4)
                           ? reinterpret_cast<long long *>(pl.trace) + 2048 + it * 8 : nullptr);
            }
            ppar ^= group_mask(rows);
            if (p.lt) {
                mbar_wait(&ltbar, ltpar);
                ltpar ^= 1u;
            }
            __syncthreads();   // all rows of the group transformed
            trace(0, it, 1);
            auto xrow = [&](int rr) { return regd(rr >> 1) + (rr & 1) * XR; };
            const bool first = (g0 == sg.s), last = (g0 + rows - 1 == sg.e);
            double *outg = J.out + size_t(g0) * n;
            const int mlast = p.m - 1;
            // two parts (rows [0, half), [half, rows)): the first half's regions are
            // refilled with the next group while the second half is swept
            const int half = (rows > 8) ? ((rows / 2 + 1) & ~1) : rows;
#pragma unroll 1
            for (int part = 0; part < 2; ++part) {
            const int ra = part ? half : 0, rb = part ? rows : half;
            // one mode's rows [ra, rb) of the group: local forward elimination and
            // block scalars; the state (y, w, f, s2, cc) lives with the caller
            auto sweep1 = [&](int k, double &y, double &w, double &f, double &s2, double &ccr, double l_inf,
                              double ib_inf, double ibm, int len) {
                const int xk = xi(k);
                double *og = outg + k;
                // one row of the local forward elimination (rectsolver.py:86) with
                // factors (l, 1/beta), accumulating the block scalars
                auto step = [&](int rr, double l, double ib) {
                    y = __dsub_rn(xrow(rr)[xk], __dmul_rn(l, y));
                    w = -l * w;
                    const double W = w * ib;
                    f = fma(y, W, f);
                    s2 = fma(w, W, s2);
                    if (!(FD_DIAG && (pl.dbg & 2))) og[rr * n] = y;
                };
                int rr = ra;
                if (first && ra == 0) {   // block start: y = r, pi = 1, P_i = -l_s pi_i
                    double l0 = l_inf, ib0 = (g0 == mlast) ? ibm : ib_inf;
                    if (k < ktg) {
                        l0 = lts[k];
                        ib0 = lts[ktpg + k];
                    } else if (g0 < len) {
                        if (g0 < p.ecap) {
                            l0 = __ldg(p.dl + size_t(g0) * n + k);
                            ib0 = __ldg(p.dib + size_t(g0) * n + k);
                        } else {
                            double bm1;
                            factors_slow(p, k, g0, len, l_inf, ib_inf, ibm, 0.0, &l0, &ib0, &bm1);
                        }
                    }
                    y = xrow(0)[xk];
                    w = 1.0;
                    f = y * ib0;
                    s2 = ib0;
                    ccr = (g0 == 0) ? 0.0 : -l0;
                    og[0] = y;
                    rr = 1;
                }
                if (k < ktg) {
                    // slowly converging low mode: reference factors from the table
                    const double *tb = lts + k;
#pragma unroll 4
                    for (; rr < rb; ++rr) step(rr, tb[rr * 3 * ktpg], tb[rr * 3 * ktpg + ktpg]);
                } else if (g0 + rr < len && g0 + rb <= p.ecap) {
                    // transient rows: the reference factors (rectsolver.py:72-73) from
                    // the row-major tables, 8 rows of loads ahead of their sweep
#pragma unroll 1
                    for (; rr < rb; rr += 8) {
                        double lv[8], ibv[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const int i = g0 + rr + q;
                            const bool tr = (rr + q < rb) && (i < len);
                            lv[q] = tr ? __ldg(p.dl + size_t(i) * n + k) : l_inf;
                            ibv[q] = tr ? __ldg(p.dib + size_t(i) * n + k) : ((i == mlast) ? ibm : ib_inf);
                        }
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            if (rr + q < rb) step(rr + q, lv[q], ibv[q]);
                    }
                } else if (g0 + rr < len) {
#pragma unroll 1
                    for (; rr < rb; ++rr) {   // beyond the tables (capped long-transient table)
                        double l, ib, bm1;
                        factors_slow(p, k, g0 + rr, len, l_inf, ib_inf, ibm, 0.0, &l, &ib, &bm1);
                        step(rr, l, ib);
                    }
                } else {
                    if (g0 + rb - 1 < mlast) {
#pragma unroll 4
                        for (; rr < rb; ++rr) step(rr, l_inf, ib_inf);
                    } else {
#pragma unroll 1
                        for (; rr < rb; ++rr) step(rr, l_inf, (g0 + rr == mlast) ? ibm : ib_inf);
                    }
                }
                const double cc = ccr;
                if (last && rb == rows) {
                    const int cn = pl.cn;
                    double *cb = pl.carry + size_t(sg.blk) * kCarryVals * cn + k;
                    const int e = sg.e;
                    // Q = pi_e * (-l_{e+1}),  l_{e+1} = delta / beta_e
                    double lnext = l_inf;
                    if (k < p.kt && e + 1 < p.lt_need)
                        lnext = __ldg(p.lt + size_t(e + 1) * 3 * p.ktp + k);
                    else if (k < p.kta)
                        lnext = (e + 1 < p.m) ? __ldg(p.lta + size_t(e + 1) * 3 * p.ktpa + k) : 0.0;
                    else if (k < p.kt)
                        lnext = l_inf;
                    else if (e + 1 < len && e + 1 < p.ecap)
                        lnext = __ldg(p.dl + size_t(e + 1) * n + k);
                    else if (e + 1 < len) {
                        double ib_, bm1_;
                        factors_slow(p, k, e + 1, len, l_inf, ib_inf, ibm, 0.0, &lnext, &ib_, &bm1_);
                    }
                    const double Q = (e < p.m - 1) ? w * (-lnext) : 0.0;
                    __stcg(cb + 0 * cn, y);
                    __stcg(cb + 1 * cn, f);
                    __stcg(cb + 2 * cn, cc * w);
                    __stcg(cb + 3 * cn, cc * s2);
                    __stcg(cb + 4 * cn, Q);
                }
            };
            if constexpr (kTm) {
                // long transforms: a mode's state and fixed-point factors live in one
                // 8-double tensor-memory slot of the thread (y, w, f, s2, cc, l_inf,
                // 1/beta_inf, fixed-point row); the factors are fetched once per
                // segment, every fetch of the thread in flight at once
                if (first && ra == 0) {
                    double2 ca[MPT];
                    double cd[MPT];
#pragma unroll
                    for (int u = 0; u < MPT; ++u) {
                        const double2 *rec = reinterpret_cast<const double2 *>(p.mode) + 4 * min(tid + u * NT, n - 1);
                        ca[u] = __ldg(rec);
                        cd[u] = __ldg(reinterpret_cast<const double *>(rec + 3) + 1);
                    }
#pragma unroll
                    for (int u = 0; u < MPT; ++u) {
                        const double st[8] = {0.0, 0.0, 0.0, 0.0, 0.0, ca[u].x, ca[u].y, cd[u]};
                        tmem_st8d(tm + u * 16, st);
                    }
                    tmem_wait_st();
                }
                if (ra < rb) {
#pragma unroll kTmUnroll
                    for (int u = 0; u < MPT; ++u) {
                        const int k = tid + u * NT;
                        double st[8];
                        __syncwarp();
                        tmem_ld8d(tm + u * 16, st);
                        if (k < n && !(FD_DIAG && (pl.dbg & 16))) {
                            const double ibm = (g0 + rb - 1 >= p.m - 1) ? 1.0 / mode_blast(p, k) : st[6];
                            sweep1(k, st[0], st[1], st[2], st[3], st[4], st[5], st[6], ibm,
                                   int(__double_as_longlong(st[7])));
                        }
                        __syncwarp();
                        tmem_st8d(tm + u * 16, st);
                    }
                    tmem_wait_st();
                }
            } else {
#pragma unroll
                for (int u = 0; u < MPT; ++u) {
                    const int k = tid + u * NT;
                    if (k >= n || ra >= rb || (FD_DIAG && (pl.dbg & 16))) continue;
                    if (first && part == 0) {
                        ModeRec c;
                        c.load(p, k);
                        cl[u] = c.l_inf;
                        cib[u] = c.ib_inf;
                        cibl[u] = 1.0 / c.b_last;
                        clen[u] = c.len;
                    }
                    sweep1(k, ys[u], pis[u], fss[u], s2s[u], ccs[u], cl[u], cib[u], cibl[u], clen[u]);
                }
            }
            __syncthreads();   // this part's rows consumed (after part 1: the table slice too)
            if (it + 1 < nitems) {
                int si2, g2, rows2;
                item_of(it + 1, si2, g2, rows2, false);
                const PJob &J2 = pl.job[segs[si2].job];
                if (t == 0 && (part ? 2 * pr >= half : 2 * pr < half)) tail = issue_pair(J2.in, g2, rows2, J2.p.m);
                if (part == 1 && tid == 0 && J2.p.lt) issue_lts(J2.p, g2, rows2);
            }
            }   // parts
            trace(1, it, 1);
        }
    }
    stamp(1);
    grid.sync();
    stamp(2);
    trace(11, 0, 0);

    // ===================== phase 2: block carries =====================================
    // Per (job, mode) chain over the job's blocks b:
    //   Y_b = yhat_b + P_b Y_{b-1}                  (forward)
    //   X_b = F_b + Y_{b-1} xi_b + Q_b X_{b+1}      (backward)
    // Items of (job, W modes), W ~ chains / grid so every CTA takes about one.  The
    // item's block scalars arrive by 16-byte async copies (the carry rows have an
    // even pitch, so every row of W values starts 16-byte aligned), then one
    // thread per mode walks its chain forward and back -- the jobs have a few
    // dozen blocks, so two serial passes of FMAs over shared memory are shorter
    // than scans of composed maps -- and Y, X go back coalesced.
    {
        const int warp = tid >> 5;
        constexpr int NW = NT / 32;
        const int cn = pl.cn;
        const size_t bs = size_t(kCarryVals) * cn;
        int nbmax = 1;
        for (int j = 0; j < pl.count; ++j) nbmax = max(nbmax, pl.job[j].nblk);
        const int cap = int(C::OFF_TW / (7 * 8)) / nbmax;   // modes per item that fit the regions
        const int cpj = max(1, int(gridDim.x) / pl.count);   // CTAs per job
        int W = (n + cpj - 1) / cpj;
        W = max(2, min(min((W + 1) & ~1, 64), cap & ~1));    // even: rows start 16-byte aligned
        const int per_job = (n + W - 1) / W;
        double *sv = reinterpret_cast<double *>(smem_raw);   // [nb][7][W]
        for (int item = blockIdx.x; item < pl.count * per_job; item += gridDim.x) {
            const PJob &J = pl.job[item / per_job];
            const int k0 = (item % per_job) * W, w = min(W, n - k0);
            double *cb = pl.carry + size_t(J.blk_base) * bs + k0;
            const int nb = J.nblk;
            const uint32_t rb = uint32_t((w + 1) & ~1) * 8u;   // bytes per row (the pitch pads odd n)
            // 16-byte async copies global -> shared, every copy of the item in flight at once
            {
                const int cpr = int(rb / 16);   // chunks per row
                const int total = nb * 5 * cpr;
#pragma unroll 1
                for (int c = tid; c < total; c += NT) {
                    const int bv = c / cpr, q = c - bv * cpr;
                    const int b = bv / 5, v = bv - 5 * b;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sv + (b * 7 + v) * W + 2 * q)),
                                 "l"(cb + b * bs + v * cn + 2 * q)
                                 : "memory");
                }
                asm volatile("cp.async.wait_all;" ::: "memory");
            }
            __syncthreads();
            trace(12, item / gridDim.x, 1);
            if (tid < w) {
                // eight blocks of coefficients are read ahead of each stretch of the
                // dependent chain (the stores in between would otherwise order every
                // load behind the previous link)
                double *c = sv + tid;
                double Y = 0.0;
#pragma unroll 1
                for (int b0 = 0; b0 < nb; b0 += 8) {
                    double A[8], B[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int b = min(b0 + q, nb - 1);
                        A[q] = c[(b * 7 + 2) * W];
                        B[q] = c[(b * 7 + 0) * W];
                    }
                    if (b0 == 0) A[0] = 0.0;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        if (b0 + q < nb) {
                            Y = fma(A[q], Y, B[q]);
                            c[((b0 + q) * 7 + 5) * W] = Y;
                        }
                }
                double X = 0.0;
#pragma unroll 1
                for (int b1 = nb - 1; b1 >= 0; b1 -= 8) {
                    double A[8], B[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int b = max(b1 - q, 0);
                        B[q] = c[(b * 7 + 1) * W];
                        if (b > 0) B[q] = fma(c[((b - 1) * 7 + 5) * W], c[(b * 7 + 3) * W], B[q]);
                        A[q] = (b < nb - 1) ? c[(b * 7 + 4) * W] : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        if (b1 - q >= 0) {
                            X = fma(A[q], X, B[q]);
                            c[((b1 - q) * 7 + 6) * W] = X;
                        }
                }
            }
            trace(13, item / gridDim.x, 0);
            __syncthreads();
            trace(13, item / gridDim.x, 1);
#pragma unroll 1
            for (int bv = warp; bv < nb * 2; bv += NW) {
                const int b = bv >> 1, v = 5 + (bv & 1);
#pragma unroll 1
                for (int m = lane; m < w; m += 32) __stcg(cb + b * bs + v * cn + m, sv[(b * 7 + v) * W + m]);
            }
            __syncthreads();
            trace(14, item / gridDim.x, 0);
        }
    }
    stamp(3);
    grid.sync();
    stamp(4);

    // ===================== phase 3: back-substitution + inverse DST ===================
    {
        constexpr int SR = kTm ? 1 : MPT;
        double xs[SR], yins[SR], pcs[SR];
        double cib_inf[SR], cinv[SR], cibl[SR];
        int clen[SR];
        Tail tail{0.0, -1};
        if (nitems > 0) {
            int si, g0, rows;
            item_of(0, si, g0, rows, true);
            const PJob &J = pl.job[segs[si].job];
            if (t == 0) {
                asm volatile("fence.proxy.async.global;" ::: "memory");
                tail = issue_pair(J.out, g0, rows, J.p.m);
            }
            if (tid == 0 && J.p.lt) issue_lts(J.p, g0, rows);
        }
#pragma unroll 1
        for (int it = 0; it < nitems; ++it) {
            int si, g0, rows;
            item_of(it, si, g0, rows, true);
            const Seg sg = segs[si];
            const PJob &J = pl.job[sg.job];
            const PlanDev &p = J.p;
            const double off = p.off;
            const bool top = (g0 + rows - 1 == sg.e);
            const bool has_in = sg.blk > J.blk_base;                 // block does not start at row 0
            const bool has_next = sg.blk < J.blk_base + J.nblk - 1;  // a block below carries X
            const int so = stg_off(J.out, g0, n);
            const int ktg = g0 < p.lt_need ? p.kt : p.kta, ktpg = g0 < p.lt_need ? p.ktp : p.ktpa;   // see phase 1
            trace(2, it, 0);
            const uint32_t gm = group_mask(rows);
#pragma unroll 1
            for (int q = 0; q < P; ++q)
                if ((gm >> q) & 1u) mbar_wait(&pbar[q], (ppar >> q) & 1u);
            ppar ^= gm;
            if (p.lt) {
                mbar_wait(&ltbar, ltpar);
                ltpar ^= 1u;
            }
            if (has_tail(J.out, g0, rows, n, p.m)) {
                if (t == 0 && tail.idx >= 0) regd(pr)[tail.idx] = tail.v;
                __syncthreads();
            }
            trace(2, it, 1);
            auto yrow = [&](int rr) { return regd(rr >> 1) + so + (rr & 1) * n; };
            // one mode's rows of the group, descending: carry fix-up and
            // back-substitution in place on the staged rows
            auto sweep3 = [&](int k, double &x, double &Pc, double yin, double ib_inf, double inl_, double iblast,
                              int len) {
                if (k < ktg) {
                    const double *tb = lts + k;
#pragma unroll 4
                    for (int rr = rows - 1; rr >= 0; --rr) {
                        double *yp = yrow(rr) + k;
                        double y = *yp;
                        if (has_in) {
                            y = fma(Pc, yin, y);
                            Pc *= tb[rr * 3 * ktpg + 2 * ktpg];   // P_{i-1} = -P_i beta_{i-1} / delta
                        }
                        x = __dsub_rn(y, __dmul_rn(off, x)) * tb[rr * 3 * ktpg + ktpg];   // rectsolver.py:90
                        *yp = x;
                    }
                } else if (g0 < len && g0 + rows <= p.ecap) {
                    // transient rows: reference factors from the row-major tables,
                    // 8 rows of loads ahead of their sweep
                    const double ib_m = iblast, inl = inl_, nio = -1.0 / off;
                    const int mlast = p.m - 1;
#pragma unroll 1
                    for (int r1 = rows; r1 > 0; r1 -= 8) {   // rows r1 - 1, r1 - 2, ... descending
                        double ibv[8], pmv[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const int i = g0 + r1 - 1 - q;
                            const bool in = q < r1;
                            ibv[q] = (in && i < len) ? __ldg(p.dib + size_t(i) * n + k) : ((i == mlast) ? ib_m : ib_inf);
                            pmv[q] = (in && i >= 1 && i - 1 < len) ? __ldg(p.db + size_t(i - 1) * n + k) * nio : inl;
                        }
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            if (q < r1) {
                                double *yp = yrow(r1 - 1 - q) + k;
                                double y = *yp;
                                if (has_in) {
                                    y = fma(Pc, yin, y);
                                    Pc *= pmv[q];   // P_{i-1} = P_i / (-l_i) = -P_i beta_{i-1} / delta
                                }
                                x = __dsub_rn(y, __dmul_rn(off, x)) * ibv[q];   // rectsolver.py:90
                                *yp = x;
                            }
                        }
                    }
                } else if (g0 < len) {
                    const double nio = -1.0 / off;
#pragma unroll 1
                    for (int rr = rows - 1; rr >= 0; --rr) {   // beyond the tables (rare)
                        double l, ib, bm1;
                        factors_slow(p, k, g0 + rr, len, 0.0, ib_inf, iblast, mode_binf(p, k), &l, &ib, &bm1);
                        double *yp = yrow(rr) + k;
                        double y = *yp;
                        if (has_in) {
                            y = fma(Pc, yin, y);
                            Pc *= bm1 * nio;
                        }
                        x = __dsub_rn(y, __dmul_rn(off, x)) * ib;   // rectsolver.py:90
                        *yp = x;
                    }
                } else {
                    const double ib_m = iblast, inl = inl_;
                    const int mlast = p.m - 1;
                    if (has_in && g0 + rows - 1 < mlast) {   // interior rows, carry fix-up
#pragma unroll 4
                        for (int rr = rows - 1; rr >= 0; --rr) {
                            double *yp = yrow(rr) + k;
                            const double y = fma(Pc, yin, *yp);
                            Pc *= inl;
                            x = __dsub_rn(y, __dmul_rn(off, x)) * ib_inf;   // rectsolver.py:90
                            *yp = x;
                        }
                    } else {
#pragma unroll 1
                        for (int rr = rows - 1; rr >= 0; --rr) {
                            double *yp = yrow(rr) + k;
                            double y = *yp;
                            if (has_in) {
                                y = fma(Pc, yin, y);
                                Pc *= inl;
                            }
                            const double ib = (g0 + rr == mlast) ? ib_m : ib_inf;
                            x = __dsub_rn(y, __dmul_rn(off, x)) * ib;   // rectsolver.py:90
                            *yp = x;
                        }
                    }
                }
            };
            if constexpr (kTm) {
                // slot: x, P, Y_in, 1/beta_inf, 1/(-l_inf), fixed-point row (see phase 1)
                if (top) {
                    double cx[MPT], cy[MPT], cp[MPT], cib[MPT], cnl[MPT], cd[MPT];
                    const int cn = pl.cn;
                    const size_t bs = size_t(kCarryVals) * cn;
#pragma unroll
                    for (int u = 0; u < MPT; ++u) {
                        const int k = min(tid + u * NT, n - 1);
                        const double *rec = p.mode + 8 * size_t(k);
                        const double *cb = pl.carry + size_t(sg.blk) * kCarryVals * cn + k;
                        cib[u] = __ldg(rec + 1);
                        cnl[u] = __ldg(rec + 3);
                        cd[u] = __ldg(rec + 7);
                        cx[u] = has_next ? __ldcg(cb + bs + 6 * cn) : 0.0;
                        cy[u] = has_in ? __ldcg(cb - bs + 5 * cn) : 0.0;
                        cp[u] = __ldcg(cb + 2 * cn);
                    }
#pragma unroll
                    for (int u = 0; u < MPT; ++u) {
                        const double st[8] = {cx[u], cp[u], cy[u], cib[u], cnl[u], cd[u], 0.0, 0.0};
                        tmem_st8d(tm + u * 16, st);
                    }
                    tmem_wait_st();
                }
#pragma unroll kTmUnroll
                for (int u = 0; u < MPT; ++u) {
                    const int k = tid + u * NT;
                    double st[8];
                    __syncwarp();
                    tmem_ld8d(tm + u * 16, st);
                    if (k < n && !(FD_DIAG && (pl.dbg & 64))) {
                        const double iblast = (g0 + rows - 1 >= p.m - 1) ? 1.0 / mode_blast(p, k) : st[3];
                        sweep3(k, st[0], st[1], st[2], st[3], st[4], iblast, int(__double_as_longlong(st[5])));
                    }
                    __syncwarp();
                    tmem_st8d(tm + u * 16, st);
                }
                tmem_wait_st();
            } else {
#pragma unroll
                for (int u = 0; u < MPT; ++u) {
                    const int k = tid + u * NT;
                    if (k >= n || (FD_DIAG && (pl.dbg & 64))) continue;
                    if (top) {
                        ModeRec c;
                        c.load(p, k);
                        cib_inf[u] = c.ib_inf;
                        cinv[u] = c.inv_nl;
                        cibl[u] = 1.0 / c.b_last;
                        clen[u] = c.len;
                        const int cn = pl.cn;
                        const double *cb = pl.carry + size_t(sg.blk) * kCarryVals * cn + k;
                        const size_t bs = size_t(kCarryVals) * cn;
                        xs[u] = has_next ? __ldcg(cb + bs + 6 * cn) : 0.0;
                        yins[u] = has_in ? __ldcg(cb - bs + 5 * cn) : 0.0;
                        pcs[u] = __ldcg(cb + 2 * cn);
                    }
                    sweep3(k, xs[u], pcs[u], yins[u], cib_inf[u], cinv[u], cibl[u], clen[u]);
                }
            }
            trace(5, it, 0);
            __syncthreads();   // swept rows complete, table slice consumed
            trace(3, it, 0);
            int si2 = 0, g2 = 0, rows2 = 0;
            const bool more = it + 1 < nitems;
            if (more) item_of(it + 1, si2, g2, rows2, true);
            if (tid == 0 && more && pl.job[segs[si2].job].p.lt) issue_lts(pl.job[segs[si2].job].p, g2, rows2);
            const int rp = min(2, rows - 2 * pr);
            if (rp > 0) {
                trace(8 + pr, it, 0);
                double *base = regd(pr) + so;
                double *XA = regd(pr), *XB = regd(pr) + XR;
                if (!(FD_DIAG && (pl.dbg & 32)))
                F::run(regc(pr), base, rp > 1 ? base + n : nullptr, al, 0.5 * p.scale, m16, la, scr, t, pr, lane,
                       XA, rp > 1 ? XB : nullptr,
                       (FD_DIAG && pl.trace && (pl.dbg & 4) && blockIdx.x == pl.trace_cta && it < 4)
                           ? reinterpret_cast<long long *>(pl.trace) + 2048 + 32 + it * 8 : nullptr);
                rsync<T>(pr);
                trace(8 + pr, it, 1);
                // epilogue out = alpha x + beta other, row by row from the padded X
                // layout; 8 independent loads/stores in flight per thread
                const double al_ = J.alpha, be_ = J.beta;
                for (int h = 0; h < rp; ++h) {
                    const double *Xh = XA + h * XR;
                    double *oh = J.out + size_t(g0 + 2 * pr + h) * n;
                    const double *qh = J.other ? J.other + size_t(g0 + 2 * pr + h) * n : nullptr;
                    if (qh) {
#pragma unroll 8
                        for (int q = t; q < n; q += T) oh[q] = fma(be_, __ldg(qh + q), al_ * Xh[xi(q)]);
                    } else if (al_ == 1.0) {
#pragma unroll 8
                        for (int q = t; q < n; q += T) oh[q] = Xh[xi(q)];
                    } else {
#pragma unroll 8
                        for (int q = t; q < n; q += T) oh[q] = al_ * Xh[xi(q)];
                    }
                }
                rsync<T>(pr);   // region free
                trace(4, it, 1);
            }
            if (more && t == 0) tail = issue_pair(pl.job[segs[si2].job].out, g2, rows2, pl.job[segs[si2].job].p.m);
            // no CTA barrier here: the next item's sweep starts only after every
            // pair's refill (issued after that pair's stores) has landed
            trace(3, it, 1);
        }
    }
    stamp(5);
    if constexpr (kTm) {
        tmem_fence_before();
        __syncthreads();
        if (tid < 32) {
            tmem_fence_after();
            tmem_dealloc512(tmem_base_s);
        }
    }
}

// ---------------------------------------------------------------------------
template <int NL>
struct RsK {
    static constexpr int NT = RS<NL>::NT, G = RS<NL>::G;
    static constexpr size_t SMEM = RS<NL>::SMEM;
    static const void *fn() { return (const void *)rsolve_kernel<NL>; }
};

// the FFT-path solve of a batch of plans with one transform length
bool launch_persist(const std::vector<SolveJob> &jobs, cudaStream_t s, Workspace &ws) {
    const int n = jobs[0].p.n;
    if (!rs_supported(n) || !jobs[0].p.ralpha) return false;
    switch (n + 1) {
        case 256: run_persist<RsK<8>>(jobs, s, ws); return true;
        case 512: run_persist<RsK<9>>(jobs, s, ws); return true;
        case 1024: run_persist<RsK<10>>(jobs, s, ws); return true;
        case 2048: run_persist<RsK<11>>(jobs, s, ws); return true;
        case 4096: run_persist<RsK<12>>(jobs, s, ws); return true;
        default: return false;
    }
}

}  // namespace fd
