// Persistent fused rectangle solve for the FFT transform lengths (n + 1 = 2^p).
//
// One cooperative launch per batched solve, one CTA set resident on every SM:
//   phase 1  rows of all jobs (rectangles) are split evenly over the CTAs; each
//            CTA streams its row groups global -> shared with TMA bulk copies
//            (cp.async.bulk + mbarrier; the next group is in flight while the
//            current one is transformed), DST-I's them (radix-16 Stockham FFT
//            of packed row pairs) and runs the local forward elimination of its
//            block; yhat goes to the output buffer, the block scalars
//            (yhat_e, F_s, P_e, xi_s, Q) to the carry workspace.
//   grid sync
//   phase 2  carries: per (rectangle, 32 modes) one warp runs the block
//            recurrences Y_b = yhat_e + P_e Y_{b-1},
//            X_b = F_s + Y_{b-1} xi_s + Q X_{b+1} (L2-resident data).
//   grid sync
//   phase 3  per CTA, groups descending: TMA-streamed yhat rows, carry fix-up
//            y_i = yhat_i + P_i Y_{b-1}, the reference back-substitution
//            x_i = (y_i - delta x_{i+1}) / beta_i (rectsolver.py:88-90) with
//            x_{e+1} = X_{b+1}, inverse DST-I, epilogue out = alpha x + beta o.
// Between the phases yhat (8 B/pt) normally stays in the 126 MB L2 for the
// BASELINE config-1 batch; the algorithmic traffic is 32 B/pt either way.
#include "persist_common.cuh"



namespace fd {

constexpr int kPersistThreads = 512;   // one CTA per SM, 128 registers per thread

template <int LG>
struct PCfg {
    using F = FftDst<LG, kPersistThreads>;
    static constexpr int NT = F::NT, G = F::G;
    static constexpr int MPT = (F::N - 1 + NT - 1) / NT;
    static constexpr size_t XBUF = F::SMEM;
    static constexpr size_t STG = (size_t(G) * (F::N - 1) + 4) * sizeof(double);
    static constexpr size_t TWS = (16 + 256 + 256 + 16) * sizeof(double2);
    static constexpr size_t LTB = 13 * 1024;   // one group's slice of the long-transient table
    static constexpr size_t SMEM = XBUF + STG + TWS + LTB;
};

template <int LG>
__global__ void __launch_bounds__(PCfg<LG>::NT, 1) persist_kernel(const __grid_constant__ PList pl) {
    using F = typename PCfg<LG>::F;
    using FL = Fft2<LG, kPersistThreads>;
    using C = PCfg<LG>;
    constexpr int NT = C::NT, G = C::G, MPT = C::MPT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *xbuf = reinterpret_cast<double2 *>(smem_raw);
    // group row rr lives inside the exchange buffer of its pair (rr / 2)
    auto rowp = [&](int rr) { return reinterpret_cast<double *>(xbuf + (rr >> 1) * F::PADL) + (rr & 1) * pl.n; };
    // two spare rows per pair region (4.25 n doubles each): phase-3 transient 1/beta
    static_assert(F::PADL * 2 >= 4 * F::N, "pair region holds 4 rows");
    auto auxp = [&](int rr) {
        return reinterpret_cast<double *>(xbuf + (rr >> 1) * F::PADL) + (2 + (rr & 1)) * pl.n;
    };
    double *stg = reinterpret_cast<double *>(smem_raw + C::XBUF);
    double2 *tw16 = reinterpret_cast<double2 *>(smem_raw + C::XBUF + C::STG);
    double2 *tw256 = tw16 + 16, *twla = tw256 + 256, *twlb = twla + 256;
    double *lts = reinterpret_cast<double *>(smem_raw + C::XBUF + C::STG + C::TWS);   // [G][3][ktp]
    __shared__ __align__(8) uint64_t bar;
    __shared__ Seg segs[kMaxSegs];
    __shared__ int nseg_s, nitems_s;

    const int tid = threadIdx.x;
    const int n = pl.n;
    const int pr = tid / F::T, t = tid % F::T;
    cg::grid_group grid = cg::this_grid();
    auto stamp = [&](int slot) {
        if (pl.tstamp && tid == 0) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
            pl.tstamp[blockIdx.x * 8 + slot] = g;
        }
    };
    stamp(0);
    // FD_TRACE=<cta>: per-item timeline of one CTA -> pl.trace[role][item][2]
    auto trace = [&](int role, int item, int which) {
        if (pl.trace && tid == 0 && blockIdx.x == pl.trace_cta && item < 64) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
            pl.trace[(role * 64 + item) * 2 + which] = g;
        }
    };

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
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    {   // twiddle base tables from the exact L-point table (all jobs share n)
        constexpr int L = F::L, NBL = L / F::RL;
        const double2 *tw = pl.job[0].p.tw;
        for (int q = tid; q < 16; q += NT) tw16[q] = __ldg(tw + q * (L / 256));
        if constexpr (L >= 4096)
            for (int q = tid; q < 256; q += NT) tw256[q] = __ldg(tw + q * (L / 4096));
        for (int q = tid; q < 256; q += NT) twla[q] = __ldg(tw + q * (NBL <= 256 ? 1 : 16));
        for (int q = tid; q < 16; q += NT) twlb[q] = __ldg(tw + q);
    }
    __syncthreads();
    const TwPow tws{tw16, tw256, twla, twlb};
    const int nseg = nseg_s, nitems = nitems_s;
    uint32_t parity = 0;
    // per-CTA beta checkpoints: slot it (phase-1 item) = beta at the item's last
    // row; slot bstride-1-si = beta_{s-1} of segment si
    double *bsave = pl.bsave + size_t(blockIdx.x) * pl.bstride * n;

    auto item_of = [&](int it, int &si, int &g0, int &rows, bool desc) {
        si = 0;
        while (si + 1 < nseg && it >= segs[si + 1].item0) ++si;
        const Seg &sg = segs[si];
        const int gi = it - sg.item0;
        const int gg = desc ? (sg.ngroups - 1 - gi) : gi;
        g0 = sg.s + gg * G;
        rows = min(G, sg.e - g0 + 1);
    };

    // ===================== phase 1: DST + local forward elimination ===================
    {
        // per mode: yhat, pi (running product), F_s, sum pi^2/beta, beta of the
        // previous row, -l_s (P_i = -l_s pi_i)
        double ys[MPT], pis[MPT], fss[MPT], s2s[MPT], bps[MPT], ccs[MPT];
        double cl[MPT], cib[MPT], cbl[MPT], cibl[MPT], clam[MPT];   // l_inf, 1/beta_inf, beta_{m-1}, 1/beta_{m-1}, lambda
        int clen[MPT];
        Tail tail{0.0, -1};
        if (tid == 0 && nitems > 0) {
            int si, g0, rows;
            item_of(0, si, g0, rows, false);
            const PJob &J = pl.job[segs[si].job];
            tail = issue_rows(stg, J.in, g0, rows, n, J.p.m, &bar, lts, J.p.lt, J.p.ktp);
        }
#pragma unroll 1
        for (int it = 0; it < nitems; ++it) {
            int si, g0, rows;
            item_of(it, si, g0, rows, false);
            const Seg sg = segs[si];
            const PJob &J = pl.job[sg.job];
            const PlanDev &p = J.p;
            const double off = p.off;
            trace(0, it, 0);
            mbar_wait(&bar, parity);
            parity ^= 1u;
            trace(0, it, 1);
            if (has_tail(J.in, g0, rows, n, p.m)) {
                if (tid == 0) stg[tail.idx] = tail.v;
                __syncthreads();
            }
            const int so = stg_off(J.in, g0, n);
            {
                const int ra = 2 * pr, rb = 2 * pr + 1;
                double2 *buf = xbuf + pr * F::PADL;
                double2 v[16];
                FL::load(v, ra < rows ? stg + so + ra * n : nullptr, rb < rows ? stg + so + rb * n : nullptr, t);
                __syncthreads();   // staging consumed
                if (tid == 0 && it + 1 < nitems) {
                    int si2, g2, rows2;
                    item_of(it + 1, si2, g2, rows2, false);
                    const PJob &J2 = pl.job[segs[si2].job];
                    tail = issue_rows(stg, J2.in, g2, rows2, n, J2.p.m, &bar, lts, J2.p.lt, J2.p.ktp,
                                      /*defer_lt=*/true);
                }
                FL::store(buf, v, t, pr);
                FL::template mids<F::NMID, 16>(buf, tws, t, pr);
                double *oa = rowp(ra), *ob = rowp(rb);   // pair-local rows
                const bool va = ra < rows, vb = rb < rows;
                FL::last(buf, tws, t, pr, p.scale, [&](int k, double a, double b) {
                    if (va) oa[k] = a;
                    if (vb) ob[k] = b;
                });
                __syncthreads();   // all rows of the group transformed
            }
            trace(1, it, 0);
            const bool first = (g0 == sg.s), last = (g0 + rows - 1 == sg.e);
            double *outg = J.out + size_t(g0) * n;
            const int mlast = p.m - 1;
#pragma unroll
            for (int u = 0; u < MPT; ++u) {
                const int k = tid + u * NT;
                if (k >= n) continue;
                double y = ys[u], w = pis[u], f = fss[u], s2 = s2s[u], bp = bps[u];
                if (first) {
                    ModeRec c;
                    c.load(p, k);
                    cl[u] = c.l_inf;
                    cib[u] = c.ib_inf;
                    cbl[u] = c.b_last;
                    cibl[u] = 1.0 / c.b_last;
                    clam[u] = c.lam;
                    clen[u] = c.len;
                    bp = g0 > 0 ? beta_at(p, c, k, g0 - 1) : 0.0;
                    __stcg(bsave + size_t(pl.bstride - 1 - si) * n + k, bp);
                }
                const int len = clen[u];
                const double l_inf = cl[u], ib_inf = cib[u];
                const double cbinf = mode_binf(p, k);
#pragma unroll
                for (int rr = 0; rr < G; ++rr) {
                    if (rr >= rows) break;
                    const int i = g0 + rr;
                    const double r = rowp(rr)[k];
                    double l, ib;
                    if (k < p.kt) {
                        // slowly converging low mode: reference factors from the table
                        l = lts[rr * 3 * p.ktp + k];
                        ib = lts[rr * 3 * p.ktp + p.ktp + k];
                    } else if (i < len) {
                        // transient row: the reference factorisation, recomputed
                        // bitwise (rectsolver.py:72-73), no table traffic
                        const double d = diag_at(p, clam[u], i);
                        double b;
                        if (i == 0) {
                            l = 0.0;
                            b = d;
                        } else {
                            l = __ddiv_rn(off, bp);
                            b = __dsub_rn(d, __dmul_rn(off, l));
                        }
                        ib = 1.0 / b;
                        bp = b;
                    } else {
                        l = l_inf;
                        ib = (i == mlast) ? cibl[u] : ib_inf;
                    }
                    if (first && rr == 0) {
                        y = r;
                        w = 1.0;
                        f = 0.0;
                        s2 = 0.0;
                        ccs[u] = (i == 0) ? 0.0 : -l;   // P_i = -l_s pi_i
                    } else {
                        y = __dsub_rn(r, __dmul_rn(l, y));   // rectsolver.py:86
                        w = -l * w;
                    }
                    const double W = w * ib;
                    f = fma(y, W, f);
                    s2 = fma(w, W, s2);
                    outg[rr * n + k] = y;
                }
                const int ie = g0 + rows - 1;
                const double bend = ie < len ? bp : (ie == mlast ? cbl[u] : cbinf);
                __stcg(bsave + size_t(it) * n + k, bend);
                ys[u] = y;
                pis[u] = w;
                fss[u] = f;
                s2s[u] = s2;
                bps[u] = bp;
                if (last) {
                    double *cb = pl.carry + size_t(sg.blk) * kCarryVals * n + k;
                    const int e = sg.e;
                    const double cc = ccs[u];
                    // Q = pi_e * (-l_{e+1}),  l_{e+1} = delta / beta_e
                    const double lnext = (k < p.kt) ? ((e + 1 < p.m) ? __ldg(p.lt + size_t(e + 1) * 3 * p.ktp + k) : 0.0)
                                                    : ((e + 1 < len) ? __ddiv_rn(off, bend) : l_inf);
                    const double Q = (e < p.m - 1) ? w * (-lnext) : 0.0;
                    __stcg(cb + 0 * n, y);
                    __stcg(cb + 1 * n, f);
                    __stcg(cb + 2 * n, cc * w);
                    __stcg(cb + 3 * n, cc * s2);
                    __stcg(cb + 4 * n, Q);
                }
            }
            __syncthreads();   // rowbuf and the table slice consumed
            trace(1, it, 1);
            if (tid == 0 && it + 1 < nitems) {
                int si2, g2, rows2;
                item_of(it + 1, si2, g2, rows2, false);
                const PJob &J2 = pl.job[segs[si2].job];
                if (J2.p.lt) issue_lt(lts, J2.p.lt, g2, rows2, J2.p.ktp, &bar);
            }
        }
    }
    stamp(1);
    grid.sync();
    stamp(2);

    // ===================== phase 2: block carries =====================================
    // One CTA per (job, 32 modes): all blocks' scalars are staged through shared
    // memory in one round trip (every thread issues loads), warp 0 (lane = mode)
    // runs both short recurrences out of shared memory, then Y and X go back.
    {
        constexpr int CHB = 96;                               // blocks per staged chunk
        double *sv = reinterpret_cast<double *>(smem_raw);   // [CHB][7][32]
        const int chunks = (n + 31) / 32;
        const size_t bs = size_t(kCarryVals) * n;
        for (int item = blockIdx.x; item < pl.count * chunks; item += gridDim.x) {
            const PJob &J = pl.job[item / chunks];
            const int k0 = (item % chunks) * 32;
            double *cb = pl.carry + size_t(J.blk_base) * bs + k0;
            const int nb = J.nblk, lane = tid & 31;
            const bool lane_ok = (tid < 32) && (k0 + lane < n);
            double prev = 0.0, next = 0.0;
            if (nb <= CHB) {
                for (int idx = tid; idx < nb * 160; idx += NT) {   // 5 values x 32 modes per block
                    const int b = idx / 160, v = (idx >> 5) % 5, kk = idx & 31;
                    sv[(b * 7 + v) * 32 + kk] = (k0 + kk < n) ? __ldcg(cb + b * bs + v * n + kk) : 0.0;
                }
                __syncthreads();
                if (lane_ok) {
                    for (int b = 0; b < nb; ++b) {
                        const double *q = sv + b * 7 * 32 + lane;
                        const double y = (b == 0) ? q[0] : fma(q[2 * 32], prev, q[0]);
                        sv[(b * 7 + 5) * 32 + lane] = y;
                        prev = y;
                    }
                    for (int b = nb - 1; b >= 0; --b) {
                        const double *q = sv + b * 7 * 32 + lane;
                        double x = q[1 * 32];
                        if (b > 0) x = fma(sv[((b - 1) * 7 + 5) * 32 + lane], q[3 * 32], x);
                        if (b < nb - 1) x = fma(q[4 * 32], next, x);
                        sv[(b * 7 + 6) * 32 + lane] = x;
                        next = x;
                    }
                }
                __syncthreads();
                for (int idx = tid; idx < nb * 64; idx += NT) {
                    const int b = idx >> 6, v = 5 + ((idx >> 5) & 1), kk = idx & 31;
                    if (k0 + kk < n) __stcg(cb + b * bs + v * n + kk, sv[(b * 7 + v) * 32 + kk]);
                }
                __syncthreads();
            } else {
                // long block lists: direct (slower) sweeps
                if (lane_ok) {
                    for (int b = 0; b < nb; ++b) {
                        const double ye = __ldcg(cb + b * bs + lane), pe = __ldcg(cb + b * bs + 2 * n + lane);
                        const double y = (b == 0) ? ye : fma(pe, prev, ye);
                        __stcg(cb + b * bs + 5 * n + lane, y);
                        prev = y;
                    }
                    for (int b = nb - 1; b >= 0; --b) {
                        double x = __ldcg(cb + b * bs + 1 * n + lane);
                        if (b > 0) x = fma(__ldcg(cb + (b - 1) * bs + 5 * n + lane), __ldcg(cb + b * bs + 3 * n + lane), x);
                        if (b < nb - 1) x = fma(__ldcg(cb + b * bs + 4 * n + lane), next, x);
                        __stcg(cb + b * bs + 6 * n + lane, x);
                        next = x;
                    }
                }
            }
        }
    }
    stamp(3);
    grid.sync();
    stamp(4);

    // ===================== phase 3: back-substitution + inverse DST ===================
    {
        double xs[MPT], yins[MPT], pcs[MPT], bnx[MPT];
        double cib_inf[MPT], cinv[MPT], cibl[MPT];   // 1/beta_inf, 1/(-l_inf), 1/beta_{m-1}
        int clen[MPT];
        Tail tail{0.0, -1};
        auto beta_before = [&](int it3, int k) {   // beta_{g0-1} of phase-3 item it3 (from bsave)
            int si, g0, rows;
            item_of(it3, si, g0, rows, true);
            const int gg = (g0 - segs[si].s) / G;
            return gg > 0 ? __ldcg(bsave + size_t(segs[si].item0 + gg - 1) * n + k)
                          : __ldcg(bsave + size_t(pl.bstride - 1 - si) * n + k);
        };
        if (tid == 0 && nitems > 0) {
            int si, g0, rows;
            item_of(0, si, g0, rows, true);
            asm volatile("fence.proxy.async.global;" ::: "memory");
            const PJob &J = pl.job[segs[si].job];
            tail = issue_rows(stg, J.out, g0, rows, n, J.p.m, &bar, lts, J.p.lt, J.p.ktp);
        }
        if (nitems > 0) {
#pragma unroll
            for (int u = 0; u < MPT; ++u) {
                const int k = tid + u * NT;
                bnx[u] = (k < n) ? beta_before(0, k) : 0.0;
            }
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
            trace(2, it, 0);
            mbar_wait(&bar, parity);
            parity ^= 1u;
            trace(2, it, 1);
            if (has_tail(J.out, g0, rows, n, p.m)) {
                if (tid == 0) stg[tail.idx] = tail.v;
                __syncthreads();
            }
            const int so = stg_off(J.out, g0, n);
#pragma unroll
            for (int u = 0; u < MPT; ++u) {
                const int k = tid + u * NT;
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
                const double bstart = bnx[u];
                if (it + 1 < nitems) bnx[u] = beta_before(it + 1, k);   // prefetch
                double x = xs[u], Pc = pcs[u];
                const double yin = yins[u];
                const int len = clen[u];
                const double ib_inf = cib_inf[u];
                const double *yg = stg + so + k;
                if (k < p.kt) {
                    const double *tb = lts + k;
#pragma unroll
                    for (int rr = G - 1; rr >= 0; --rr) {
                        if (rr >= rows) continue;
                        double y = yg[rr * n];
                        if (has_in) {
                            y = fma(Pc, yin, y);
                            Pc *= tb[rr * 3 * p.ktp + 2 * p.ktp];   // P_{i-1} = -P_i beta_{i-1} / delta
                        }
                        x = __dsub_rn(y, __dmul_rn(off, x)) * tb[rr * 3 * p.ktp + p.ktp];   // rectsolver.py:90
                        rowp(rr)[k] = x;
                    }
                } else if (g0 < len) {
                    // transient rows: rebuild the reference factors forward (bitwise,
                    // rectsolver.py:72-73); 1/beta_i goes to the spare rows of the
                    // pair buffers
                    double bp = bstart;
#pragma unroll
                    for (int rr = 0; rr < G; ++rr) {
                        if (rr >= rows) break;
                        const int i = g0 + rr;
                        double b;
                        if (i < len) {
                            const double d = diag_at(p, mode_lam(p, k), i);
                            b = (i == 0) ? d : __dsub_rn(d, __dmul_rn(off, __ddiv_rn(off, bp)));
                        } else {
                            b = (i == p.m - 1) ? mode_blast(p, k) : mode_binf(p, k);
                        }
                        auxp(rr)[k] = 1.0 / b;
                        bp = b;
                    }
#pragma unroll
                    for (int rr = G - 1; rr >= 0; --rr) {
                        if (rr >= rows) continue;
                        double y = yg[rr * n];
                        if (has_in) {
                            y = fma(Pc, yin, y);
                            // P_{i-1} = P_i / (-l_i) = -P_i beta_{i-1} / delta
                            const double bm1 = rr > 0 ? 1.0 / auxp(rr - 1)[k] : bstart;
                            Pc = -Pc * bm1 / off;
                        }
                        x = __dsub_rn(y, __dmul_rn(off, x)) * auxp(rr)[k];   // rectsolver.py:90
                        rowp(rr)[k] = x;
                    }
                } else {
                    const double ib_m = cibl[u], inl = cinv[u];
                    const int mlast = p.m - 1;
#pragma unroll
                    for (int rr = G - 1; rr >= 0; --rr) {
                        if (rr >= rows) continue;
                        double y = yg[rr * n];
                        if (has_in) {
                            y = fma(Pc, yin, y);
                            Pc *= inl;
                        }
                        const double ib = (g0 + rr == mlast) ? ib_m : ib_inf;
                        x = __dsub_rn(y, __dmul_rn(off, x)) * ib;   // rectsolver.py:90
                        rowp(rr)[k] = x;
                    }
                }
                xs[u] = x;
                pcs[u] = Pc;
            }
            __syncthreads();   // staging consumed, rowbuf complete
            trace(3, it, 0);
            if (tid == 0 && it + 1 < nitems) {
                int si2, g2, rows2;
                item_of(it + 1, si2, g2, rows2, true);
                const PJob &J2 = pl.job[segs[si2].job];
                tail = issue_rows(stg, J2.out, g2, rows2, n, J2.p.m, &bar, lts, J2.p.lt, J2.p.ktp);
            }
            {
                const int ra = 2 * pr, rb = 2 * pr + 1;
                double2 *buf = xbuf + pr * F::PADL;
                FL::first(buf, ra < rows ? rowp(ra) : nullptr, rb < rows ? rowp(rb) : nullptr, t, pr);
                FL::template mids<F::NMID, 16>(buf, tws, t, pr);
                const bool va = ra < rows, vb = rb < rows;
                double *oa = J.out + size_t(g0 + ra) * n, *ob = J.out + size_t(g0 + rb) * n;
                if (J.other) {
                    const double *qa = J.other + size_t(g0 + ra) * n, *qb = J.other + size_t(g0 + rb) * n;
                    const double al = J.alpha, be = J.beta;
                    FL::last(buf, tws, t, pr, p.scale, [&](int k, double a, double b) {
                        if (va) oa[k] = fma(be, __ldg(qa + k), al * a);
                        if (vb) ob[k] = fma(be, __ldg(qb + k), al * b);
                    });
                } else if (J.alpha == 1.0) {
                    FL::last(buf, tws, t, pr, p.scale, [&](int k, double a, double b) {
                        if (va) oa[k] = a;
                        if (vb) ob[k] = b;
                    });
                } else {
                    const double al = J.alpha;
                    FL::last(buf, tws, t, pr, p.scale, [&](int k, double a, double b) {
                        if (va) oa[k] = al * a;
                        if (vb) ob[k] = al * b;
                    });
                }
                __syncthreads();
            }
            trace(3, it, 1);
        }
    }
    stamp(5);
}

// ---------------------------------------------------------------------------
// traits + dispatch
template <int LG>
struct PersistA {
    static constexpr int NT = PCfg<LG>::NT, G = PCfg<LG>::G;
    static constexpr size_t SMEM = PCfg<LG>::SMEM;
    static const void *fn() { return (const void *)persist_kernel<LG>; }
};

bool launch_rsolve(const std::vector<SolveJob> &jobs, cudaStream_t s, Workspace &ws);
bool launch_rsws(const std::vector<SolveJob> &jobs, cudaStream_t s, Workspace &ws);

bool launch_persist(const std::vector<SolveJob> &jobs, cudaStream_t s, Workspace &ws) {
    if (launch_rsws(jobs, s, ws)) return true;
    if (launch_rsolve(jobs, s, ws)) return true;
    const int n = jobs[0].p.n;
    int lg = 0;
    while ((1 << lg) < 2 * (n + 1)) ++lg;
    switch (lg) {
        case 9: run_persist<PersistA<9>>(jobs, s, ws); return true;
        case 10: run_persist<PersistA<10>>(jobs, s, ws); return true;
        case 11: run_persist<PersistA<11>>(jobs, s, ws); return true;
        case 12: run_persist<PersistA<12>>(jobs, s, ws); return true;
        case 13: run_persist<PersistA<13>>(jobs, s, ws); return true;
        default: return false;
    }
}

}  // namespace fd
