// Warp-specialised persistent fused solve for n + 1 <= 1024 (the BASELINE
// config-1 shape n = 1023).
//
// Same arithmetic as persist.cu (three phases between grid syncs), but the
// CTA is split into two teams that run concurrently instead of in lockstep:
//   FFT team   (256 threads = P row-pair teams of T threads): each pair team
//              streams its own row pairs through a private 2-stage TMA ring,
//              transforms them (Stockham radix-16, per-pair named barriers)
//              and hands the spectra to the Thomas team through a
//              double-buffered output slot (mbarrier full/empty protocol);
//   Thomas team (256 threads, <= 4 modes each, state in registers): consumes
//              row pairs strictly in order and runs the per-mode recurrences
//              (phase 1: local forward elimination; phase 3: carry fix-up and
//              back-substitution, feeding the FFT team the other way round).
// So shared-memory-heavy FFT passes of one pair overlap fp64-heavy passes of
// the other and the latency-bound Thomas chains overlap both.
#include "persist_common.cuh"

namespace fd {

template <int LG>
struct WsCfg {
    using F = FftDst<LG, 256>;
    using FL = Fft2<LG, 256>;
    static constexpr int T = F::T, P = F::PAIRS, NF = P * T;   // FFT team
    static constexpr int NTT = 256;                            // Thomas team
    static constexpr int NT = NF + NTT;
    static constexpr int G = 2;                                // rows per item
    static constexpr int N = F::N, PADL = F::PADL;
    static constexpr int MT = (N - 1 + NTT - 1) / NTT;         // modes per Thomas thread
    static constexpr int KTMAX = 96;                           // long-transient table width
    static constexpr size_t ROWS2 = (size_t(2) * (N - 1) + 4) * 8;   // row pair + TMA slack
    static constexpr size_t LTS = size_t(2) * 3 * KTMAX * 8;
    static constexpr size_t OSLOT = ROWS2 + LTS;               // output slot: rows + table slice
    static constexpr int RING = 2;                             // phase-1 stages per pair
    static constexpr size_t XB = size_t(P) * PADL * 16;
    static constexpr size_t RB = size_t(P) * RING * ROWS2;     // phase 1 rings / phase 3 Thomas ring
    static constexpr size_t OB = size_t(P) * 2 * OSLOT;        // phase 1 outputs / phase 3 inputs
    static constexpr int RING3 = int(RB / OSLOT);              // phase-3 Thomas ring stages
    static constexpr size_t TWS = (16 + 256 + 256 + 16) * sizeof(double2);
    static constexpr size_t SMEM = XB + RB + OB + TWS;
    static_assert(RING3 >= 2, "phase-3 ring");
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void team_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int LG>
__global__ void __launch_bounds__(WsCfg<LG>::NT, 1) persist_ws_kernel(const __grid_constant__ PList pl) {
    using C = WsCfg<LG>;
    using F = typename C::F;
    using FL = typename C::FL;
    constexpr int T = C::T, P = C::P, NF = C::NF, NTT = C::NTT, MT = C::MT, NT = C::NT;
    constexpr int THOMAS_BAR = 1 + P;   // named barrier of the Thomas team
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *xbuf = reinterpret_cast<double2 *>(smem_raw);
    unsigned char *rbase = smem_raw + C::XB;
    unsigned char *obase = rbase + C::RB;
    double2 *tw16 = reinterpret_cast<double2 *>(obase + C::OB);
    double2 *tw256 = tw16 + 16, *twla = tw256 + 256, *twlb = twla + 256;
    __shared__ __align__(8) uint64_t rf[P][C::RING], of[P][2], oe[P][2];   // phase 1
    __shared__ __align__(8) uint64_t tf[8], if_[P][2], ie[P][2];           // phase 3
    __shared__ Seg segs[kMaxSegs];
    __shared__ int nseg_s, nitems_s;

    const int tid = threadIdx.x;
    const int n = pl.n;
    const bool fft = tid < NF;
    const int pr = fft ? tid / T : 0, t = fft ? tid % T : 0;
    const int tt = tid - NF;   // Thomas thread index (valid when !fft)
    cg::grid_group grid = cg::this_grid();
    auto stamp = [&](int slot) {
        if (pl.tstamp && tid == 0) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
            pl.tstamp[blockIdx.x * 8 + slot] = g;
        }
    };
    stamp(0);
    auto ring_stage = [&](int p, int s) { return reinterpret_cast<double *>(rbase + (size_t(p) * C::RING + s) * C::ROWS2); };
    auto oslot = [&](int p, int b) { return reinterpret_cast<double *>(obase + (size_t(p) * 2 + b) * C::OSLOT); };
    auto oslot_lt = [&](int p, int b) { return reinterpret_cast<double *>(obase + (size_t(p) * 2 + b) * C::OSLOT + C::ROWS2); };
    auto tstage = [&](int s) { return reinterpret_cast<double *>(rbase + size_t(s) * C::OSLOT); };
    // FD_TRACE: per-item timeline of CTA 0 -> pl.trace[role][item][2]
    auto trace = [&](int role, int item, int which) {
        if (pl.trace && blockIdx.x == pl.trace_cta && item < 64) {
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
                    sg.ngroups = (sg.e - sg.s + 2) / 2;
                    sg.item0 = items;
                    items += sg.ngroups;
                    segs[ns++] = sg;
                }
            }
        }
        nseg_s = ns;
        nitems_s = items;
        for (int p = 0; p < P; ++p) {
            for (int s = 0; s < C::RING; ++s) mbar_init(&rf[p][s], 1);
            for (int b = 0; b < 2; ++b) {
                mbar_init(&of[p][b], T + 1);
                mbar_init(&oe[p][b], NTT);
                mbar_init(&if_[p][b], NTT);
                mbar_init(&ie[p][b], T);
            }
        }
        for (int s = 0; s < 8; ++s) mbar_init(&tf[s], 1);
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
    double *bsave = pl.bsave + size_t(blockIdx.x) * pl.bstride * n;

    // item -> (segment, first row, rows); desc: groups of a segment top-down
    auto item_of = [&](int it, int &si, int &g0, int &rows, bool desc) {
        si = 0;
        while (si + 1 < nseg && it >= segs[si + 1].item0) ++si;
        const Seg &sg = segs[si];
        const int gi = it - sg.item0;
        const int gg = desc ? (sg.ngroups - 1 - gi) : gi;
        g0 = sg.s + gg * 2;
        rows = min(2, sg.e - g0 + 1);
    };

    // ================================ phase 1 ======================================
    if (fft) {
        // ---- FFT pair team: items pr, pr + P, ...
        double2 *buf = xbuf + pr * C::PADL;
        Tail tails[C::RING];
        auto issue = [&](int k) {
            const int it = pr + k * P;
            int si, g0, rows;
            item_of(it, si, g0, rows, false);
            const PJob &J = pl.job[segs[si].job];
            tails[k % C::RING] = issue_rows(ring_stage(pr, k % C::RING), J.in, g0, rows, n, J.p.m,
                                            &rf[pr][k % C::RING]);
        };
        if (t == 0)
            for (int k = 0; k < C::RING && pr + k * P < nitems; ++k) issue(k);
#pragma unroll 1
        for (int k = 0; pr + k * P < nitems; ++k) {
            const int it = pr + k * P, s = k % C::RING, b = k & 1;
            int si, g0, rows;
            item_of(it, si, g0, rows, false);
            const PJob &J = pl.job[segs[si].job];
            const PlanDev &p = J.p;
            if (t == 0) trace(pr, k, 0);
            mbar_wait(&rf[pr][s], (k / C::RING) & 1);
            if (t == 0) trace(pr, k, 1);
            double *stg = ring_stage(pr, s);
            if (has_tail(J.in, g0, rows, n, p.m)) {
                if (t == 0) stg[tails[s].idx] = tails[s].v;
                pair_sync<T>(pr);
            }
            const int so = stg_off(J.in, g0, n);
            double2 v[16];
            FL::load(v, stg + so, rows > 1 ? stg + so + n : nullptr, t);
            pair_sync<T>(pr);   // stage consumed by the whole pair
            if (t == 0 && pr + (k + C::RING) * P < nitems) issue(k + C::RING);
            FL::store(buf, v, t, pr);
            FL::template mids<F::NMID, 16>(buf, tws, t, pr);
            // output slot b must have been consumed by the Thomas team (item k-2)
            mbar_wait(&oe[pr][b], ((k >> 1) & 1) ^ 1);
            double *oa = oslot(pr, b), *ob = oa + n;
            if (t == 0) {
                if (p.lt) {
                    const uint32_t bytes = uint32_t(rows) * 3u * uint32_t(p.ktp) * 8u;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(&of[pr][b], bytes);
                    tma_load_1d(oslot_lt(pr, b), p.lt + size_t(g0) * 3 * p.ktp, bytes, &of[pr][b]);
                } else {
                    mbar_arrive(&of[pr][b]);
                }
            }
            const bool vb = rows > 1;
            FL::last(buf, tws, t, pr, p.scale, [&](int kk, double a, double bb) {
                oa[kk] = a;
                if (vb) ob[kk] = bb;
            });
            mbar_arrive(&of[pr][b]);
        }
    } else {
        // ---- Thomas team: all items in order
        double ys[MT], pis[MT], fss[MT], s2s[MT], bps[MT], ccs[MT];
        double cl[MT], cib[MT], cbl[MT], cbi[MT], clam[MT];
        int cfix[MT];
#pragma unroll 1
        for (int it = 0; it < nitems; ++it) {
            const int pp = it % P, k2 = it / P, b = k2 & 1;
            int si, g0, rows;
            item_of(it, si, g0, rows, false);
            const Seg sg = segs[si];
            const PJob &J = pl.job[sg.job];
            const PlanDev &p = J.p;
            const double off = p.off;
            const int mlast = p.m - 1, kt = p.kt, ktp = p.ktp;
            const bool first = (g0 == sg.s), last = (g0 + rows - 1 == sg.e);
            const bool has_last_row = (g0 + rows - 1 == mlast);
            if (tt == 0) trace(8, it, 0);
            mbar_wait(&of[pp][b], (k2 >> 1) & 1);
            if (tt == 0) trace(8, it, 1);
            const double *orow = oslot(pp, b);
            const double *lts = oslot_lt(pp, b);
            double *outg = J.out + size_t(g0) * n;
#pragma unroll
            for (int u = 0; u < MT; ++u) {
                const int k = tt + u * NTT;
                if (k >= n) continue;
                if (first) {
                    ModeRec c;
                    c.load(p, k);
                    cl[u] = c.l_inf;
                    cib[u] = c.ib_inf;
                    cbi[u] = c.b_inf;
                    cbl[u] = c.b_last;
                    clam[u] = c.lam;
                    cfix[u] = c.len;
                    bps[u] = g0 > 0 ? beta_at(p, c, k, g0 - 1) : 0.0;
                    __stcg(bsave + size_t(pl.bstride - 1 - si) * n + k, bps[u]);
                }
                // per-row factors (l_i, 1/beta_i) for this item's rows
                double lr[2], ibr[2];
                if (k < kt) {                                       // long transient: table slice
                    lr[0] = lts[k];
                    ibr[0] = lts[ktp + k];
                    lr[1] = lts[3 * ktp + k];
                    ibr[1] = lts[4 * ktp + k];
                } else if (g0 < cfix[u]) {                          // short transient: recompute
                    double bp = bps[u];
#pragma unroll
                    for (int rr = 0; rr < 2; ++rr) {
                        const int i = g0 + rr;
                        double l = cl[u], ib = cib[u];
                        if (rr < rows && i < cfix[u]) {
                            const double d = diag_at(p, clam[u], i);
                            double bb;
                            if (i == 0) {
                                l = 0.0;
                                bb = d;
                            } else {
                                l = __ddiv_rn(off, bp);
                                bb = __dsub_rn(d, __dmul_rn(off, l));
                            }
                            ib = 1.0 / bb;
                            bp = bb;
                        }
                        lr[rr] = l;
                        ibr[rr] = ib;
                    }
                    bps[u] = bp;
                } else {                                            // converged
                    lr[0] = lr[1] = cl[u];
                    ibr[0] = ibr[1] = cib[u];
                }
                if (has_last_row && k >= kt) {   // east end modifier row
                    if (rows == 2) ibr[1] = 1.0 / cbl[u];
                    else ibr[0] = 1.0 / cbl[u];
                }
                double y = ys[u], w = pis[u], f = fss[u], s2 = s2s[u];
                const double r0 = orow[k];
                if (first) {
                    y = r0;
                    w = 1.0;
                    f = 0.0;
                    s2 = 0.0;
                    ccs[u] = (g0 == 0) ? 0.0 : -lr[0];
                } else {
                    y = __dsub_rn(r0, __dmul_rn(lr[0], y));   // rectsolver.py:86
                    w = -lr[0] * w;
                }
                double W = w * ibr[0];
                f = fma(y, W, f);
                s2 = fma(w, W, s2);
                outg[k] = y;
                if (rows > 1) {
                    const double r1 = orow[n + k];
                    y = __dsub_rn(r1, __dmul_rn(lr[1], y));
                    w = -lr[1] * w;
                    W = w * ibr[1];
                    f = fma(y, W, f);
                    s2 = fma(w, W, s2);
                    outg[n + k] = y;
                }
                const int ie_ = g0 + rows - 1;
                const double bend = (k >= kt && ie_ < cfix[u]) ? bps[u] : (ie_ == mlast ? cbl[u] : cbi[u]);
                __stcg(bsave + size_t(it) * n + k, bend);
                ys[u] = y;
                pis[u] = w;
                fss[u] = f;
                s2s[u] = s2;
                if (last) {
                    double *cb = pl.carry + size_t(sg.blk) * kCarryVals * n + k;
                    const int e = sg.e;
                    const double cc = ccs[u];
                    double lnext = cl[u];
                    if (k < kt) lnext = (e + 1 < p.m) ? __ldg(p.lt + size_t(e + 1) * 3 * ktp + k) : 0.0;
                    else if (e + 1 < cfix[u]) lnext = __ddiv_rn(off, bend);
                    const double Q = (e < mlast) ? w * (-lnext) : 0.0;
                    __stcg(cb + 0 * n, y);
                    __stcg(cb + 1 * n, f);
                    __stcg(cb + 2 * n, cc * w);
                    __stcg(cb + 3 * n, cc * s2);
                    __stcg(cb + 4 * n, Q);
                }
            }
            mbar_arrive(&oe[pp][b]);   // slot consumed
        }
    }
    stamp(1);
    grid.sync();
    stamp(2);

    // ================================ phase 2 ======================================
    {
        constexpr int CHB = 96;
        double *sv = reinterpret_cast<double *>(smem_raw);   // [CHB][7][32] over xbuf/rings
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
                for (int idx = tid; idx < nb * 160; idx += NT) {
                    const int bb = idx / 160, v = (idx >> 5) % 5, kk = idx & 31;
                    sv[(bb * 7 + v) * 32 + kk] = (k0 + kk < n) ? __ldcg(cb + bb * bs + v * n + kk) : 0.0;
                }
                __syncthreads();
                if (lane_ok) {
                    for (int bb = 0; bb < nb; ++bb) {
                        const double *q = sv + bb * 7 * 32 + lane;
                        const double y = (bb == 0) ? q[0] : fma(q[2 * 32], prev, q[0]);
                        sv[(bb * 7 + 5) * 32 + lane] = y;
                        prev = y;
                    }
                    for (int bb = nb - 1; bb >= 0; --bb) {
                        const double *q = sv + bb * 7 * 32 + lane;
                        double x = q[1 * 32];
                        if (bb > 0) x = fma(sv[((bb - 1) * 7 + 5) * 32 + lane], q[3 * 32], x);
                        if (bb < nb - 1) x = fma(q[4 * 32], next, x);
                        sv[(bb * 7 + 6) * 32 + lane] = x;
                        next = x;
                    }
                }
                __syncthreads();
                for (int idx = tid; idx < nb * 64; idx += NT) {
                    const int bb = idx >> 6, v = 5 + ((idx >> 5) & 1), kk = idx & 31;
                    if (k0 + kk < n) __stcg(cb + bb * bs + v * n + kk, sv[(bb * 7 + v) * 32 + kk]);
                }
                __syncthreads();
            } else if (lane_ok) {
                for (int bb = 0; bb < nb; ++bb) {
                    const double ye = __ldcg(cb + bb * bs + lane), pe = __ldcg(cb + bb * bs + 2 * n + lane);
                    const double y = (bb == 0) ? ye : fma(pe, prev, ye);
                    __stcg(cb + bb * bs + 5 * n + lane, y);
                    prev = y;
                }
                for (int bb = nb - 1; bb >= 0; --bb) {
                    double x = __ldcg(cb + bb * bs + 1 * n + lane);
                    if (bb > 0) x = fma(__ldcg(cb + (bb - 1) * bs + 5 * n + lane), __ldcg(cb + bb * bs + 3 * n + lane), x);
                    if (bb < nb - 1) x = fma(__ldcg(cb + bb * bs + 4 * n + lane), next, x);
                    __stcg(cb + bb * bs + 6 * n + lane, x);
                    next = x;
                }
            }
        }
    }
    stamp(3);
    grid.sync();
    stamp(4);

    // ================================ phase 3 ======================================
    if (!fft) {
        // ---- Thomas team: items in phase-3 order, producing x rows for the FFT pairs
        constexpr int R3 = C::RING3 > 8 ? 8 : C::RING3;
        Tail tails3[R3];
        auto issue3 = [&](int j) {
            int si, g0, rows;
            item_of(j, si, g0, rows, true);
            const PJob &J = pl.job[segs[si].job];
            tails3[j % R3] = issue_rows(tstage(j % R3), J.out, g0, rows, n, J.p.m, &tf[j % R3],
                                        tstage(j % R3) + C::ROWS2 / 8, J.p.lt, J.p.ktp);
        };
        if (tt == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");
            for (int j = 0; j < R3 && j < nitems; ++j) issue3(j);
        }
        double xs[MT], yins[MT], pcs[MT], bnx[MT];
        double cibi[MT], cinv[MT], cibl[MT], clam3[MT], cbinf[MT], cblast[MT];
        int cfix[MT];
        auto beta_before = [&](int j, int k) {
            int si, g0, rows;
            item_of(j, si, g0, rows, true);
            const int gg = (g0 - segs[si].s) / 2;
            return gg > 0 ? __ldcg(bsave + size_t(segs[si].item0 + gg - 1) * n + k)
                          : __ldcg(bsave + size_t(pl.bstride - 1 - si) * n + k);
        };
        if (nitems > 0) {
#pragma unroll
            for (int u = 0; u < MT; ++u) {
                const int k = tt + u * NTT;
                bnx[u] = (k < n) ? beta_before(0, k) : 0.0;
            }
        }
#pragma unroll 1
        for (int j = 0; j < nitems; ++j) {
            const int s = j % R3, pp = j % P, k2 = j / P, b = k2 & 1;
            int si, g0, rows;
            item_of(j, si, g0, rows, true);
            const Seg sg = segs[si];
            const PJob &J = pl.job[sg.job];
            const PlanDev &p = J.p;
            const double off = p.off;
            const int mlast = p.m - 1;
            const bool top = (g0 + rows - 1 == sg.e);
            const bool has_in = sg.blk > J.blk_base;
            const bool has_next = sg.blk < J.blk_base + J.nblk - 1;
            if (tt == 0) trace(9, j, 0);
            mbar_wait(&tf[s], (j / R3) & 1);
            if (tt == 0) trace(9, j, 1);
            double *stg = tstage(s);
            if (has_tail(J.out, g0, rows, n, p.m)) {
                if (tt == 0) stg[tails3[s].idx] = tails3[s].v;
                team_sync(THOMAS_BAR, NTT);
            }
            const int so = stg_off(J.out, g0, n);
            const double *lts = stg + C::ROWS2 / 8;
            mbar_wait(&ie[pp][b], ((k2 >> 1) & 1) ^ 1);   // input slot free (FFT consumed item j-2P)
            double *irow = oslot(pp, b);
#pragma unroll
            for (int u = 0; u < MT; ++u) {
                const int k = tt + u * NTT;
                if (k >= n) continue;
                if (top) {
                    ModeRec c;
                    c.load(p, k);
                    cibi[u] = c.ib_inf;
                    cinv[u] = c.inv_nl;
                    cibl[u] = 1.0 / c.b_last;
                    clam3[u] = c.lam;
                    cbinf[u] = c.b_inf;
                    cblast[u] = c.b_last;
                    cfix[u] = c.len;
                    const double *cb = pl.carry + size_t(sg.blk) * kCarryVals * n + k;
                    const size_t bs = size_t(kCarryVals) * n;
                    xs[u] = has_next ? __ldcg(cb + bs + 6 * n) : 0.0;
                    yins[u] = has_in ? __ldcg(cb - bs + 5 * n) : 0.0;
                    pcs[u] = __ldcg(cb + 2 * n);
                }
                const double bstart = bnx[u];
                if (j + 1 < nitems) bnx[u] = beta_before(j + 1, k);
                double ibr[2], pmr[2];
                if (k < p.kt) {
                    ibr[0] = lts[p.ktp + k];
                    pmr[0] = lts[2 * p.ktp + k];
                    ibr[1] = lts[4 * p.ktp + k];
                    pmr[1] = lts[5 * p.ktp + k];
                } else if (g0 < cfix[u]) {
                    double bp = bstart;
#pragma unroll
                    for (int rr = 0; rr < 2; ++rr) {
                        const int i = g0 + rr;
                        double bb = (i == mlast) ? cblast[u] : cbinf[u];
                        if (rr < rows && i < cfix[u]) {
                            const double d = diag_at(p, clam3[u], i);
                            bb = (i == 0) ? d : __dsub_rn(d, __dmul_rn(off, __ddiv_rn(off, bp)));
                        }
                        ibr[rr] = 1.0 / bb;
                        pmr[rr] = -bp / off;
                        bp = bb;
                    }
                } else {
                    ibr[0] = ibr[1] = cibi[u];
                    pmr[0] = pmr[1] = cinv[u];
                    if (g0 + rows - 1 == mlast) {
                        if (rows == 2) ibr[1] = cibl[u];
                        else ibr[0] = cibl[u];
                    }
                }
                double x = xs[u], Pc = pcs[u];
                const double yin = yins[u];
                const double *yg = stg + so + k;
                if (rows > 1) {
                    double y = yg[n];
                    if (has_in) {
                        y = fma(Pc, yin, y);
                        Pc *= pmr[1];   // P_{i-1} = P_i / (-l_i)
                    }
                    x = __dsub_rn(y, __dmul_rn(off, x)) * ibr[1];   // rectsolver.py:90
                    irow[n + k] = x;
                }
                {
                    double y = yg[0];
                    if (has_in) {
                        y = fma(Pc, yin, y);
                        Pc *= pmr[0];
                    }
                    x = __dsub_rn(y, __dmul_rn(off, x)) * ibr[0];
                    irow[k] = x;
                }
                xs[u] = x;
                pcs[u] = Pc;
            }
            mbar_arrive(&if_[pp][b]);            // x rows ready for FFT pair pp
            team_sync(THOMAS_BAR, NTT);          // staging stage s consumed
            if (tt == 0 && j + R3 < nitems) issue3(j + R3);
        }
    } else {
        // ---- FFT pair team: items pr, pr + P, ... of the phase-3 order
        double2 *buf = xbuf + pr * C::PADL;
#pragma unroll 1
        for (int k = 0; pr + k * P < nitems; ++k) {
            const int j = pr + k * P, b = k & 1;
            int si, g0, rows;
            item_of(j, si, g0, rows, true);
            const PJob &J = pl.job[segs[si].job];
            const PlanDev &p = J.p;
            if (t == 0) trace(10 + pr, k, 0);
            mbar_wait(&if_[pr][b], (k >> 1) & 1);
            if (t == 0) trace(10 + pr, k, 1);
            const double *irow = oslot(pr, b);
            double2 v[16];
            FL::load(v, irow, rows > 1 ? irow + n : nullptr, t);
            mbar_arrive(&ie[pr][b]);             // input slot consumed (values are in registers)
            FL::store(buf, v, t, pr);
            FL::template mids<F::NMID, 16>(buf, tws, t, pr);
            const bool vb = rows > 1;
            double *oa = J.out + size_t(g0) * n, *ob = oa + n;
            if (J.other) {
                const double *qa = J.other + size_t(g0) * n, *qb = qa + n;
                const double al = J.alpha, be = J.beta;
                FL::last(buf, tws, t, pr, p.scale, [&](int kk, double a, double bb) {
                    oa[kk] = fma(be, __ldg(qa + kk), al * a);
                    if (vb) ob[kk] = fma(be, __ldg(qb + kk), al * bb);
                });
            } else if (J.alpha == 1.0) {
                FL::last(buf, tws, t, pr, p.scale, [&](int kk, double a, double bb) {
                    oa[kk] = a;
                    if (vb) ob[kk] = bb;
                });
            } else {
                const double al = J.alpha;
                FL::last(buf, tws, t, pr, p.scale, [&](int kk, double a, double bb) {
                    oa[kk] = al * a;
                    if (vb) ob[kk] = al * bb;
                });
            }
        }
    }
    stamp(5);
}

template <int LG>
struct PersistWS {
    static constexpr int NT = WsCfg<LG>::NT, G = WsCfg<LG>::G;
    static constexpr size_t SMEM = WsCfg<LG>::SMEM;
    static const void *fn() { return (const void *)persist_ws_kernel<LG>; }
};

bool launch_persist_ws(const std::vector<SolveJob> &jobs, cudaStream_t s, Workspace &ws) {
    // opt-in (FD_WS=1): correct, but slower than persist.cu on B200 so far
    // (8 FFT warps cannot hide the fp64 dependency chains); kept for tuning
    static const bool enabled = getenv("FD_WS") != nullptr;
    if (!enabled) return false;
    const int n = jobs[0].p.n;
    for (const auto &j : jobs)
        if (j.p.kt > WsCfg<11>::KTMAX) return false;
    int lg = 0;
    while ((1 << lg) < 2 * (n + 1)) ++lg;
    switch (lg) {
        case 11: run_persist<PersistWS<11>>(jobs, s, ws); return true;
        default: return false;
    }
}

}  // namespace fd
