// ARCHIVED EXPERIMENT (not built; moved out of the package).  Measured on a
// B200 at c1 (5 x 1023^2, tools/k3_check.py, FD_PHASE_TIMING stamps):
//   * correct (rel. err <= 1.6e-14 vs the oracle), but 207-323 us per batched
//     apply against 90 us for the shipped lockstep kernel (csrc/rsolve.cu);
//   * 32 complex points per lane needed ~168 registers for the F warps; the
//     setmaxnreg split (F 168 / S 88) deadlocked when an S warpgroup grew back
//     before a pending F setmaxnreg.inc was granted (fixed by a CTA barrier),
//     and both roles still spilled (2.3 M local-memory instructions per
//     launch, a 35-70 us store drain at the grid barrier);
//   * with 16 points per lane (2 warps per pair, no setmaxnreg) the F role
//     alone takes ~26 us per phase and the S role alone 38 / 110 us per phase:
//     the S threads walk ~18 row pairs per phase serially, and the factor-table
//     and yhat loads sit on that chain (without them: 14 / 17 us).
// Kept for the record of what was tried.
// K3: the fused batched rectangle solve (rectsolver.py:183-213: DST-I along y,
// per-mode Thomas sweep along x with the kappa shift, inverse DST-I) as one
// persistent cooperative kernel with warp-specialised roles.
//
// Transform of a row pair (a, b), N = n + 1 = 2^NL, one N-point complex FFT:
//   y_j = alpha_j x_j + (alpha_j - s/2) x_{N-j},  alpha_j = s/2 sin(pi j/N) + s/4
//   c = y_a + i y_b,  C = FFT_N(c)
//   X_{2k} = S_k (prefix sum of Re/Im (C_k + C_{N-k})),  X_{2k+1} = e_{k+1}
//   (e_k = Im C_{N-k} - Im C_k for row a, Re C_k - Re C_{N-k} for row b)
// with s = sqrt(2/N) (the orthonormal DST-I).
//
// Data flow per SM (one CTA of 512 threads; 8 "F" warps, 8 "S" warps):
//   F team (L = N/32 lanes, 32 complex points per lane) = one row pair:
//     class-pair loads: lane t owns the residue classes t and Q - t of
//       j mod Q (Q = N/16): every element of both rows is read exactly once
//       (from HBM in phase 1, from the pair's shared-memory slot in phase 3)
//       and the mirror x_{N-j} needed by the pre-weighting is in the lane;
//     two radix-16 DFTs in registers, twiddles by power chains;
//     ONE exchange through the slot, a radix-32 DFT in registers and a
//       radix-R3 step across R3 = Q/32 lanes (shuffles, R3 = 2 at N = 1024);
//     C to the slot in natural order, post-processing reads C_k, C_{N-k} with
//       16 consecutive k per lane (in-lane + warp scan), transformed rows back
//       into the slot in natural mode order.
//   S threads (256): thread s owns modes s, s + 256, ...; sweeps the rows of
//     its CTA's range in order (phase 1: the reference forward elimination,
//     rectsolver.py:86, with the block scalars of the carry scheme) straight
//     from the slots, writes yhat to the output array with coalesced stores;
//     phase 3 reads yhat back, applies the carry fix-up and the reference
//     back-substitution (rectsolver.py:90) and writes x into the slots for the
//     F teams' inverse transform and the epilogue out = alpha x + beta other.
//   Slots are handed over with one full/empty mbarrier pair per team.
// Phase 2 (block carries between the CTAs' row ranges) is carries_phase().
// Shared-memory traffic per grid point: ~60 B (phase 1) / ~70 B (phase 3),
// against ~120 B each for the lockstep radix-16/16/4 kernel (rsolve.cu).
#include <type_traits>

#include "rsolve_common.cuh"

namespace fd {
namespace k3 {

// cos(2 pi p / 64), p = 0..16 (quarter wave)
constexpr double kQ64[17] = {1.0,
                                        0.99518472667219688624,
                                        0.98078528040323044913,
                                        0.95694033573220886494,
                                        0.92387953251128675613,
                                        0.88192126434835502971,
                                        0.83146961230254523708,
                                        0.77301045336273696081,
                                        0.70710678118654752440,
                                        0.63439328416364549822,
                                        0.55557023301960222474,
                                        0.47139673682599764856,
                                        0.38268343236508977173,
                                        0.29028467725446236764,
                                        0.19509032201612826785,
                                        0.098017140329560601994,
                                        0.0};
__host__ __device__ constexpr double cos64(int p) {
    p &= 63;
    return p <= 16 ? kQ64[p] : p <= 32 ? -kQ64[32 - p] : p <= 48 ? -kQ64[p - 32] : kQ64[64 - p];
}
__host__ __device__ constexpr double sin64(int p) { return cos64(p - 16); }

// a * e^{-2 pi i P / 64}
template <int P>
__device__ __forceinline__ double2 tw64(double2 a) {
    constexpr int p = P & 63;
    if constexpr (p == 0) return a;
    else if constexpr (p == 16) return mul_mi(a);
    else if constexpr (p == 32) return make_double2(-a.x, -a.y);
    else if constexpr (p == 48) return make_double2(-a.y, a.x);
    else if constexpr ((p & 3) == 0) return tw16<p / 4>(a);
    else return cmul(a, make_double2(cos64(p), -sin64(p)));
}

// compile-time loop: f(std::integral_constant<int, I>) for I in [B, E)
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

// 32-point forward DFT in registers, natural order: n = 4 n1 + n2, k = k1 + 8 k2
__device__ __forceinline__ void dft32(double2 (&v)[32]) {
    double2 y[4][8];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
#pragma unroll
        for (int n1 = 0; n1 < 8; ++n1) y[n2][n1] = v[4 * n1 + n2];
        dft<8>(y[n2]);
    }
    static_for<1, 8>([&](auto kk) {
        constexpr int k1 = decltype(kk)::value;
        y[1][k1] = tw64<2 * k1>(y[1][k1]);
        y[2][k1] = tw64<4 * k1>(y[2][k1]);
        y[3][k1] = tw64<6 * k1>(y[3][k1]);
    });
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) {
        double2 a = y[0][k1], b = y[1][k1], c = y[2][k1], d = y[3][k1];
        dft4(a, b, c, d);
        v[k1] = a;
        v[k1 + 8] = b;
        v[k1 + 16] = c;
        v[k1 + 24] = d;
    }
}

// v[r] *= s * w^r (r = 0..R-1), one power chain
template <int R>
__device__ __forceinline__ void chain_twiddle(double2 (&v)[R], double2 w, double s) {
    double2 p = make_double2(s * w.x, s * w.y);
    v[0] = make_double2(s * v[0].x, s * v[0].y);
#pragma unroll
    for (int r = 1; r < R; ++r) {
        v[r] = cmul(v[r], p);
        if (r + 1 < R) p = cmul(p, w);
    }
}

template <int NL>
struct Cfg {
    static constexpr int N = 1 << NL;
    static constexpr int Q = N / 16;              // residue classes j mod Q of the first pass
    static constexpr int L = Q;                   // lanes per row pair (one class each)
    static_assert(NL == 10, "K3 is instantiated for N = 1024 (c1); other lengths use rsolve.cu");
    static constexpr int NT = 512;
#ifndef FD_K3_NFW
#define FD_K3_NFW 10
#endif
    static constexpr int NFW = FD_K3_NFW, NSW = 16 - NFW;   // F warps, S warps
    static constexpr int TEAMS = NFW * 32 / L;    // row pairs in flight (one slot each)
    static constexpr int NST = NSW * 32;          // S threads
    static constexpr int U = (N - 1 + NST - 1) / NST;   // modes per S thread
    // slot layout (complex units of 16 B), conflict-free for every access of
    // the transform (tools/k3v2/model16.py):
    //   E(k1, c)   = 68 k1 + c                      pass-1 output, units [0, 1088)
    //   F(l, k2')  = FOFF + 19 l + k2' + (k2' >> 2 & 3)  pass-2 output
    //   C_k at pc(k) = k + k/8 + 2 (k/64)          units [0, 1181)
    __host__ __device__ static constexpr int eix(int k1, int c) { return 68 * k1 + c; }
    static constexpr int FOFF = 1184;
    __host__ __device__ static constexpr int fix(int l, int k2) { return FOFF + 19 * l + k2 + ((k2 >> 2) & 3); }
    __host__ __device__ static constexpr int pc(int k) { return k + (k >> 3) + 2 * (k >> 6); }
    static constexpr int SP = pc(N - 1) + 1;      // spare unit (lane 0's row-b pair 0)
    static_assert(SP < FOFF, "C and F regions overlap");
    static constexpr int SLOTU = (fix(L - 1, 15) + 1 + 7) & ~7;
    // transformed rows after the post-processing (doubles): mode position q of row a / b
    __host__ __device__ static constexpr int xa(int q) { return 2 * pc(q >> 1) + (q & 1); }
    __host__ __device__ static constexpr int xb(int q) { return (q < 2 ? 2 * SP : 2 * pc(N - (q >> 1))) + (q & 1); }
    static constexpr int XB = N;                  // phase-3 input rows: natural order, row b at N doubles
    static constexpr size_t SLOT_BYTES = size_t(SLOTU) * 16;
    static constexpr size_t OFF_AL = size_t(TEAMS) * SLOT_BYTES;
    static constexpr size_t OFF_SC = OFF_AL + size_t(N) * 8;   // per team: warp-0 scan totals
    static constexpr size_t SMEM = OFF_SC + size_t(TEAMS) * 16;
    static_assert(SMEM <= 227 * 1024, "shared memory");
    static_assert(NFW % 2 == 0, "two warps per team");
};

#ifdef FD_K3_DEBUG
__device__ __forceinline__ void mbar_wait_dbg(uint64_t *bar, uint32_t parity, int tag) {
    uint32_t done = 0;
    for (long long it = 0; !done; ++it) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 100000;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (it == 20000) {
            printf("k3 hang: cta %d tid %d tag %d parity %u\n", blockIdx.x, threadIdx.x, tag, parity);
            asm volatile("trap;");
        }
    }
}
#define MBAR_WAIT(b, par, tag) mbar_wait_dbg(b, par, tag)
#elif defined(FD_K3_SPIN)
__device__ __forceinline__ void mbar_wait_spin(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
#define MBAR_WAIT(b, par, tag) mbar_wait_spin(b, par)
#else
#define MBAR_WAIT(b, par, tag) mbar_wait(b, par)
#endif

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#define MBAR_ARRIVE(b) mbar_arrive(b)

// pre-weighted complex input of index j from the row values x_j, x_{N-j}
__device__ __forceinline__ double2 prew(double al, double h, double ao, double am, double bo, double bm) {
    const double b = al - h;
    return make_double2(fma(al, ao, b * am), fma(al, bo, b * bm));
}

// Row source of the transform: rows a and b through generic pointers -- the
// input rows in global memory (phase 1) or the x rows the S threads wrote into
// the slot in natural order (phase 3).  One instantiation of the transform
// serves both phases (instruction-cache footprint).
struct RowSrc {
    const double *a, *b;
    __device__ double ga(int q) const { return a[q]; }
    __device__ double gb(int q) const { return b[q]; }
};

// team barrier: the two warps of a row pair (named barrier 1 + team)
__device__ __forceinline__ void team_sync(int team) {
    asm volatile("bar.sync %0, 64;" ::"r"(1 + team) : "memory");
}

// Forward transform of one row pair by its team (64 lanes, lane t owns the
// residue class t of j mod 64): rows from src, result (transformed rows a, b;
// xa / xb layout) in the slot.  scr: the team's two scan doubles.
template <class C>
__device__ __forceinline__ void transform_pair(double2 *slot, const RowSrc src, const double *al, double h,
                                               const double2 *tw, int t, int team, double *scr, bool sync_in) {
    constexpr int N = C::N, Q = C::Q;
    static_assert(C::L == 64, "two warps per pair");
    double2 v[16];
    // ---- loads + pre-weighting: y_j = al_j x_j + (al_j - h) x_{N-j}, j = t + 64 r
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const int j = t + Q * r;
        const bool z = (j == 0);   // x_0 = x_N = 0
        const int po = z ? 0 : j - 1, pm = z ? 0 : N - j - 1;
        double ao = src.ga(po), am = src.ga(pm), bo = src.gb(po), bm = src.gb(pm);
        if (z) ao = am = bo = bm = 0.0;
        v[r] = prew(al[j], h, ao, am, bo, bm);
    }
    if (sync_in) team_sync(team);   // phase 3: the slot's rows are consumed before E overwrites them
    // ---- pass 1: radix 16 over r, twiddle W_N^{t k1}
    dft<16>(v);
    chain_twiddle<16>(v, tw[2 * t], 1.0);
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) slot[C::eix(k1, t)] = v[k1];
    team_sync(team);
    // ---- pass 2: lane (k1, c0) = (t >> 2, t & 3): radix 16 over c' (c = c0 + 4 c'),
    //      twiddle W_64^{c0 k2'}
    const int k1 = t >> 2, c0 = t & 3;
#pragma unroll
    for (int cp = 0; cp < 16; ++cp) v[cp] = slot[C::eix(k1, c0 + 4 * cp)];
    dft<16>(v);
    chain_twiddle<16>(v, tw[(2 * N / 64) * c0], 1.0);
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) slot[C::fix(t, k2)] = v[k2];
    team_sync(team);
    // ---- pass 3: radix 4 over c0 for k2' in [4 c0, 4 c0 + 4):
    //      C[k1 + 16 (k2' + 16 k3)] = sum_c0' W_4^{c0' k3} H_{c0'}[k2']
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k2 = 4 * c0 + i;
        double2 a0 = slot[C::fix(4 * k1 + 0, k2)], a1 = slot[C::fix(4 * k1 + 1, k2)];
        double2 a2 = slot[C::fix(4 * k1 + 2, k2)], a3 = slot[C::fix(4 * k1 + 3, k2)];
        dft4(a0, a1, a2, a3);
        const int k = k1 + 16 * k2;
        slot[C::pc(k)] = a0;
        slot[C::pc(k + 256)] = a1;
        slot[C::pc(k + 512)] = a2;
        slot[C::pc(k + 768)] = a3;
    }
    team_sync(team);
    // ---- post: lane t owns k in [8 t, 8 t + 8); it reads C_k from its "own"
    // units pc(8 t + i) and C_{N-k} from its "mirror" units pc(N - 8 t - i) and
    // writes the transformed rows back into exactly those units (row a: own,
    // row b: mirror; lane 0's missing mirror unit of k = 0 is the spare unit).
    //   pass A: lane totals of Re/Im (C_k + C_{N-k}), scan over the 64 lanes
    //   pass B: streamed outputs (D_k, e_{k+1}) per unit
    auto mir = [&](int i) { return (t == 0 && i == 0) ? C::SP : C::pc(N - 8 * t - i); };
    double ra = 0.0, rb = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const double2 c = slot[C::pc(8 * t + i)];
        const double2 c2 = (t == 0 && i == 0) ? make_double2(0.0, 0.0) : slot[mir(i)];
        ra += c.x + c2.x;
        rb += c.y + c2.y;
    }
    double2 cn = make_double2(0.0, 0.0), c2n = cn;   // k = 8 t + 8 (e_{N/2} = 0: position n is not a mode)
    if (t < Q - 1) {
        cn = slot[C::pc(8 * t + 8)];
        c2n = slot[C::pc(N - 8 * t - 8)];
    }
    const int lane = t & 31;
    double ia = ra, ib = rb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double xa = __shfl_up_sync(0xffffffffu, ia, o), xb = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) {
            ia += xa;
            ib += xb;
        }
    }
    if (t == 31) {
        scr[0] = ia;
        scr[1] = ib;
    }
    team_sync(team);   // every lane has read its C values (pass B writes) and warp 0's total is out
    double sa = ia - ra, sb = ib - rb;   // exclusive prefix of the lane
    if (t >= 32) {
        sa += scr[0];
        sb += scr[1];
    }
    double2 c = slot[C::pc(8 * t)];
    double2 c2 = (t == 0) ? make_double2(0.0, 0.0) : slot[mir(0)];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        sa += c.x + c2.x;
        sb += c.y + c2.y;
        double2 d = cn, d2 = c2n;
        if (i < 7) {
            d = slot[C::pc(8 * t + i + 1)];
            d2 = slot[mir(i + 1)];
        }
        slot[C::pc(8 * t + i)] = make_double2(sa, d2.y - d.y);
        slot[mir(i)] = make_double2(sb, d.x - d2.x);
        c = d;
        c2 = d2;
    }
}

// Factors of mode k at row i (rectsolver.py:62-77): rows i < ecap from the
// row-major tables of every mode, later rows of the slowly converging modes
// k < kt from the long-transient table (built without a cap for K3 lengths,
// so every other mode has reached its bitwise fixed point by row ecap), the
// rest from the per-mode fixed point; row m-1 carries the east modifier.
struct FwdF {
    double l, ib;
};
// the plan fields the factor lookups touch, held in registers per job (an S
// thread would otherwise re-read them from the launch parameters per call)
struct FacTab {
    const double *dl, *dib, *db, *lt, *last;
    int n, m, ecap, kt, ktp;
    double off, nio;
    __device__ void load(const PlanDev &p) {
        dl = p.dl;
        dib = p.dib;
        db = p.db;
        lt = p.lt;
        last = p.last;
        n = p.n;
        m = p.m;
        ecap = p.ecap;
        kt = p.kt;
        ktp = p.ktp;
        off = p.off;
        nio = p.nio;
    }
};
template <class P>
__device__ __forceinline__ FwdF fwd_factors(const P &p, int k, int i, double l_inf, double ib_inf) {
    if (i < p.ecap) return FwdF{__ldg(p.dl + size_t(i) * p.n + k), __ldg(p.dib + size_t(i) * p.n + k)};
    if (k < p.kt) {
        const double *tb = p.lt + size_t(i) * 3 * p.ktp + k;
        return FwdF{__ldg(tb), __ldg(tb + p.ktp)};
    }
    return FwdF{l_inf, (i == p.m - 1) ? __ldg(p.last + 2 * k + 1) : ib_inf};
}
// back-substitution factors: 1/beta_i and pm_i = -beta_{i-1}/delta
struct BwdF {
    double ib, pm;
};
template <class P>
__device__ __forceinline__ BwdF bwd_factors(const P &p, int k, int i, double ib_inf, double inv_nl) {
    BwdF f;
    const double *tb = p.lt + size_t(i) * 3 * p.ktp + k;
    if (i < p.ecap) f.ib = __ldg(p.dib + size_t(i) * p.n + k);
    else if (k < p.kt) f.ib = __ldg(tb + p.ktp);
    else f.ib = (i == p.m - 1) ? __ldg(p.last + 2 * k + 1) : ib_inf;
    if (i >= 1 && i - 1 < p.ecap) f.pm = __ldg(p.db + size_t(i - 1) * p.n + k) * p.nio;
    else if (k < p.kt) f.pm = __ldg(tb + 2 * p.ktp);
    else f.pm = inv_nl;
    return f;
}

__device__ __forceinline__ int seg_index(const int *pair0, int nseg, int p) {
    int si = 0;
    while (si + 1 < nseg && p >= pair0[si + 1]) ++si;
    return si;
}

// S role, phase 1: the reference forward elimination (rectsolver.py:86) over
// the CTA's rows in order, straight from the slots; yhat to the output array
// (coalesced: thread s owns modes s + NST u); block scalars at segment ends.
// Registers are tight (SREG): only the sweep state and the fixed-point
// factors live across pairs; mode group 0 (the slowly converging modes
// k < kt, which load a table row on every row) has its factors prefetched one
// pair ahead; the other groups load only in rows i < ecap and the last row.
#ifndef FD_K3_SKIP
#define FD_K3_SKIP 0
#endif
template <class C>
__device__ __noinline__ void s_forward(const PList &pl, const Seg *segs, const int *pair0, int nseg, int npairs,
                                          uint64_t *full, uint64_t *empty, unsigned char *smem_raw, int st) {
    constexpr int U = C::U, NST = C::NST, TEAMS = C::TEAMS;
    const int n = pl.n;
    double ys[U], ws[U], fs[U], s2s[U], l_inf[U], ib_inf[U];
    int cur_job = -1;
    FacTab ft;
    FwdF pf0{0.0, 0.0}, pf1{0.0, 0.0};
    auto valid = [&](int uu) { return uu < U - 1 || st + NST * uu < n; };
    auto prefetch = [&](int p) {
        if (p >= npairs) return;
        const int si = seg_index(pair0, nseg, p);
        if (segs[si].job != cur_job) return;   // job change: fetched after the constants
        const int r0 = segs[si].s + 2 * (p - pair0[si]);
        pf0 = fwd_factors(ft, st, r0, l_inf[0], ib_inf[0]);
        if (r0 + 1 <= segs[si].e) pf1 = fwd_factors(ft, st, r0 + 1, l_inf[0], ib_inf[0]);
    };
#pragma unroll 1
    for (int p = 0; p < npairs; ++p) {
        const int si = seg_index(pair0, nseg, p);
        const int job = segs[si].job, s0 = segs[si].s, e0 = segs[si].e;
        const int r0 = s0 + 2 * (p - pair0[si]);
        const int rows = min(2, e0 - r0 + 1);
        const PlanDev &pd = pl.job[job].p;
        if (job != cur_job) {
            cur_job = job;
            ft.load(pd);
#pragma unroll
            for (int uu = 0; uu < U; ++uu)
                if (valid(uu)) {
                    const double2 a = __ldg(reinterpret_cast<const double2 *>(pd.mode) + 4 * (st + NST * uu));
                    l_inf[uu] = a.x;
                    ib_inf[uu] = a.y;
                }
            prefetch(p);
        }
        const int mlast = ft.m - 1, ecap = ft.ecap, kt = ft.kt;
        const int sl = p % TEAMS;
        MBAR_WAIT(&full[sl], (p / TEAMS) & 1, 2);
        const double *X = reinterpret_cast<const double *>(smem_raw + size_t(sl) * C::SLOT_BYTES);
        double *og = pl.job[job].out + size_t(r0) * n + st;
#pragma unroll
        for (int r = 0; r < 2 * !(FD_K3_SKIP & 2); ++r) {
            if (r >= rows) break;
            const int i = r0 + r;
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                if (!valid(uu)) continue;
                const int k = st + NST * uu;
                const double xv = X[r ? C::xb(k) : C::xa(k)];
                FwdF f;
                if (FD_K3_SKIP & 4) f = FwdF{l_inf[uu], ib_inf[uu]};
                else if (uu == 0) f = r ? pf1 : pf0;
                else if (i < ecap || i == mlast || k < kt) f = fwd_factors(ft, k, i, l_inf[uu], ib_inf[uu]);
                else f = FwdF{l_inf[uu], ib_inf[uu]};
                if (i == s0) {   // block start: y = r, pi = 1
                    ys[uu] = xv;
                    ws[uu] = 1.0;
                    fs[uu] = xv * f.ib;
                    s2s[uu] = f.ib;
                } else {
                    const double y = __dsub_rn(xv, __dmul_rn(f.l, ys[uu]));
                    const double w = -f.l * ws[uu];
                    const double W = w * f.ib;
                    fs[uu] = fma(y, W, fs[uu]);
                    s2s[uu] = fma(w, W, s2s[uu]);
                    ys[uu] = y;
                    ws[uu] = w;
                }
                og[size_t(r) * n + NST * uu] = ys[uu];
            }
        }
        MBAR_ARRIVE(&empty[sl]);
        prefetch(p + 1);   // group-0 factors of the next pair: loads in flight across the next wait
        if (r0 + rows - 1 == e0) {   // block end: scalars for the carries (phase 2)
            const int blk = segs[si].blk;
#pragma unroll 1
            for (int uu = 0; uu < U; ++uu) {
                if (!valid(uu)) continue;
                const int k = st + NST * uu;
                double y = ys[0], w = ws[0], f = fs[0], s2 = s2s[0];
#pragma unroll
                for (int q = 1; q < U; ++q)
                    if (uu == q) {
                        y = ys[q];
                        w = ws[q];
                        f = fs[q];
                        s2 = s2s[q];
                    }
                double *cb = pl.carry + size_t(blk) * kCarryVals * n + k;
                const double lnext = (e0 < mlast) ? fwd_factors(ft, k, e0 + 1, l_inf[uu], ib_inf[uu]).l : 0.0;
                const double cc = (s0 == 0) ? 0.0 : -fwd_factors(ft, k, s0, l_inf[uu], ib_inf[uu]).l;   // -l_s
                __stcg(cb + 0 * n, y);
                __stcg(cb + 1 * n, f);
                __stcg(cb + 2 * n, cc * w);
                __stcg(cb + 3 * n, cc * s2);
                __stcg(cb + 4 * n, (e0 < mlast) ? w * (-lnext) : 0.0);
            }
        }
    }
}

// S role, phase 3: pairs of a segment from its last row down; carry fix-up
// and the reference back-substitution (rectsolver.py:90) of yhat (prefetched
// one pair ahead), x into the slot in natural order for the F team.
template <class C>
__device__ __noinline__ void s_backward(const PList &pl, const Seg *segs, const int *pair0, int nseg, int npairs,
                                           uint64_t *full, uint64_t *empty, unsigned char *smem_raw, int st) {
    constexpr int U = C::U, NST = C::NST, TEAMS = C::TEAMS;
    const int n = pl.n;
    double xs[U], pcs[U], yins[U], ib_inf[U], inv_nl[U];
    int cur_job = -1;
    FacTab ft;
    BwdF pf0{0.0, 0.0}, pf1{0.0, 0.0};
    double py0[U], py1[U];
    auto valid = [&](int uu) { return uu < U - 1 || st + NST * uu < n; };
    auto prefetch = [&](int p) {
        if (p >= npairs || (FD_K3_SKIP & 8)) return;
        const int si = seg_index(pair0, nseg, p);
        const int rh = segs[si].e - 2 * (p - pair0[si]);
        const bool two = rh - 1 >= segs[si].s;
        const double *yr = pl.job[segs[si].job].out + size_t(rh) * n + st;
#pragma unroll
        for (int uu = 0; uu < U; ++uu)
            if (valid(uu)) {
                py0[uu] = __ldcg(yr + NST * uu);
                if (two) py1[uu] = __ldcg(yr - n + NST * uu);
            }
        if (segs[si].job != cur_job) return;
        pf0 = bwd_factors(ft, st, rh, ib_inf[0], inv_nl[0]);
        if (two) pf1 = bwd_factors(ft, st, rh - 1, ib_inf[0], inv_nl[0]);
    };
    prefetch(0);
#pragma unroll 1
    for (int p = 0; p < npairs; ++p) {
        const int si = seg_index(pair0, nseg, p);
        const int job = segs[si].job, s0 = segs[si].s, e0 = segs[si].e, blk = segs[si].blk;
        const int rh = e0 - 2 * (p - pair0[si]);
        const int rows = min(2, rh - s0 + 1);
        const PJob &J = pl.job[job];
        const PlanDev &pd = J.p;
        if (job != cur_job) {
            cur_job = job;
            ft.load(pd);
#pragma unroll
            for (int uu = 0; uu < U; ++uu)
                if (valid(uu)) {
                    const double2 *rec = reinterpret_cast<const double2 *>(pd.mode) + 4 * (st + NST * uu);
                    ib_inf[uu] = __ldg(rec).y;
                    inv_nl[uu] = __ldg(rec + 1).y;
                }
            pf0 = bwd_factors(ft, st, rh, ib_inf[0], inv_nl[0]);
            if (rows > 1) pf1 = bwd_factors(ft, st, rh - 1, ib_inf[0], inv_nl[0]);
        }
        const bool has_in = blk > J.blk_base;                 // block does not start at row 0
        if (p == pair0[si]) {                                 // top of the block: carries from phase 2
            const bool has_next = blk < J.blk_base + J.nblk - 1;   // a block below carries X
            const size_t bs = size_t(kCarryVals) * n;
            const double *cb = pl.carry + size_t(blk) * bs + st;
#pragma unroll
            for (int uu = 0; uu < U; ++uu)
                if (valid(uu)) {
                    xs[uu] = has_next ? __ldcg(cb + bs + 6 * n + NST * uu) : 0.0;
                    yins[uu] = has_in ? __ldcg(cb - bs + 5 * n + NST * uu) : 0.0;
                    pcs[uu] = __ldcg(cb + 2 * n + NST * uu);
                }
        }
        const int mlast = ft.m - 1, ecap = ft.ecap, kt = ft.kt;
        const double off = ft.off;
        const int sl = p % TEAMS;
        MBAR_WAIT(&empty[sl], ((p / TEAMS) & 1) ^ 1, 3);
        double *X = reinterpret_cast<double *>(smem_raw + size_t(sl) * C::SLOT_BYTES) + st;
#pragma unroll
        for (int r = 0; r < 2 * !(FD_K3_SKIP & 2); ++r) {
            if (r >= rows) break;
            const int i = rh - r;
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                if (!valid(uu)) continue;
                const int k = st + NST * uu;
                BwdF f;
                if (FD_K3_SKIP & 4) f = BwdF{ib_inf[uu], inv_nl[uu]};
                else if (uu == 0) f = r ? pf1 : pf0;
                else if (i <= ecap || i == mlast || k < kt) f = bwd_factors(ft, k, i, ib_inf[uu], inv_nl[uu]);
                else f = BwdF{ib_inf[uu], inv_nl[uu]};
                double y = (FD_K3_SKIP & 8) ? xs[uu] : (r ? py1[uu] : py0[uu]);
                if (has_in) {
                    y = fma(pcs[uu], yins[uu], y);
                    pcs[uu] *= f.pm;   // P_{i-1} = P_i / (-l_i)
                }
                const double x = __dsub_rn(y, __dmul_rn(off, xs[uu])) * f.ib;   // rectsolver.py:90
                xs[uu] = x;
                X[r * C::XB + NST * uu] = x;
            }
        }
        MBAR_ARRIVE(&full[sl]);
        prefetch(p + 1);   // yhat rows and group-0 factors of the next pair
    }
}

// F role of one phase (phase 1: DST of the input rows into the slots; phase
// 3: inverse DST of the S threads' x rows and the epilogue).  Out of line,
// like the S roles: each role gets the whole register file to itself.
template <class C>
__device__ __noinline__ void f_role(const PList &pl, int ph, const Seg *segs, const int *pair0, int nseg, int npairs,
                                    uint64_t *full, uint64_t *empty, unsigned char *smem_raw, int team, int t) {
    constexpr int TEAMS = C::TEAMS, L = C::L;
    const int n = pl.n;
    const double *al = reinterpret_cast<const double *>(smem_raw + C::OFF_AL);
    const double2 *tw = pl.job[0].p.tw;   // e^{-2 pi i q / 2N}
    auto slot_of = [&](int q) { return reinterpret_cast<double2 *>(smem_raw + size_t(q) * C::SLOT_BYTES); };
    auto seg_of = [&](int p) { return seg_index(pair0, nseg, p); };
    int u = 0;
    for (int p = team; p < npairs; p += TEAMS, ++u) {
        const int si = seg_of(p);
        const Seg &sg = segs[si];
        const PJob &J = pl.job[sg.job];
        // phase 1 pairs run up from the segment start, phase 3 pairs down
        // from its end: (e, e-1), (e-2, e-3), ...
        const int rb = ph ? sg.e - 2 * (p - pair0[si]) : sg.s + 2 * (p - pair0[si]);
        const int rows = ph ? min(2, rb - sg.s + 1) : min(2, sg.e - rb + 1);
        double2 *slot = slot_of(team);
        const double *X = reinterpret_cast<const double *>(slot);
        RowSrc src;
        if (ph == 0) {
            MBAR_WAIT(&empty[team], (u & 1) ^ 1, 1);
            src.a = J.in + size_t(rb) * n;
            src.b = rows > 1 ? src.a + n : src.a;
        } else {
            MBAR_WAIT(&full[team], u & 1, 4);
            src.a = X;
            src.b = rows > 1 ? X + C::XB : X;
        }
#ifndef FD_K3_SKIP
#define FD_K3_SKIP 0
#endif
        if (!(FD_K3_SKIP & 1))   // timing experiments only (results invalid)
        transform_pair<C>(slot, src, al, 0.5 * J.p.scale, tw, t, team,
                          reinterpret_cast<double *>(smem_raw + C::OFF_SC) + 2 * team, ph == 1);
        if (ph == 0) {
            mbar_arrive(&full[team]);
            continue;
        }
        team_sync(team);   // both warps' rows are in the slot
        // epilogue out = alpha x + beta other, coalesced rows
        const double a_ = J.alpha, b_ = J.beta;
        for (int h = 0; h < rows; ++h) {
            double *oh = J.out + size_t(rb - h) * n;
            const double *qh = J.other ? J.other + size_t(rb - h) * n : nullptr;
            auto xv = [&](int q) { return X[h ? C::xb(q) : C::xa(q)]; };
            if (qh) {
#pragma unroll 4
                for (int q = t; q < n; q += L) oh[q] = fma(b_, __ldg(qh + q), a_ * xv(q));
            } else if (a_ == 1.0) {
#pragma unroll 4
                for (int q = t; q < n; q += L) oh[q] = xv(q);
            } else {
#pragma unroll 4
                for (int q = t; q < n; q += L) oh[q] = a_ * xv(q);
            }
        }
        mbar_arrive(&empty[team]);
    }
}

template <int NL>
__global__ void __launch_bounds__(512, 1) k3_kernel(const __grid_constant__ PList pl) {
    using C = Cfg<NL>;
    constexpr int N = C::N, TEAMS = C::TEAMS, U = C::U, NST = C::NST, L = C::L;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    auto slot_of = [&](int q) { return reinterpret_cast<double2 *>(smem_raw + size_t(q) * C::SLOT_BYTES); };
    double *al = reinterpret_cast<double *>(smem_raw + C::OFF_AL);
    __shared__ __align__(8) uint64_t full[TEAMS], empty[TEAMS];
    __shared__ Seg segs[kMaxSegs];
    __shared__ int pair0[kMaxSegs + 1];
    __shared__ int nseg_s;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n = pl.n;
    cg::grid_group grid = cg::this_grid();
    auto stamp = [&](int slot) {   // FD_PHASE_TIMING (launcher): per-CTA phase timestamps
        if (pl.tstamp && tid == 0) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
            pl.tstamp[blockIdx.x * 8 + slot] = g;
        }
    };
    stamp(0);

    if (tid == 0) {
        int ns = 0, np = 0;
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
                    sg.item0 = np;
                    pair0[ns] = np;
                    np += sg.ngroups;
                    segs[ns++] = sg;
                }
            }
        }
        nseg_s = ns;
        pair0[ns] = np;
        for (int q = 0; q < TEAMS; ++q) {
            mbar_init(&full[q], L);
            mbar_init(&empty[q], NST);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    {
        const double *ra = pl.job[0].p.ralpha;
        for (int q = tid; q < N; q += C::NT) al[q] = __ldg(ra + q);
    }
    __syncthreads();
    const int nseg = nseg_s, npairs = pair0[nseg];
    const double2 *tw = pl.job[0].p.tw;   // e^{-2 pi i q / 2N}
    auto seg_of = [&](int p) {
        int si = 0;
        while (si + 1 < nseg && p >= pair0[si + 1]) ++si;
        return si;
    };
    const bool isF = warp < C::NFW;
    const int team = (tid / L), t = tid % L;      // F roles
    const int st = tid - C::NFW * 32;             // S roles

    // Phase 1 (ph = 0): DST + local forward elimination; phase 2: block
    // carries; phase 3 (ph = 1): back-substitution + inverse DST.  The F role
    // is one loop over both phases so the transform is inlined once
    // (instruction-cache footprint).
#pragma unroll 1
    for (int ph = 0; ph < 2; ++ph) {
        if (ph == 1) {
            // Give the registers back only after the F warps have released
            // theirs: an S warp that grew back at once could take the registers
            // a still-pending F setmaxnreg.inc is waiting for (a CTA without
            // rows gets there first).
            __syncthreads();
            stamp(1);
            __threadfence();
            stamp(6);
            grid.sync();
            stamp(2);
            // ===================== phase 2: block carries =============================
            carries_phase<C::NT>(pl, smem_raw, C::OFF_AL, tid, lane);
            stamp(3);
            grid.sync();
            stamp(4);
            // re-arm the slot barriers with the phase-3 roles (S fills, F drains)
            if (tid == 0) {
                for (int q = 0; q < TEAMS; ++q) {
                    mbar_init(&full[q], NST);
                    mbar_init(&empty[q], L);
                }
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            }
            __syncthreads();
        }
        if (isF) {
            f_role<C>(pl, ph, segs, pair0, nseg, npairs, full, empty, smem_raw, team, t);
        } else if (ph == 0) {
            s_forward<C>(pl, segs, pair0, nseg, npairs, full, empty, smem_raw, st);
        } else {
            s_backward<C>(pl, segs, pair0, nseg, npairs, full, empty, smem_raw, st);
        }
    }
    // registers are released at exit: no rebalancing after phase 3
    __syncthreads();
    stamp(5);
}

// Test entry: one team transforms rows (a, b) of length N - 1 into the DST-I
// of both rows (xa / xb layouts read back into natural order).
template <int NL>
__global__ void __launch_bounds__(64) k3_transform_test(const double *a, const double *b, double *oa, double *ob,
                                                        const double *ralpha, const double2 *tw, double scale) {
    using C = Cfg<NL>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *slot = reinterpret_cast<double2 *>(smem_raw);
    double *al = reinterpret_cast<double *>(smem_raw + C::SLOT_BYTES);
    double *scr = al + C::N;
    for (int q = threadIdx.x; q < C::N; q += 64) al[q] = ralpha[q];
    __syncthreads();
    transform_pair<C>(slot, RowSrc{a, b}, al, 0.5 * scale, tw, threadIdx.x, 0, scr, false);
    __syncthreads();
    const double *X = reinterpret_cast<const double *>(slot);
    for (int q = threadIdx.x; q < C::N - 1; q += 64) {
        oa[q] = X[C::xa(q)];
        ob[q] = X[C::xb(q)];
    }
}

template <int NL>
struct K3K {
    static constexpr int NT = Cfg<NL>::NT, G = 2;
    static constexpr size_t SMEM = Cfg<NL>::SMEM;
    static const void *fn() { return (const void *)k3_kernel<NL>; }
};

}  // namespace k3

// debug/test hook: the K3 row-pair transform of one pair (n = 1023)
void k3_test_transform(const double *a, const double *b, double *oa, double *ob, const double *ralpha,
                       const double2 *tw, double scale, cudaStream_t s) {
    using C = k3::Cfg<10>;
    const size_t smem = C::SLOT_BYTES + C::N * 8 + 16;
    FD_CUDA(cudaFuncSetAttribute(k3::k3_transform_test<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k3::k3_transform_test<10><<<1, 64, smem, s>>>(a, b, oa, ob, ralpha, tw, scale);
    FD_CUDA(cudaGetLastError());
}

// the warp-specialised solve for the lengths it is built for; false otherwise
bool launch_k3(const std::vector<SolveJob> &jobs, cudaStream_t s, Workspace &ws) {
    const int n = jobs[0].p.n;
    if (!jobs[0].p.ralpha) return false;
    switch (n + 1) {
        case 1024: run_persist<k3::K3K<10>>(jobs, s, ws); return true;
        default: return false;
    }
}

}  // namespace fd
