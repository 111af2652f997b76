// Persistent fused rectangle solve for n + 1 = N = 1024 with warp-private
// transforms (the c1 / BASELINE config-1 length).
//
// Same mathematics and the same three phases as rsolve.cu (real-symmetric
// DST-I + local forward elimination | block carries | back-substitution +
// inverse DST-I, rectsolver.py:183-213), but the data flow is rebuilt around
// one warp per row pair:
//
//   * a row pair's N-point complex FFT lives in ONE warp: 32 points per lane,
//     N = 32 x 32 four-step (a 32-point DFT in registers over j = lane + 32 r,
//     the W_N^{lane k1} twiddle, one transpose through the warp's own shared
//     region, a second 32-point DFT) -- one shared-memory exchange per
//     transform instead of three radix passes, and no CTA or named barriers
//     inside the transform (only __syncwarp);
//   * phase-1 rows are read straight from HBM into registers (coalesced over
//     the lanes, the mirror x_{N-j} from the same lines), no TMA staging;
//   * the post-processing (mirror pairs + the odd-output prefix sum) gives each
//     lane a contiguous run of 16 k's and writes the transformed pair IN PLACE
//     into the 32 slots that lane read ("xslot" permutation below, both rows of
//     a mode in one 16-byte slot), so the mode-parallel sweep reads two rows
//     per LDS.128 and the epilogue stores rows coalesced;
//   * small CTAs (4 warps = 4 pairs = 8 rows per wave, 70 KB of shared
//     memory), several per SM, so one CTA's loads, barriers and sweeps overlap
//     another's transforms.
// The sweeps keep the reference recurrence row order inside each block
// (rectsolver.py:86,90); the block carries are the ones of rsolve.cu.
// ARCHIVED (not built into the library): measured slower than rsolve.cu, see
// tools/experimental/README.md.  Builds only inside the library tree
// (copy to paper_2509_23180_b200/csrc/ and add its dispatch to solve.cu).
#include "../../paper_2509_23180_b200/csrc/rsolve_common.cuh"

namespace fd {
namespace r32 {

constexpr int N = 1024;      // transform length n + 1
constexpr int W = 4;         // warps (= row pairs) per CTA
constexpr int NT = 32 * W;   // threads per CTA
constexpr int G = 2 * W;     // rows per wave
constexpr int MPT = (N - 1 + NT - 1) / NT;   // modes per thread in the sweeps
constexpr int SLOTS = 1088;  // phys(1023) + 1 >= 32 * 33 (exchange)
constexpr size_t REG = size_t(SLOTS) * 16;
constexpr size_t OFF_ST = size_t(W) * REG;   // per-thread sweep state [5][MPT][NT] doubles
constexpr size_t SMEM = OFF_ST + size_t(5) * MPT * NT * 8;

// padded slot index: 16-byte slots, one pad slot per 16 (lane-contiguous runs
// of 16 slots land on distinct bank groups)
__device__ __forceinline__ int phys(int s) { return s + (s >> 4); }
// slot of transform output position p (X_{p+1}, p = 0..N-2):
//   X_{2k}   (p = 2k - 1) -> slot k              (k = 1..N/2-1)
//   X_{2k+1} (p = 2k)     -> slot N - k (k >= 1), N/2 (k = 0)
// i.e. exactly the slots C_k / C_{N-k} the post-processing lane read.
__device__ __forceinline__ int xslot(int p) { return (p & 1) ? ((p + 1) >> 1) : (p == 0 ? N / 2 : N - (p >> 1)); }

// cos(pi a / 32), a = 0..16, correctly rounded
__device__ __forceinline__ constexpr double c32(int a) {
    constexpr double c[17] = {0x1.0000000000000p+0, 0x1.fd88da3d12526p-1, 0x1.f6297cff75cb0p-1,
                              0x1.e9f4156c62ddap-1, 0x1.d906bcf328d46p-1, 0x1.c38b2f180bdb1p-1,
                              0x1.a9b66290ea1a3p-1, 0x1.8bc806b151741p-1, 0x1.6a09e667f3bcdp-1,
                              0x1.44cf325091dd6p-1, 0x1.1c73b39ae68c8p-1, 0x1.e2b5d3806f63bp-2,
                              0x1.87de2a6aea963p-2, 0x1.294062ed59f06p-2, 0x1.8f8b83c69a60bp-3,
                              0x1.917a6bc29b42cp-4, 0.0};
    return c[a];
}
// cos / sin of pi a / 32 for a = 0..31
__device__ __forceinline__ constexpr double cosa(int a) { return a <= 16 ? c32(a) : -c32(32 - a); }
__device__ __forceinline__ constexpr double sina(int a) { return a <= 16 ? c32(16 - a) : c32(a - 16); }

// a * W_32^P = a * e^{-2 pi i P / 32}, P = 0..15 known at compile time
template <int P>
__device__ __forceinline__ double2 tw32(double2 a) {
    if constexpr ((P & 1) == 0) return tw16<P / 2>(a);
    else return cmul(a, make_double2(cosa(2 * P), -sina(2 * P)));
}

// forward 32-point DFT in registers, natural order in and out
__device__ __forceinline__ void dft32(double2 (&v)[32]) {
    double2 e[16], o[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        e[i] = v[2 * i];
        o[i] = v[2 * i + 1];
    }
    dft<16>(e);
    dft<16>(o);
    o[1] = tw32<1>(o[1]);
    o[2] = tw32<2>(o[2]);
    o[3] = tw32<3>(o[3]);
    o[4] = tw32<4>(o[4]);
    o[5] = tw32<5>(o[5]);
    o[6] = tw32<6>(o[6]);
    o[7] = tw32<7>(o[7]);
    o[8] = tw32<8>(o[8]);
    o[9] = tw32<9>(o[9]);
    o[10] = tw32<10>(o[10]);
    o[11] = tw32<11>(o[11]);
    o[12] = tw32<12>(o[12]);
    o[13] = tw32<13>(o[13]);
    o[14] = tw32<14>(o[14]);
    o[15] = tw32<15>(o[15]);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        v[k] = cadd(e[k], o[k]);
        v[k + 16] = csub(e[k], o[k]);
    }
}

// Per-lane constants of the transform: sin/cos(pi lane / N) for the
// pre-weights, W_N^lane for the four-step twiddle.
struct LaneK {
    double sl, cl;
    double2 wl;
    __device__ void init(int lane) {
        sincospi(double(lane) / N, &sl, &cl);
        double s2, c2;
        sincospi(double(lane) / (N / 2), &s2, &c2);
        wl = make_double2(c2, -s2);
    }
    // pre-weight alpha_j = s/2 sin(pi j / N) + s/4 at j = lane + 32 r
    __device__ __forceinline__ double alpha(int r, double h2) const {
        const double sj = fma(sl, cosa(r), cl * sina(r));
        return fma(h2, sj, 0.5 * h2);
    }
};

// FFT of the pre-weighted pair c (v[r] = c_{lane + 32 r}) and the
// real-symmetric post-processing; on return the warp's region holds the
// transformed rows in the xslot layout (.x = row a, .y = row b).
__device__ __forceinline__ void transform(double2 (&v)[32], double2 *reg, int lane, const LaneK &lk) {
    dft32(v);                      // over r: lane holds V_lane[k1], k1 = 0..31
    apply_powers<32>(v, lk.wl);    // * W_N^{lane k1}
#pragma unroll
    for (int k1 = 0; k1 < 32; ++k1) reg[k1 * 33 + lane] = v[k1];
    __syncwarp();
#pragma unroll
    for (int l = 0; l < 32; ++l) v[l] = reg[lane * 33 + l];
    __syncwarp();
    dft32(v);                      // over l: lane k1 holds C_{k1 + 32 k2} at v[k2]
#pragma unroll
    for (int k2 = 0; k2 < 32; ++k2) reg[phys(lane + 32 * k2)] = v[k2];
    __syncwarp();
    // post: lane owns k = 16 lane + i.  X_{2k} = (Im C_{N-k} - Im C_k, Re C_k - Re C_{N-k}),
    // X_{2k+1} = sum_{k' <= k} d_{k'},  d_0 = C_0, d_k = C_k + C_{N-k}
    double da[16], db[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int k = 16 * lane + i;
        const double2 c = reg[phys(k)];
        double2 c2 = make_double2(0.0, 0.0);
        if (i > 0 || lane > 0) c2 = reg[phys(N - k)];
        da[i] = c.x + c2.x;
        db[i] = c.y + c2.y;
        if (i > 0 || lane > 0) reg[phys(k)] = make_double2(c2.y - c.y, c.x - c2.x);
    }
#pragma unroll
    for (int i = 1; i < 16; ++i) {
        da[i] += da[i - 1];
        db[i] += db[i - 1];
    }
    double ia = da[15], ib = db[15];
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
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int k = 16 * lane + i;
        const int s = (i == 0 && lane == 0) ? N / 2 : N - k;
        reg[phys(s)] = make_double2(da[i] + pa, db[i] + pb);
    }
    __syncwarp();
}

// Phase-1 transform of rows A, B (B = A for a single row) read from HBM.  Out
// of line: the kernel's sweep state does not compete with the 32 complex
// points per lane for registers.
__device__ __noinline__ void xform_global(const double *A, const double *B, double h2, double2 *reg, int lane,
                                          LaneK lk) {
    double2 v[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
        const int j = lane + 32 * r;
        if (r == 0 && lane == 0) {
            v[0] = make_double2(0.0, 0.0);
            continue;
        }
        const double a = lk.alpha(r, h2), b = a - h2;
        v[r].x = fma(a, __ldg(A + j - 1), b * __ldg(A + (N - 1 - j)));
        v[r].y = fma(a, __ldg(B + j - 1), b * __ldg(B + (N - 1 - j)));
    }
    transform(v, reg, lane, lk);
}
// Phase-3 transform of the swept pair held in the region (xslot layout).
__device__ __noinline__ void xform_region(double h2, double2 *reg, int lane, LaneK lk) {
    double2 v[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
        const int j = lane + 32 * r;
        if (r == 0 && lane == 0) {
            v[0] = make_double2(0.0, 0.0);
            continue;
        }
        const double a = lk.alpha(r, h2), b = a - h2;
        const double2 x1 = reg[phys(xslot(j - 1))], x2 = reg[phys(xslot(N - 1 - j))];
        v[r] = make_double2(fma(a, x1.x, b * x2.x), fma(a, x1.y, b * x2.y));
    }
    __syncwarp();   // every lane has its inputs before the exchange overwrites them
    transform(v, reg, lane, lk);
}

}  // namespace r32


// Rare paths (only when the plan's row-major transient table was capped):
// one wave of one mode with the factors rebuilt row by row (factors_slow).
// Kept out of line so the unrolled fast paths carry no call.
static __device__ __noinline__ void r32_p1_slow(const PlanDev &p, int k, int g0, int rows, bool first, int len,
                                               double l_inf, double ib_inf, const unsigned char *smem, int xs,
                                               double *og, double *st) {
    using namespace r32;
    const int n = p.n;
    const double ibl = 1.0 / mode_blast(p, k);
    double y = st[0], w = st[MPT * NT], f = st[2 * MPT * NT], s2 = st[3 * MPT * NT];
    for (int q = 0; q < rows; ++q) {
        const double2 t = reinterpret_cast<const double2 *>(smem + size_t(q >> 1) * REG)[xs];
        const double xq = (q & 1) ? t.y : t.x;
        double l, ib, bm1;
        factors_slow(p, k, g0 + q, len, l_inf, ib_inf, ibl, 0.0, &l, &ib, &bm1);
        if (q == 0 && first) {
            y = xq;
            w = 1.0;
            f = y * ib;
            s2 = ib;
            st[4 * MPT * NT] = (g0 == 0) ? 0.0 : -l;
        } else {
            y = __dsub_rn(xq, __dmul_rn(l, y));
            w = -l * w;
            const double Wq = w * ib;
            f = fma(y, Wq, f);
            s2 = fma(w, Wq, s2);
        }
        og[size_t(q) * n] = y;
    }
    st[0] = y;
    st[MPT * NT] = w;
    st[2 * MPT * NT] = f;
    st[3 * MPT * NT] = s2;
}
static __device__ __noinline__ void r32_p3_slow(const PlanDev &p, int k, int g0, int rows, bool has_in, int len,
                                               double ib_inf, double iblast, const double *yg, double *smem, int xs,
                                               double *st) {
    using namespace r32;
    const int n = p.n;
    const double nio = -1.0 / p.off;
    double x = st[0], Pc = st[MPT * NT];
    const double yin = st[2 * MPT * NT];
    for (int q = rows - 1; q >= 0; --q) {
        double l, ib, bm1;
        factors_slow(p, k, g0 + q, len, 0.0, ib_inf, iblast, mode_binf(p, k), &l, &ib, &bm1);
        double y = __ldcg(yg + size_t(q) * n);
        if (has_in) {
            y = fma(Pc, yin, y);
            Pc *= bm1 * nio;
        }
        x = __dsub_rn(y, __dmul_rn(p.off, x)) * ib;   // rectsolver.py:90
        double *dst = reinterpret_cast<double *>(reinterpret_cast<double2 *>(smem + size_t(q >> 1) * (REG / 8)) + xs);
        dst[q & 1] = x;
    }
    st[0] = x;
    st[MPT * NT] = Pc;
}

template <int CTAS>
__global__ void __launch_bounds__(r32::NT, CTAS) rsolve32_kernel(const __grid_constant__ PList pl) {
    using namespace r32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    auto regc = [&](int q) { return reinterpret_cast<double2 *>(smem_raw + size_t(q) * REG); };
    __shared__ Seg segs[kMaxSegs];
    __shared__ int nseg_s, nitems_s;

    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    const int n = pl.n;
    cg::grid_group grid = cg::this_grid();
    auto stamp = [&](int slot) {   // FD_PHASE_TIMING
        if (pl.tstamp && tid == 0) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
            pl.tstamp[blockIdx.x * 8 + slot] = g;
        }
    };
    stamp(0);

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
    }
    __syncthreads();
    const int nseg = nseg_s, nitems = nitems_s;
    LaneK lk;
    lk.init(lane);
    double2 *myreg = regc(wp);
    // sweep state of mode u of this thread, value v: st[(v * MPT + u) * NT + tid]
    double *st = reinterpret_cast<double *>(smem_raw + OFF_ST) + tid;
    auto S = [&](int v, int u) -> double & { return st[(v * MPT + u) * NT]; };

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
#pragma unroll 1
    for (int it = 0; it < nitems; ++it) {
        int si, g0, rows;
        item_of(it, si, g0, rows, false);
        const Seg sg = segs[si];
        const PJob &J = pl.job[sg.job];
        const PlanDev &p = J.p;
        const int rp = min(2, rows - 2 * wp);
        if (rp > 0) {
            // rows straight from HBM: c_j = y_a(j) + i y_b(j), j = lane + 32 r
            const double *A = J.in + size_t(g0 + 2 * wp) * n;
            xform_global(A, rp > 1 ? A + n : A, 0.5 * p.scale, myreg, lane, lk);
        }
        __syncthreads();   // every pair of the wave transformed
        const bool first = (g0 == sg.s), last = (g0 + rows - 1 == sg.e);
        double *outg = J.out + size_t(g0) * n;
        const int mlast = p.m - 1;
#pragma unroll
        for (int u = 0; u < MPT; ++u) {
            const int k = tid + u * NT;
            if (k >= n) continue;
            const double2 *rec = reinterpret_cast<const double2 *>(p.mode) + 4 * k;
            const double2 ra = __ldg(rec), rd = __ldg(rec + 3);
            const double l_inf = ra.x, ib_inf = ra.y;
            const int len = int(__double_as_longlong(rd.y));
            const int xs = phys(xslot(k));
            double *og = outg + k;
            double *su = &S(0, u);
            if (k >= p.kt && g0 < len && min(g0 + rows, len) > p.ecap) {
                r32_p1_slow(p, k, g0, rows, first, len, l_inf, ib_inf, smem_raw, xs, og, su);
            } else {
                const double ibm = (g0 + rows - 1 >= mlast) ? 1.0 / mode_blast(p, k) : ib_inf;
                // this wave's transformed values of mode k, two rows per slot
                double xv[G];
#pragma unroll
                for (int q = 0; q < G; q += 2) {
                    if (q < rows) {
                        const double2 t = regc(q >> 1)[xs];
                        xv[q] = t.x;
                        xv[q + 1] = t.y;
                    }
                }
                // factors (l_i, 1/beta_i) of the wave's rows (rectsolver.py:72-73)
                double lv[G], ibv[G];
                if (k < p.kt) {
                    const double *tb = p.lt + size_t(g0) * 3 * p.ktp + k;
#pragma unroll
                    for (int q = 0; q < G; ++q)
                        if (q < rows) {
                            lv[q] = __ldg(tb + size_t(q) * 3 * p.ktp);
                            ibv[q] = __ldg(tb + size_t(q) * 3 * p.ktp + p.ktp);
                        }
                } else if (g0 < len) {
#pragma unroll
                    for (int q = 0; q < G; ++q)
                        if (q < rows) {
                            const int i = g0 + q;
                            const bool tr = i < len;
                            lv[q] = tr ? __ldg(p.dl + size_t(i) * n + k) : l_inf;
                            ibv[q] = tr ? __ldg(p.dib + size_t(i) * n + k) : ((i == mlast) ? ibm : ib_inf);
                        }
                } else {
#pragma unroll
                    for (int q = 0; q < G; ++q) {
                        lv[q] = l_inf;
                        ibv[q] = (g0 + q == mlast) ? ibm : ib_inf;
                    }
                }
                double y = su[0], w = su[MPT * NT], f = su[2 * MPT * NT], s2 = su[3 * MPT * NT];
                int q0 = 0;
                if (first) {   // block start: y = r, pi = 1 (rectsolver.py:86 with zero carry-in)
                    const double ib0 = ibv[0];
                    y = xv[0];
                    w = 1.0;
                    f = y * ib0;
                    s2 = ib0;
                    su[4 * MPT * NT] = (g0 == 0) ? 0.0 : -lv[0];
                    og[0] = y;
                    q0 = 1;
                }
#pragma unroll
                for (int q = 0; q < G; ++q) {
                    if (q >= q0 && q < rows) {
                        const double l = lv[q], ib = ibv[q];
                        y = __dsub_rn(xv[q], __dmul_rn(l, y));   // rectsolver.py:86
                        w = -l * w;
                        const double Wq = w * ib;
                        f = fma(y, Wq, f);
                        s2 = fma(w, Wq, s2);
                        og[size_t(q) * n] = y;
                    }
                }
                su[0] = y;
                su[MPT * NT] = w;
                su[2 * MPT * NT] = f;
                su[3 * MPT * NT] = s2;
            }
            if (last) {
                const double y = su[0], w = su[MPT * NT], f = su[2 * MPT * NT], s2 = su[3 * MPT * NT];
                const double cc = su[4 * MPT * NT];
                double *cb = pl.carry + size_t(sg.blk) * kCarryVals * n + k;
                const int e = sg.e;
                // Q = pi_e * (-l_{e+1}),  l_{e+1} = delta / beta_e
                double lnext = l_inf;
                if (k < p.kt) lnext = (e + 1 < p.m) ? __ldg(p.lt + size_t(e + 1) * 3 * p.ktp + k) : 0.0;
                else if (e + 1 < len && e + 1 < p.ecap)
                    lnext = __ldg(p.dl + size_t(e + 1) * n + k);
                else if (e + 1 < len) {
                    double ib_, bm1_;
                    factors_slow(p, k, e + 1, len, l_inf, ib_inf, 1.0 / mode_blast(p, k), 0.0, &lnext, &ib_, &bm1_);
                }
                const double Q = (e < p.m - 1) ? w * (-lnext) : 0.0;
                __stcg(cb + 0 * n, y);
                __stcg(cb + 1 * n, f);
                __stcg(cb + 2 * n, cc * w);
                __stcg(cb + 3 * n, cc * s2);
                __stcg(cb + 4 * n, Q);
            }
        }
        __syncthreads();   // regions free for the next wave
    }
    stamp(1);
    grid.sync();
    stamp(2);

    // ===================== phase 2: block carries =====================================
    carries_phase<NT>(pl, smem_raw, SMEM, tid, lane);
    stamp(3);
    grid.sync();
    stamp(4);

    // ===================== phase 3: back-substitution + inverse DST ===================
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
        const int mlast = p.m - 1;
#pragma unroll
        for (int u = 0; u < MPT; ++u) {
            const int k = tid + u * NT;
            if (k >= n) continue;
            double *su = &S(0, u);
            if (top) {
                const double *cb = pl.carry + size_t(sg.blk) * kCarryVals * n + k;
                const size_t bs = size_t(kCarryVals) * n;
                su[0] = has_next ? __ldcg(cb + bs + 6 * n) : 0.0;         // X_{b+1}
                su[MPT * NT] = __ldcg(cb + 2 * n);                        // P_e
                su[2 * MPT * NT] = has_in ? __ldcg(cb - bs + 5 * n) : 0.0; // Y_{b-1}
            }
            const double2 *rec = reinterpret_cast<const double2 *>(p.mode) + 4 * k;
            const double2 ra = __ldg(rec), rb = __ldg(rec + 1), rd = __ldg(rec + 3);
            const double ib_inf = ra.y, inl = rb.y;
            const int len = int(__double_as_longlong(rd.y));
            const double iblast = (g0 + rows - 1 >= mlast) ? 1.0 / mode_blast(p, k) : ib_inf;
            const double *yg = J.out + size_t(g0) * n + k;
            const int xsl = phys(xslot(k));
            if (k >= p.kt && g0 < len && min(g0 + rows, len + 1) > p.ecap) {
                r32_p3_slow(p, k, g0, rows, has_in, len, ib_inf, iblast, yg, reinterpret_cast<double *>(smem_raw),
                            xsl, su);
                continue;
            }
            double yv[G];
#pragma unroll
            for (int q = 0; q < G; ++q)
                if (q < rows) yv[q] = __ldcg(yg + size_t(q) * n);
            // per row: 1/beta_i and the fix-up multiplier P_{i-1} / P_i
            double ibv[G], pmv[G];
            if (k < p.kt) {
                const double *tb = p.lt + size_t(g0) * 3 * p.ktp + k;
#pragma unroll
                for (int q = 0; q < G; ++q)
                    if (q < rows) {
                        ibv[q] = __ldg(tb + size_t(q) * 3 * p.ktp + p.ktp);
                        pmv[q] = __ldg(tb + size_t(q) * 3 * p.ktp + 2 * p.ktp);   // -beta_{i-1} / delta
                    }
            } else if (g0 < len) {
                const double nio = -1.0 / off;
#pragma unroll
                for (int q = 0; q < G; ++q)
                    if (q < rows) {
                        const int i = g0 + q;
                        ibv[q] = (i < len) ? __ldg(p.dib + size_t(i) * n + k) : ((i == mlast) ? iblast : ib_inf);
                        pmv[q] = (i >= 1 && i - 1 < len) ? __ldg(p.db + size_t(i - 1) * n + k) * nio : inl;
                    }
            } else {
#pragma unroll
                for (int q = 0; q < G; ++q) {
                    ibv[q] = (g0 + q == mlast) ? iblast : ib_inf;
                    pmv[q] = inl;
                }
            }
            double x = su[0], Pc = su[MPT * NT];
            const double yin = su[2 * MPT * NT];
            double xv[G];
#pragma unroll
            for (int q = G - 1; q >= 0; --q) {
                if (q < rows) {
                    double y = yv[q];
                    if (has_in) {
                        y = fma(Pc, yin, y);
                        Pc *= pmv[q];   // P_{i-1} = P_i / (-l_i) = -P_i beta_{i-1} / delta
                    }
                    x = __dsub_rn(y, __dmul_rn(off, x)) * ibv[q];   // rectsolver.py:90
                    xv[q] = x;
                }
            }
#pragma unroll
            for (int q = 0; q < G; q += 2)
                if (q < rows) regc(q >> 1)[xsl] = make_double2(xv[q], q + 1 < rows ? xv[q + 1] : 0.0);
            su[0] = x;
            su[MPT * NT] = Pc;
        }
        __syncthreads();   // the wave's swept rows are in the regions
        const int rp = min(2, rows - 2 * wp);
        if (rp > 0) {
            xform_region(0.5 * p.scale, myreg, lane, lk);
            // epilogue out = alpha x + beta other, coalesced rows
            const double al_ = J.alpha, be_ = J.beta;
            double *oa = J.out + size_t(g0 + 2 * wp) * n;
            double *ob = oa + n;
            const double *qa = J.other ? J.other + size_t(g0 + 2 * wp) * n : nullptr;
            const double *qb = qa ? qa + n : nullptr;
#pragma unroll 8
            for (int q = lane; q < N - 1; q += 32) {
                const double2 t = myreg[phys(xslot(q))];
                if (qa) {
                    oa[q] = fma(be_, __ldg(qa + q), al_ * t.x);
                    if (rp > 1) ob[q] = fma(be_, __ldg(qb + q), al_ * t.y);
                } else {
                    oa[q] = al_ * t.x;
                    if (rp > 1) ob[q] = al_ * t.y;
                }
            }
        }
        __syncthreads();   // regions free for the next wave's sweep
    }
    stamp(5);
}

template <int CTAS>
struct Rs32K {
    static constexpr int NT = r32::NT, G = r32::G;
    static constexpr size_t SMEM = r32::SMEM;
    static const void *fn() { return (const void *)rsolve32_kernel<CTAS>; }
};

bool launch_rs32(const std::vector<SolveJob> &jobs, cudaStream_t s, Workspace &ws) {
    static const int mode = getenv("FD_RS32") ? atoi(getenv("FD_RS32")) : 1;
    if (!mode || jobs[0].p.n + 1 != r32::N || jobs[0].p.tpair != kPairDD || jobs[0].p.cyclic || jobs[0].p.nsing)
        return false;
    run_persist<Rs32K<2>>(jobs, s, ws);
    return true;
}

}  // namespace fd
