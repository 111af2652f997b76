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
    static constexpr int Q = N / 16;              // residue classes of the first pass
    static constexpr int L = Q / 2;               // lanes per row pair
    static constexpr int R3 = Q >= 64 ? Q / 32 : 1;
    static_assert(NL == 10, "K3 is instantiated for N = 1024 (c1); other lengths use rsolve.cu");
    static constexpr int NT = 512;
    static constexpr int NFW = 8, NSW = 8;        // F warps, S warps
    static constexpr int FREG = 168, SREG = 88;  // setmaxnreg split (2 warpgroups each)
    static_assert(NFW * 32 * FREG + NSW * 32 * SREG == 65536, "register file");
    static constexpr int TEAMS = NFW * 32 / L;    // row pairs in flight (one slot each)
    static constexpr int NST = NSW * 32;          // S threads
    static constexpr int U = (N - 1 + NST - 1) / NST;   // modes per S thread
    // slot layout (complex units of 16 B)
    static constexpr int ES = Q + 2;              // exchange: E(k1, c) = k1 ES + c
    __host__ __device__ static constexpr int pc(int k) { return k + (k >> 4) + 4 * (k >> 8); }   // C_k
    __host__ __device__ static constexpr int px(int q) { return q + 2 * (q >> 5); }              // X row (doubles)
    static constexpr int XB = px(N);              // row b offset (doubles)
    static constexpr int SLOTU0 = 16 * ES > pc(N - 1) + 1 ? 16 * ES : pc(N - 1) + 1;
    static constexpr int SLOTU1 = SLOTU0 > XB ? SLOTU0 : XB;
    static constexpr int SLOTU = (SLOTU1 + 1 + 7) & ~7;
    static constexpr int SP = SLOTU - 1;          // spare unit (lane 0's row-b pair 0)
    // transformed rows after the post-processing (doubles): mode position q of
    // row a / row b
    __host__ __device__ static constexpr int xa(int q) { return 2 * pc(q >> 1) + (q & 1); }
    __host__ __device__ static constexpr int xb(int q) { return (q < 2 ? 2 * SP : 2 * pc(N - (q >> 1))) + (q & 1); }
    static constexpr size_t SLOT_BYTES = size_t(SLOTU) * 16;
    static constexpr size_t OFF_AL = size_t(TEAMS) * SLOT_BYTES;
    static constexpr size_t SMEM = OFF_AL + size_t(N) * 8;
    static_assert(SMEM <= 227 * 1024, "shared memory");
};

template <int R>
__device__ __forceinline__ void regs_inc() {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(R));
}
template <int R>
__device__ __forceinline__ void regs_dec() {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(R));
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// pre-weighted complex input of index j from the row values x_j, x_{N-j}
__device__ __forceinline__ double2 prew(double al, double h, double ao, double am, double bo, double bm) {
    const double b = al - h;
    return make_double2(fma(al, ao, b * am), fma(al, bo, b * bm));
}

// Row sources of the transform: global rows (phase 1) or slot rows (phase 3)
struct GSrc {
    const double *a, *b;
    __device__ double ga(int q) const { return __ldg(a + q); }
    __device__ double gb(int q) const { return __ldg(b + q); }
};
template <class C>
struct SSrc {
    const double *a, *b;
    __device__ double ga(int q) const { return a[C::px(q)]; }
    __device__ double gb(int q) const { return b[C::px(q)]; }
};

// Forward transform of one row pair by its team: rows from src, result
// (transformed rows a, b in natural mode order, px layout) in the slot.
// t: lane within the team.  Every lane of the team must call it.
template <class C, class Src>
__device__ __forceinline__ void transform_pair(double2 *slot, const Src &src, const double *al, double h,
                                               const double2 *tw, int t) {
    constexpr int N = C::N, Q = C::Q, L = C::L;
    static_assert(L == 32 && C::R3 == 2, "one warp per pair");
    double2 v1[16], v2[16];
    // ---- class-pair loads + pre-weighting
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const int j = t + Q * r;   // lane 0: class 0 (v2 fixed below)
        const bool z = (j == 0);   // x_0 = x_N = 0
        const int po = z ? 0 : j - 1, pm = z ? 0 : N - j - 1;
        double ao = src.ga(po), am = src.ga(pm), bo = src.gb(po), bm = src.gb(pm);
        if (z) ao = am = bo = bm = 0.0;
        const double a = al[j];
        v1[r] = prew(a, h, ao, am, bo, bm);
        v2[15 - r] = prew(a, h, am, ao, bm, bo);
    }
    if (t == 0) {   // class Q/2 (self-mirrored): j = Q/2 + Q r <-> N - j = Q/2 + Q (15 - r)
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int j = Q / 2 + Q * r;
            const int po = j - 1, pm = N - j - 1;
            const double ao = src.ga(po), am = src.ga(pm), bo = src.gb(po), bm = src.gb(pm);
            const double a = al[j];
            v2[r] = prew(a, h, ao, am, bo, bm);
            v2[15 - r] = prew(a, h, am, ao, bm, bo);
        }
    }
    __syncwarp();   // phase 3: the slot's rows are consumed before the exchange overwrites them
    // ---- pass 1: radix 16 over r; B_c[k1] = s(c) W_N^{c k1} A_c[k1], s(c) = (-1)^(c>>1) for odd c
    //      (the sign rotates the odd-c0 lanes' radix-32 output by 16, see below)
    dft<16>(v1);
    dft<16>(v2);
    const int cl1 = t, cl2 = (t == 0) ? Q / 2 : Q - t;
    auto sgn = [](int c) { return ((c & 1) && ((c >> 1) & 1)) ? -1.0 : 1.0; };
    chain_twiddle<16>(v1, tw[2 * cl1], sgn(cl1));
    chain_twiddle<16>(v2, tw[2 * cl2], sgn(cl2));
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) {
        slot[k1 * C::ES + cl1] = v1[k1];
        slot[k1 * C::ES + cl2] = v2[k1];
    }
    __syncwarp();
    // ---- pass 2: lane (k1, c0) = (t >> 1, t & 1): radix 32 over c' (c = c0 + 2 c')
    const int k1 = t >> 1, c0 = t & 1;
    double2 g[32];
#pragma unroll
    for (int cp = 0; cp < 32; ++cp) g[cp] = slot[k1 * C::ES + c0 + 2 * cp];
    __syncwarp();
    dft32(g);
    // c0 = 1: the inputs carried (-1)^c', so g[i] = G_1[(i + 16) mod 32]; twiddle W_64^{k2'}
    // c0 = 0: g[i] = G_0[i], no twiddle
    static_for<0, 32>([&](auto ii) {
        constexpr int i = decltype(ii)::value, kp = (i + 16) & 31;
        constexpr double cr = cos64(kp), ci = -sin64(kp);
        const double wr = c0 ? cr : 1.0, wi = c0 ? ci : 0.0;
        g[i] = cmul(g[i], make_double2(wr, wi));
    });
    // radix 2 across the lane pair: lane c0 finishes k2' in [16 c0, 16 c0 + 16)
    //   own = g[i] (c0 = 0: G_0[i]; c0 = 1: H[16 + i]), send g[16 + i]
    //   C[k1 + 16 k2'] = G_0 + H,  C[k1 + 16 (k2' + 32)] = G_0 - H
    const double sg = c0 ? -1.0 : 1.0;
    const int kb = k1 + 256 * c0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        double2 rv;
        rv.x = __shfl_xor_sync(0xffffffffu, g[16 + i].x, 1);
        rv.y = __shfl_xor_sync(0xffffffffu, g[16 + i].y, 1);
        const double2 o0 = cadd(g[i], rv);
        const double2 d = csub(g[i], rv);
        const int k = kb + 16 * i;
        slot[C::pc(k)] = o0;
        slot[C::pc(k + 512)] = make_double2(sg * d.x, sg * d.y);
    }
    __syncwarp();
    // ---- post: lane t owns k in [16 t, 16 t + 16); it reads C_k from its "own"
    // units pc(16 t + i) and C_{N-k} from its "mirror" units pc(N - 16 t - i)
    // and writes the transformed rows back into exactly those units (row a:
    // own, row b: mirror; lane 0's missing mirror unit of k = 0 is the spare
    // unit), so no lane touches another lane's units and nothing waits.  The
    // values of k = 16 t + 16 come from lane t + 1 by shuffle.
    //   pass A: lane totals of Re/Im (C_k + C_{N-k}) -> exclusive lane scan
    //   pass B: streamed outputs (D_k, e_{k+1}) per unit
    auto mir = [&](int i) { return (t == 0 && i == 0) ? C::SP : C::pc(N - 16 * t - i); };
    double ra = 0.0, rb = 0.0;
    double2 c00, c20;   // i = 0 values (sent to lane t - 1)
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const double2 c = slot[C::pc(16 * t + i)];
        const double2 c2 = (t == 0 && i == 0) ? make_double2(0.0, 0.0) : slot[mir(i)];
        if (i == 0) {
            c00 = c;
            c20 = c2;
        }
        ra += c.x + c2.x;
        rb += c.y + c2.y;
    }
    double2 cn, c2n;   // k = 16 t + 16 (lane t + 1's i = 0)
    cn.x = __shfl_down_sync(0xffffffffu, c00.x, 1);
    cn.y = __shfl_down_sync(0xffffffffu, c00.y, 1);
    c2n.x = __shfl_down_sync(0xffffffffu, c20.x, 1);
    c2n.y = __shfl_down_sync(0xffffffffu, c20.y, 1);
    if (t == L - 1) cn = c2n = make_double2(0.0, 0.0);   // e_{N/2} = 0 (position n: not a mode)
    double ia = ra, ib = rb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double xa = __shfl_up_sync(0xffffffffu, ia, o), xb = __shfl_up_sync(0xffffffffu, ib, o);
        if (t >= o) {
            ia += xa;
            ib += xb;
        }
    }
    double sa = ia - ra, sb = ib - rb;   // exclusive prefix of the lane
    double2 c = c00, c2 = c20;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        sa += c.x + c2.x;
        sb += c.y + c2.y;
        double2 d, d2;
        if (i < 15) {
            d = slot[C::pc(16 * t + i + 1)];
            d2 = slot[mir(i + 1)];
        } else {
            d = cn;
            d2 = c2n;
        }
        slot[C::pc(16 * t + i)] = make_double2(sa, d2.y - d.y);
        slot[mir(i)] = make_double2(sb, d.x - d2.x);
        c = d;
        c2 = d2;
    }
}

// factors of the forward elimination at row i (rectsolver.py:62-77,86)
struct FwdF {
    double l, ib;
};
__device__ __forceinline__ FwdF fwd_factors(const PlanDev &p, int k, int i, int len, double l_inf, double ib_inf) {
    FwdF f;
    if (k < p.kt) {
        const double *tb = p.lt + size_t(i) * 3 * p.ktp + k;
        f.l = __ldg(tb);
        f.ib = __ldg(tb + p.ktp);
    } else if (i < len) {
        if (i < p.ecap) {
            f.l = __ldg(p.dl + size_t(i) * p.n + k);
            f.ib = __ldg(p.dib + size_t(i) * p.n + k);
        } else {
            double bm1;
            factors_slow(p, k, i, len, l_inf, ib_inf, 1.0 / mode_blast(p, k), 0.0, &f.l, &f.ib, &bm1);
        }
    } else {
        f.l = l_inf;
        f.ib = (i == p.m - 1) ? __ldg(p.last + 2 * k + 1) : ib_inf;
    }
    return f;
}
// factors of the back-substitution at row i: 1/beta_i and pm_i = -beta_{i-1}/delta
struct BwdF {
    double ib, pm;
};
__device__ __forceinline__ BwdF bwd_factors(const PlanDev &p, int k, int i, int len, double ib_inf, double inv_nl) {
    BwdF f;
    if (k < p.kt) {
        const double *tb = p.lt + size_t(i) * 3 * p.ktp + k;
        f.ib = __ldg(tb + p.ktp);
        f.pm = __ldg(tb + 2 * p.ktp);
    } else if (i < len && i < p.ecap) {
        f.ib = __ldg(p.dib + size_t(i) * p.n + k);
        f.pm = (i >= 1) ? __ldg(p.db + size_t(i - 1) * p.n + k) * p.nio : inv_nl;
    } else if (i < len || (i - 1 < len && i - 1 >= p.ecap)) {
        double l, bm1;
        factors_slow(p, k, i, len, 0.0, ib_inf, 1.0 / mode_blast(p, k), mode_binf(p, k), &l, &f.ib, &bm1);
        f.pm = bm1 * p.nio;
    } else {
        f.ib = (i == p.m - 1) ? __ldg(p.last + 2 * k + 1) : ib_inf;
        f.pm = (i >= 1 && i - 1 < len) ? __ldg(p.db + size_t(i - 1) * p.n + k) * p.nio : inv_nl;
    }
    return f;
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

    // ===================== phase 1: DST + local forward elimination ===================
    if (isF) {
        regs_inc<C::FREG>();
        int u = 0;
        for (int p = team; p < npairs; p += TEAMS, ++u) {
            const int si = seg_of(p);
            const Seg &sg = segs[si];
            const PJob &J = pl.job[sg.job];
            const int r0 = sg.s + 2 * (p - pair0[si]);
            const int rows = min(2, sg.e - r0 + 1);
            mbar_wait(&empty[team], (u & 1) ^ 1);
            const double *A = J.in + size_t(r0) * n;
            GSrc src{A, rows > 1 ? A + n : A};
            transform_pair<C>(slot_of(team), src, al, 0.5 * J.p.scale, tw, t);
            mbar_arrive(&full[team]);
        }
        regs_dec<128>();
    } else {
        regs_dec<C::SREG>();
        // Registers are tight here (SREG): per mode only the sweep state and
        // the fixed-point factors live across pairs.  Factors that need a table
        // load are prefetched one pair ahead for the first mode group (it holds
        // every slowly converging mode k < kt, which loads on every row); the
        // other groups load theirs only in their transient rows (i < len_k <=
        // ecap: the first CTAs of each rectangle).
        double ys[U], ws[U], fs[U], s2s[U];
        double l_inf[U], ib_inf[U];
        int len[U];
        int cur_job = -1;
        FwdF pf[2];   // prefetched factors of mode group 0, rows of pair p
        auto load_consts = [&](const PlanDev &pd) {
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int k = st + NST * uu;
                if (k < n) {
                    const double2 a = __ldg(reinterpret_cast<const double2 *>(pd.mode) + 4 * k);
                    l_inf[uu] = a.x;
                    ib_inf[uu] = a.y;
                    len[uu] = int(__double_as_longlong(__ldg(pd.mode + 8 * size_t(k) + 7)));
                }
            }
        };
        auto pair_rows = [&](int p, int &si, int &r0, int &rows) {
            si = seg_of(p);
            r0 = segs[si].s + 2 * (p - pair0[si]);
            rows = min(2, segs[si].e - r0 + 1);
        };
        auto fac = [&](const PlanDev &pd, int uu, int i) {
            const int k = st + NST * uu;
            return fwd_factors(pd, k, i, len[uu], l_inf[uu], ib_inf[uu]);
        };
        auto prefetch = [&](int p) {
            if (p >= npairs) return;
            int si, r0, rows;
            pair_rows(p, si, r0, rows);
            const PlanDev &pd = pl.job[segs[si].job].p;
            if (segs[si].job != cur_job) return;   // job change: loaded after the constants
            if (st < n) {
                pf[0] = fac(pd, 0, r0);
                if (rows > 1) pf[1] = fac(pd, 0, r0 + 1);
            }
        };
#pragma unroll 1
        for (int p = 0; p < npairs; ++p) {
            int si, r0, rows;
            pair_rows(p, si, r0, rows);
            const Seg sg = segs[si];
            const PJob &J = pl.job[sg.job];
            const PlanDev &pd = J.p;
            if (sg.job != cur_job) {
                cur_job = sg.job;
                load_consts(pd);
                prefetch(p);
            }
            const FwdF f0 = pf[0], f1 = pf[1];
            prefetch(p + 1);
            const int sl = p % TEAMS;
            mbar_wait(&full[sl], (p / TEAMS) & 1);
            const double *X = reinterpret_cast<const double *>(slot_of(sl));
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (r >= rows) break;
                const int i = r0 + r;
                double *og = J.out + size_t(i) * n;
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    const int k = st + NST * uu;
                    if (k >= n) continue;
                    const double xv = X[r ? C::xb(k) : C::xa(k)];
                    FwdF f;
                    if (uu == 0) f = r ? f1 : f0;
                    else if (i < len[uu] || i == pd.m - 1) f = fac(pd, uu, i);
                    else f = FwdF{l_inf[uu], ib_inf[uu]};
                    const double l = f.l, ib = f.ib;
                    if (i == sg.s) {   // block start: y = r, pi = 1
                        ys[uu] = xv;
                        ws[uu] = 1.0;
                        fs[uu] = xv * ib;
                        s2s[uu] = ib;
                    } else {
                        const double y = __dsub_rn(xv, __dmul_rn(l, ys[uu]));
                        const double w = -l * ws[uu];
                        const double W = w * ib;
                        fs[uu] = fma(y, W, fs[uu]);
                        s2s[uu] = fma(w, W, s2s[uu]);
                        ys[uu] = y;
                        ws[uu] = w;
                    }
                    og[k] = ys[uu];
                    if (i == sg.e) {   // block end: scalars for the carries
                        double *cb = pl.carry + size_t(sg.blk) * kCarryVals * n + k;
                        const double lnext = (i + 1 < pd.m) ? fac(pd, uu, i + 1).l : 0.0;
                        const double cc = (sg.s == 0) ? 0.0 : -fac(pd, uu, sg.s).l;   // -l at the block start
                        const double w = ws[uu];
                        const double Qv = (i < pd.m - 1) ? w * (-lnext) : 0.0;
                        __stcg(cb + 0 * n, ys[uu]);
                        __stcg(cb + 1 * n, fs[uu]);
                        __stcg(cb + 2 * n, cc * w);
                        __stcg(cb + 3 * n, cc * s2s[uu]);
                        __stcg(cb + 4 * n, Qv);
                    }
                }
            }
            mbar_arrive(&empty[sl]);
        }
        regs_inc<128>();
    }
    grid.sync();
    // ===================== phase 2: block carries =====================================
    carries_phase<C::NT>(pl, smem_raw, C::OFF_AL, tid, lane);
    grid.sync();
    // re-arm the slot barriers with the phase-3 roles (S fills, F drains)
    if (tid == 0) {
        for (int q = 0; q < TEAMS; ++q) {
            mbar_init(&full[q], NST);
            mbar_init(&empty[q], L);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // ===================== phase 3: back-substitution + inverse DST ===================
    // pairs of a segment from its last row down: (e, e-1), (e-2, e-3), ...
    if (!isF) {
        regs_dec<C::SREG>();
        double xs[U], pcs[U], yins[U];
        double ib_inf[U], inv_nl[U];
        int len[U];
        int cur_job = -1;
        BwdF pf[2];      // prefetched factors of mode group 0 (see phase 1)
        double py[2][U]; // prefetched yhat rows of the next pair
        auto pair_rows = [&](int p, int &si, int &rh, int &rows) {
            si = seg_of(p);
            rh = segs[si].e - 2 * (p - pair0[si]);
            rows = min(2, rh - segs[si].s + 1);
        };
        auto fac = [&](const PlanDev &pd, int uu, int i) {
            const int k = st + NST * uu;
            return bwd_factors(pd, k, i, len[uu], ib_inf[uu], inv_nl[uu]);
        };
        auto prefetch = [&](int p) {
            if (p >= npairs) return;
            int si, rh, rows;
            pair_rows(p, si, rh, rows);
            const PJob &J = pl.job[segs[si].job];
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    const int k = st + NST * uu;
                    if (k < n && r < rows) py[r][uu] = __ldcg(J.out + size_t(rh - r) * n + k);
                }
            if (segs[si].job != cur_job) return;
            if (st < n) {
                pf[0] = fac(J.p, 0, rh);
                if (rows > 1) pf[1] = fac(J.p, 0, rh - 1);
            }
        };
        prefetch(0);
#pragma unroll 1
        for (int p = 0; p < npairs; ++p) {
            int si, rh, rows;
            pair_rows(p, si, rh, rows);
            const Seg sg = segs[si];
            const PJob &J = pl.job[sg.job];
            const PlanDev &pd = J.p;
            if (sg.job != cur_job) {
                cur_job = sg.job;
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    const int k = st + NST * uu;
                    if (k < n) {
                        const double2 a = __ldg(reinterpret_cast<const double2 *>(pd.mode) + 4 * k);
                        const double2 b = __ldg(reinterpret_cast<const double2 *>(pd.mode) + 4 * k + 1);
                        ib_inf[uu] = a.y;
                        inv_nl[uu] = b.y;
                        len[uu] = int(__double_as_longlong(__ldg(pd.mode + 8 * size_t(k) + 7)));
                    }
                }
                if (st < n) {
                    pf[0] = fac(pd, 0, rh);
                    if (rows > 1) pf[1] = fac(pd, 0, rh - 1);
                }
            }
            const bool has_in = sg.blk > J.blk_base;                 // block does not start at row 0
            const bool has_next = sg.blk < J.blk_base + J.nblk - 1;  // a block below carries X
            if (p == pair0[si]) {   // top of the block: carries from phase 2
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    const int k = st + NST * uu;
                    if (k >= n) continue;
                    const double *cb = pl.carry + size_t(sg.blk) * kCarryVals * n + k;
                    const size_t bs = size_t(kCarryVals) * n;
                    xs[uu] = has_next ? __ldcg(cb + bs + 6 * n) : 0.0;
                    yins[uu] = has_in ? __ldcg(cb - bs + 5 * n) : 0.0;
                    pcs[uu] = __ldcg(cb + 2 * n);
                }
            }
            double yv[2][U];
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int uu = 0; uu < U; ++uu) yv[r][uu] = py[r][uu];
            const BwdF f0 = pf[0], f1 = pf[1];
            prefetch(p + 1);
            const int sl = p % TEAMS;
            mbar_wait(&empty[sl], ((p / TEAMS) & 1) ^ 1);
            double *X = reinterpret_cast<double *>(slot_of(sl));
            const double off = pd.off;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (r >= rows) break;
                const int i = rh - r;
                double *Xr = X + r * C::XB;
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    const int k = st + NST * uu;
                    if (k >= n) continue;
                    BwdF f;
                    if (uu == 0) f = r ? f1 : f0;
                    else if (i <= len[uu] || i == pd.m - 1) f = fac(pd, uu, i);
                    else f = BwdF{ib_inf[uu], inv_nl[uu]};
                    double y = yv[r][uu];
                    if (has_in) {
                        y = fma(pcs[uu], yins[uu], y);
                        pcs[uu] *= f.pm;   // P_{i-1} = P_i / (-l_i)
                    }
                    const double x = __dsub_rn(y, __dmul_rn(off, xs[uu])) * f.ib;   // rectsolver.py:90
                    xs[uu] = x;
                    Xr[C::px(k)] = x;
                }
            }
            mbar_arrive(&full[sl]);
        }
        regs_inc<128>();
    } else {
        regs_inc<C::FREG>();
        int u = 0;
        for (int p = team; p < npairs; p += TEAMS, ++u) {
            const int si = seg_of(p);
            const Seg &sg = segs[si];
            const PJob &J = pl.job[sg.job];
            const int rh = sg.e - 2 * (p - pair0[si]);
            const int rows = min(2, rh - sg.s + 1);
            mbar_wait(&full[team], u & 1);
            double2 *slot = slot_of(team);
            const double *X = reinterpret_cast<const double *>(slot);
            SSrc<C> src{X, rows > 1 ? X + C::XB : X};
            transform_pair<C>(slot, src, al, 0.5 * J.p.scale, tw, t);
            __syncwarp();
            // epilogue out = alpha x + beta other, coalesced rows
            const double a_ = J.alpha, b_ = J.beta;
            for (int h = 0; h < rows; ++h) {
                double *oh = J.out + size_t(rh - h) * n;
                const double *qh = J.other ? J.other + size_t(rh - h) * n : nullptr;
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
        regs_dec<128>();
    }
}

template <int NL>
struct K3K {
    static constexpr int NT = Cfg<NL>::NT, G = 2;
    static constexpr size_t SMEM = Cfg<NL>::SMEM;
    static const void *fn() { return (const void *)k3_kernel<NL>; }
};

}  // namespace k3

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
