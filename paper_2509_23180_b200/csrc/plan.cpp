// Plan construction (host): eigenvalues, compressed per-mode LU factors of the
// sweep systems, block-carry tables, transform tables.  Compiled with
// -ffp-contract=off so every recurrence rounds exactly like the reference's
// numpy expressions.
//
// Reference: transforms.eigenvalues DD (transforms.py:26-31,38),
// rectsolver._factor_tridiag (rectsolver.py:62-77), plan_rect diag/end
// modifiers and pivot tolerance (rectsolver.py:122-135,153-163).
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>

#include "fd_internal.h"

namespace fd {

namespace {

struct ModeFactors {
    std::vector<double> l, b;  // rows 0..len-1 explicit
    int fix;                   // first row of the fixed point (-1 if none)
    double l_inf, b_inf;       // converged values (valid when fix >= 0)
    double b_last;             // beta_{m-1}
    bool bad;
};

// eigenvalue of mode k (0-based), exactly as numpy evaluates transforms.py:29,38
double eig_dd(int k, int n, double dt, double dor, double kappa) {
    const double j = double(k + 1);
    const double arg = j * M_PI / double(n + 1);
    double lam = -2.0 * (dt + dor) + (2.0 * dt) * cos(arg);
    return lam + kappa;
}
// PP: cos(2 pi (j - 1) / n), j = 1..n   (transforms.py:34-35)
double eig_pp(int k, int n, double dt, double dor, double kappa) {
    const double arg = 2.0 * M_PI * double(k) / double(n);
    double lam = -2.0 * (dt + dor) + (2.0 * dt) * cos(arg);
    return lam + kappa;
}
// NN: cos((j - 1) pi / n), j = 1..n   (transforms.py:32-33)
double eig_nn(int k, int n, double dt, double dor, double kappa) {
    const double jm1 = double(k);
    const double arg = jm1 * M_PI / double(n);
    double lam = -2.0 * (dt + dor) + (2.0 * dt) * cos(arg);
    return lam + kappa;
}

// Run the reference recurrence for one mode until the bitwise fixed point.
ModeFactors factor_mode(int m, double lam, double mod_w, double mod_e, double off, double tol,
                        int R) {
    ModeFactors f;
    f.bad = false;
    f.fix = -1;
    auto diag = [&](int i) {
        double d = lam;
        if (i == 0) d = d + mod_w;
        if (i == m - 1) d = d + mod_e;
        return d;
    };
    double b0 = diag(0);
    bool bad = fabs(b0) < tol;
    double safe = bad ? 1.0 : b0;
    f.l.push_back(0.0);
    f.b.push_back(b0);
    // regular rows 1..m-2 (no end modifier): stop at the fixed point
    int i = 1;
    for (; i < m; ++i) {
        const double l = off / safe;
        double b = diag(i) - off * l;
        bad = bad || fabs(b) < tol;
        safe = bad ? 1.0 : b;
        b = safe;
        f.l.push_back(l);
        f.b.push_back(b);
        if (i >= 1 && i <= m - 2 && b == f.b[i - 1] && f.fix < 0) {
            f.fix = i;
            break;
        }
    }
    f.bad = bad;
    if (f.fix >= 0) {
        f.l_inf = f.l[f.fix];
        f.b_inf = f.b[f.fix];
        // explicit region: block aligned, >= fix
        const int len = std::min(m, ((f.fix + R - 1) / R) * R);
        while ((int)f.l.size() < len) {
            f.l.push_back(f.l_inf);
            f.b.push_back(f.b_inf);
        }
        f.l.resize(len);
        f.b.resize(len);
        // last row carries the east modifier (rectsolver.py:133)
        const double l = off / f.b_inf;
        double b = diag(m - 1) - off * l;
        f.bad = f.bad || fabs(b) < tol;
        f.b_last = b;
        if (len == m) f.b[m - 1] = b;
    } else {
        f.l_inf = f.l.back();
        f.b_inf = f.b.back();
        f.b_last = f.b[m - 1];
    }
    return f;
}

std::mutex g_tab_mu;
std::map<std::pair<int, int>, void *> g_tw, g_dense;

}  // namespace

// block-relative products for rows [s, e] of one mode given l(i), b(i)
template <class GetL, class GetB>
static void block_scalars(int s, int e, int m, double off, GetL gl, GetB gb, double *Pe, double *xi,
                          double *Q, double *Pcol /* per row P, may be null */) {
    // P_i = prod_{t=s}^{i} (-l_t) (block 0: unused, 0); pi_i = prod_{t=s+1}^{i} (-l_t)
    double P = (s == 0) ? 0.0 : -gl(s);
    double pi = 1.0, xs = 0.0;
    for (int i = s; i <= e; ++i) {
        if (i > s) {
            const double nl = -gl(i);
            P = P * nl;
            pi = pi * nl;
        }
        if (Pcol) Pcol[i - s] = P;
        xs = xs + P * (pi / gb(i));
    }
    *Pe = P;
    *xi = xs;
    // Q = prod_{t=s}^{e} (-off / beta_t)
    double q = 1.0;
    for (int i = s; i <= e; ++i) q = q * (-off / gb(i));
    *Q = q;
    (void)m;
}

struct HostTables {
    std::vector<int> off, len;
    std::vector<double> ex;    // 4 per explicit row
    std::vector<double> cv;    // 4 per mode
    std::vector<double> last;  // 2 per mode
    std::vector<double> blk;   // nb * 3 * n
    std::vector<int> bad_modes;
    std::vector<double> lam;   // eigenvalues lambda_k (+ kappa)
    std::vector<int> fix;      // first row of the bitwise fixed point (m if none)
    std::vector<double> lt;    // [lt_rows][3][ktp] l_i, 1/beta_i, -beta_{i-1}/delta for modes < kt
    std::vector<double> lta;   // [m][3][ktpa] the same for the first kta = min(kt, kLtNarrow) modes
    int kta = 0, ktpa = 0, lt_rows = 0, lt_need = 0;
    std::vector<std::vector<double>> fl, fb;   // per mode: explicit l_i, beta_i (i < len)
    int kt = 0, ktp = 0;
    long long explicit_rows = 0;
    // periodic sweep axis: Sherman-Morrison correction (rectsolver.py:136-153)
    double soff = 0.0;         // sweep coupling used by the factors (2 delta when m == 2)
    std::vector<double> smq;   // [m][n] q_k
    std::vector<double> cyc;   // [n][2] delta/gamma_k, denom_k
};

// parallel loop over [0, n) in contiguous chunks on the host's cores
template <class F>
static void parallel_for(int n, F fn) {
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    const int nt = std::min(std::min(hw, 32), std::max(1, n / 64));
    if (nt <= 1) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) {
        const int lo = int((long long)n * t / nt), hi = int((long long)n * (t + 1) / nt);
        th.emplace_back([=] { fn(lo, hi); });
    }
    for (auto &x : th) x.join();
}

static HostTables build_tables(int m, int n, double dx, double dy, double kappa, double mod_w,
                               double mod_e, int R, bool carry_tables, int pair = kPairDD,
                               bool cyclic = false) {
    const double delta_x = 1.0 / (dx * dx), delta_y = 1.0 / (dy * dy);
    // periodic sweep with two rows: the wrap doubles the coupling (rectsolver.py:152-153)
    const double off = (cyclic && m == 2) ? 2.0 * delta_x : delta_x;
    std::vector<double> lam(n);
    double amax = 0.0;
    for (int k = 0; k < n; ++k) {
        lam[k] = pair == kPairNN ? eig_nn(k, n, delta_y, delta_x, kappa)
                 : pair == kPairPP ? eig_pp(k, n, delta_y, delta_x, kappa) : eig_dd(k, n, delta_y, delta_x, kappa);
        amax = std::max(amax, fabs(lam[k]));
    }
    const double tol = 1e-13 * std::max(amax, off);   // rectsolver.py:135
    const int nb = (m + R - 1) / R;
    HostTables T;
    T.lam = lam;
    T.soff = off;
    // per-mode end modifiers: the sweep-axis ends, or (periodic sweep, m > 2) the
    // rank-one split of the wrap-around entries, gamma_k = -diag_0 unless that is
    // below the pivot tolerance (rectsolver.py:139-144)
    const bool sm = cyclic && m > 2;
    std::vector<double> mwk(n, cyclic ? 0.0 : mod_w), mek(n, cyclic ? 0.0 : mod_e), gam(sm ? n : 0);
    if (sm)
        for (int k = 0; k < n; ++k) {
            gam[k] = fabs(lam[k]) > tol ? -lam[k] : delta_x;
            mwk[k] = -gam[k];
            mek[k] = -(delta_x * delta_x / gam[k]);
        }
    T.off.resize(n);
    T.len.resize(n);
    T.cv.resize(4 * size_t(n));
    T.last.resize(2 * size_t(n));
    T.fix.resize(n);
    // per mode (independent, on all host cores): factors until the fixed point,
    // block scalars of the explicit blocks, of a converged block and of the last
    std::vector<ModeFactors> mf(n);
    struct BlkS {
        std::vector<double> tr;   // [nbt][3] explicit blocks
        double conv[3], last[3];
        int nbt;
        bool has_conv;
    };
    std::vector<BlkS> bs(n);
    parallel_for(n, [&](int k0, int k1) {
        for (int k = k0; k < k1; ++k) {
            mf[k] = factor_mode(m, lam[k], mwk[k], mek[k], off, tol, R);
            if (!carry_tables) continue;
            const ModeFactors &f = mf[k];
            const int len = (int)f.l.size();
            auto gl = [&](int i) { return i < len ? f.l[i] : f.l_inf; };
            auto gb = [&](int i) { return i == m - 1 ? f.b_last : (i < len ? f.b[i] : f.b_inf); };
            BlkS &q = bs[k];
            q.nbt = std::min(nb, (len + R - 1) / R);
            q.tr.resize(3 * size_t(q.nbt));
            for (int b = 0; b < q.nbt; ++b) {
                const int s = b * R, e = std::min(m, s + R) - 1;
                block_scalars(s, e, m, off, gl, gb, &q.tr[3 * b], &q.tr[3 * b + 1], &q.tr[3 * b + 2], nullptr);
            }
            q.has_conv = false;
            for (int b = q.nbt; b < nb - 1; ++b) {   // first converged (non-last) block: all equal
                const int s = b * R, e = std::min(m, s + R) - 1;
                block_scalars(s, e, m, off, gl, gb, &q.conv[0], &q.conv[1], &q.conv[2], nullptr);
                q.has_conv = true;
                break;
            }
            if (q.nbt < nb) {
                const int s = (nb - 1) * R, e = m - 1;
                block_scalars(s, e, m, off, gl, gb, &q.last[0], &q.last[1], &q.last[2], nullptr);
            }
        }
    });
    if (sm) {   // q_k = A_k^-1 u, u = (gamma_k, 0, ..., 0, delta)   (rectsolver.py:145-150)
        T.smq.assign(size_t(m) * n, 0.0);
        T.cyc.assign(2 * size_t(n), 0.0);
        parallel_for(n, [&](int k0, int k1) {
            std::vector<double> y(m);
            for (int k = k0; k < k1; ++k) {
                ModeFactors &f = mf[k];
                const int len = (int)f.l.size();
                auto gl = [&](int i) { return i < len ? f.l[i] : f.l_inf; };
                auto gb = [&](int i) { return i == m - 1 ? f.b_last : (i < len ? f.b[i] : f.b_inf); };
                y[0] = gam[k];
                for (int i = 1; i < m; ++i) y[i] = (i == m - 1 ? delta_x : 0.0) - gl(i) * y[i - 1];
                double x = y[m - 1] / gb(m - 1);
                T.smq[size_t(m - 1) * n + k] = x;
                for (int i = m - 2; i >= 0; --i) {
                    x = (y[i] - delta_x * x) / gb(i);
                    T.smq[size_t(i) * n + k] = x;
                }
                const double r = delta_x / gam[k];
                const double den = 1.0 + T.smq[k] + r * T.smq[size_t(m - 1) * n + k];
                T.cyc[2 * k] = r;
                T.cyc[2 * k + 1] = den;
                if (fabs(den) < 1e-12) f.bad = true;   // rectsolver.py:151
            }
        });
    }
    size_t total = 0;
    for (int k = 0; k < n; ++k) {
        const ModeFactors &f = mf[k];
        if (f.bad) T.bad_modes.push_back(k);
        T.fix[k] = f.fix >= 0 ? f.fix : m;
        T.off[k] = (int)total;
        T.len[k] = (int)f.l.size();
        total += f.l.size();
    }
    T.explicit_rows = (long long)total;
    T.ex.resize(4 * (carry_tables ? total : 0));
    parallel_for(n, [&](int k0, int k1) {
        std::vector<double> Pcol(R);
        for (int k = k0; k < k1; ++k) {
            const ModeFactors &f = mf[k];
            const int len = T.len[k];
            auto gl = [&](int i) { return i < len ? f.l[i] : f.l_inf; };
            auto gb = [&](int i) { return i == m - 1 ? f.b_last : (i < len ? f.b[i] : f.b_inf); };
            T.cv[4 * k + 0] = f.l_inf;
            T.cv[4 * k + 1] = 1.0 / f.b_inf;
            T.cv[4 * k + 2] = f.b_inf;
            T.cv[4 * k + 3] = 1.0 / (-f.l_inf);
            T.last[2 * k + 0] = f.b_last;
            T.last[2 * k + 1] = 1.0 / f.b_last;
            if (!carry_tables) continue;
            const size_t base = 4 * size_t(T.off[k]);
            for (int b = 0; b * R < len; ++b) {   // explicit rows with their block-relative P
                const int s = b * R, e = std::min(m, s + R) - 1;
                double Pe, xi, Q;
                block_scalars(s, e, m, off, gl, gb, &Pe, &xi, &Q, Pcol.data());
                for (int i = s; i <= e && i < len; ++i) {
                    double *r = &T.ex[base + 4 * size_t(i)];
                    r[0] = f.l[i];
                    r[1] = 1.0 / gb(i);
                    r[2] = gb(i);
                    r[3] = Pcol[i - s];
                }
            }
        }
    });
    // per-mode factor rows kept for the row-major device tables
    T.fl.resize(n);
    T.fb.resize(n);
    for (int k = 0; k < n; ++k) {
        T.fl[k] = std::move(mf[k].l);
        T.fb[k] = std::move(mf[k].b);
    }
    if (!carry_tables) return T;
    // block table [nb][3][n], rows written contiguously
    T.blk.resize(size_t(nb) * 3 * n);
    parallel_for(nb, [&](int b0, int b1) {
        for (int b = b0; b < b1; ++b)
            for (int c = 0; c < 3; ++c) {
                double *row = &T.blk[(size_t(b) * 3 + c) * n];
                for (int k = 0; k < n; ++k) {
                    const BlkS &q = bs[k];
                    row[k] = b < q.nbt ? q.tr[3 * b + c] : (b == nb - 1 || !q.has_conv) ? q.last[c] : q.conv[c];
                }
            }
    });
    return T;
}

// Row-major factor tables of the slowly converging lowest modes (persistent
// kernel): modes k < kt whose fixed point is >= kLongTransient rows away.  Two
// tables: the wide one [lt_rows][3][ktp] holds all kt modes down to the row
// where every mode >= kLtNarrow has reached its fixed point (+ one row group
// of the kernel); below it only the first kLtNarrow modes (one warp of the sweeps) are
// still in their transient, and the narrow table [m][3][ktpa] holds just those.
constexpr int kLongTransient = 48;
#ifndef FD_ECAP
#define FD_ECAP 128   // rows of every mode kept in the row-major transient tables
#endif
static void build_long_table(HostTables &T, int m, int n, double off, int kt_cap, int group_rows) {
    int kt = 0;
    for (int k = 0; k < n; ++k)
        if (T.fix[k] >= kLongTransient) kt = k + 1;
    kt = std::min(kt, kt_cap);
    T.kt = kt;
    T.ktp = (kt + 1) & ~1;
    T.kta = std::min(kt, kLtNarrow);
    T.ktpa = (T.kta + 1) & ~1;
    T.lt_need = 0;
    for (int k = kLtNarrow; k < kt; ++k) T.lt_need = std::max(T.lt_need, std::min(T.fix[k], m));
    // a group that starts before lt_need reads all its rows from the wide table
    T.lt_rows = kt > kLtNarrow ? std::min(m, T.lt_need + group_rows) : 0;
    if (kt == 0) return;
    auto fill = [&](std::vector<double> &tab, int rows, int cnt, int pitch) {
        tab.assign(size_t(rows) * 3 * pitch, 0.0);
        parallel_for(rows, [&](int i0, int i1) {
            for (int i = i0; i < i1; ++i) {
                double *r = &tab[size_t(i) * 3 * pitch];
                for (int k = 0; k < cnt; ++k) {
                    const int len = T.len[k];
                    auto gl = [&](int q) { return q < len ? T.fl[k][q] : T.cv[4 * k + 0]; };
                    auto gb = [&](int q) {
                        return q == m - 1 ? T.last[2 * k] : (q < len ? T.fb[k][q] : T.cv[4 * k + 2]);
                    };
                    r[k] = (i == 0) ? 0.0 : gl(i);
                    r[pitch + k] = 1.0 / gb(i);
                    r[2 * pitch + k] = (i == 0) ? 0.0 : -gb(i - 1) / off;
                }
            }
        });
    };
    fill(T.lta, m, T.kta, T.ktpa);
    if (T.lt_rows > 0) fill(T.lt, T.lt_rows, kt, T.ktp);
}

// ---------------------------------------------------------------------------
// transform tables, shared per (device, n)
const double2 *twiddles_for(int device, int n) {
    if (transform_kind(n) != kFFT) return nullptr;
    std::lock_guard<std::mutex> g(g_tab_mu);
    auto key = std::make_pair(device, n);
    auto it = g_tw.find(key);
    if (it != g_tw.end()) return (const double2 *)it->second;
    const int L = 2 * (n + 1), N = n + 1;
    const long double PI = 3.141592653589793238462643383279502884L;
    // [L] twiddles, then [N] real-DST pre-weights (PlanDev::ralpha)
    std::vector<double2> h(L + (N + 1) / 2);
    for (int t = 0; t < L; ++t) {
        long double a = 2.0L * PI * (long double)t / (long double)L;
        h[t].x = (double)cosl(a);
        h[t].y = (double)(-sinl(a));
    }
    double *al = reinterpret_cast<double *>(h.data() + L);
    const long double sc = sqrtl(2.0L / (long double)N);
    for (int j = 0; j < N; ++j) al[j] = (double)(0.5L * sc * sinl(PI * (long double)j / (long double)N) + 0.25L * sc);
    void *d = nullptr;
    FD_CUDA(cudaMalloc(&d, sizeof(double2) * h.size()));
    FD_CUDA(cudaMemcpy(d, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice));
    g_tw[key] = d;
    return (const double2 *)d;
}

const double *dense_table_for(int device, int n, int pair, bool force) {
    if (transform_kind(n, pair) != kDense && !(force && n <= kDenseMax)) return nullptr;
    std::lock_guard<std::mutex> g(g_tab_mu);
    auto key = std::make_pair(device, n + (pair << 24));
    auto it = g_dense.find(key);
    if (it != g_dense.end()) return (const double *)it->second;
    const long double PI_L = 3.141592653589793238462643383279502884L;
    std::vector<double> h;
    if (pair == kPairPP) {
        // cos(2 pi q / n), q < n, then sin(2 pi q / n), q < n: the real Fourier basis at q = o i mod n
        h.resize(2 * size_t(n));
        for (long long q = 0; q < n; ++q) {
            h[q] = (double)cosl(2.0L * PI_L * (long double)q / (long double)n);
            h[n + q] = (double)sinl(2.0L * PI_L * (long double)q / (long double)n);
        }
    } else if (pair == kPairNN) {
        // cos(pi q / 2n), q < 4n: the dense DCT-II/III read their basis at q = o(2i+1) / i(2o+1) mod 4n
        h.resize(4 * size_t(n));
        for (long long q = 0; q < 4LL * n; ++q) h[q] = (double)cosl(PI_L * (long double)q / (2.0L * (long double)n));
    } else {
        // sin(pi q / (n+1)), q < 2(n+1): the dense DST-I reads S[j][k] at q = (j+1)(k+1) mod 2(n+1)
        const long long P2 = 2LL * (n + 1);
        h.resize(P2);
        for (long long q = 0; q < P2; ++q) h[q] = (double)sinl(PI_L * (long double)q / (long double)(n + 1));
    }
    void *d = nullptr;
    FD_CUDA(cudaMalloc(&d, sizeof(double) * h.size()));
    FD_CUDA(cudaMemcpy(d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
    g_dense[key] = d;
    return (const double *)d;
}

template <class T>
static T *upload(Plan *p, const std::vector<T> &h) {
    size_t bytes = std::max<size_t>(sizeof(T), sizeof(T) * h.size());
    void *d = dmalloc(bytes);
    p->allocs.push_back(d);
    if (!h.empty()) FD_CUDA(cudaMemcpy(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
    return (T *)d;
}

static Plan *build_proto(int m, int n, double dx, double dy, double kappa, double mod_w, double mod_e,
                         int device, int pair, int flags) {
    if (m < 1 || n < 1) FD_FAIL(FD_ERR_VALIDATION, "plan: empty grid");
    if (!(dx > 0) || !(dy > 0)) FD_FAIL(FD_ERR_VALIDATION, "plan: nonpositive spacing");
    const bool cyclic = flags & kPlanCyclic, pin = flags & kPlanPinMean;
    if (cyclic && (m % 2)) FD_FAIL(FD_ERR_VALIDATION, "plan: periodic sweep axis needs an even count");
    int tk = transform_kind(n, pair);
    // the correction and pseudo-inverse terms live in the three-kernel dense solve
    const bool forced = tk == kFFT && (cyclic || pin);
    if (forced) tk = n <= kDenseMax ? kDense : kSep;   // dense transform limit (dst_device.cuh kDenseMax)
    if (tk < 0) {
        std::ostringstream os;
        os << "plan: no GPU transform for n = " << n << (pair == kPairPP && (n & 1) ? " (periodic axes need an even length)" : "");
        FD_FAIL(FD_ERR_UNSUPPORTED, os.str());
    }
    const int R = forced ? 8 : rows_per_block(n, pair);   // forced: the dense path's rows per group
    HostTables T = build_tables(m, n, dx, dy, kappa, mod_w, mod_e, R, tk != kFFT, pair, cyclic);
    if (!T.bad_modes.empty() && !pin) {
        std::ostringstream os;
        os << "operator singular in spectral modes (";
        for (size_t i = 0; i < T.bad_modes.size() && i < 16; ++i) os << (i ? ", " : "") << T.bad_modes[i];
        os << ")";
        FD_FAIL(FD_ERR_SINGULAR, os.str());
    }
    FD_CUDA(cudaSetDevice(device));
    Plan *p = new Plan();
    try {
        p->device = device;
        p->m = m;
        p->n = n;
        p->dx = dx;
        p->dy = dy;
        p->kappa = kappa;
        p->mod_w = mod_w;
        p->mod_e = mod_e;
        p->delta_x = 1.0 / (dx * dx);
        p->delta_y = 1.0 / (dy * dy);
        p->transform = tk;
        p->explicit_rows = T.explicit_rows;
        PlanDev &d = p->dev;
        d.m = m;
        d.n = n;
        d.R = R;
        d.nb = (m + R - 1) / R;
        d.off = T.soff;
        d.nio = -1.0 / d.off;
        d.mod_w = mod_w;
        d.mod_e = mod_e;
        d.tpair = pair;
        d.tkind = tk;
        d.scale = (pair == kPairNN || pair == kPairPP) ? sqrt(2.0 / n) : sqrt(2.0 / (n + 1));
        d.ex_off = upload(p, T.off);
        d.ex_len = upload(p, T.len);
        d.ex = upload(p, T.ex);
        d.cv = upload(p, T.cv);
        d.last = upload(p, T.last);
        std::vector<double> rec(8 * size_t(n));
        for (int k = 0; k < n; ++k) {
            double *r = &rec[8 * size_t(k)];
            for (int c = 0; c < 4; ++c) r[c] = T.cv[4 * k + c];
            r[4] = T.last[2 * k];
            r[5] = T.lam[k];
            long long o = T.off[k], l = T.fix[k];   // exact fixed-point row (persistent kernel)
            memcpy(&r[6], &o, 8);
            memcpy(&r[7], &l, 8);
        }
        d.mode = upload(p, rec);
        // row-major copies of the first ecap rows (the transient region of most modes)
        d.ecap = std::min(m, FD_ECAP);
        std::vector<double> dl(size_t(d.ecap) * n), dib(size_t(d.ecap) * n), db(size_t(d.ecap) * n);
        parallel_for(d.ecap, [&](int i0, int i1) {
            for (int i = i0; i < i1; ++i)
                for (int k = 0; k < n; ++k) {
                    const bool ex = i < T.len[k];
                    const double b = (i == m - 1) ? T.last[2 * k] : (ex ? T.fb[k][i] : T.cv[4 * k + 2]);
                    dl[size_t(i) * n + k] = ex ? T.fl[k][i] : T.cv[4 * k + 0];
                    db[size_t(i) * n + k] = b;
                    dib[size_t(i) * n + k] = (i == m - 1) ? T.last[2 * k + 1] : (ex ? 1.0 / b : T.cv[4 * k + 1]);
                }
        });
        d.dl = upload(p, dl);
        d.dib = upload(p, dib);
        d.db = upload(p, db);
        if (tk == kFFT) {
            build_long_table(T, m, n, d.off, rs_kt_cap(n + 1), rs_rows_per_group(n + 1));
        }
        d.kt = T.kt;
        d.ktp = T.ktp;
        d.kta = T.kta;
        d.ktpa = T.ktpa;
        d.lt_rows = T.lt_rows;
        d.lt_need = T.lt_need;
        {   // transient profile of the table-free modes (row partition cost model)
            int tl = 0;
            for (int k = T.kt; k < n; ++k) tl = std::max(tl, T.len[k]);
            tl = std::min(tl, 512);
            std::vector<int> cnt(tl + 1, 0);
            for (int k = T.kt; k < n; ++k) cnt[std::min(T.len[k], tl)]++;
            p->tprof.assign(tl, 0.0f);
            int alive = n - T.kt;   // modes with len > i
            for (int i = 0; i < tl; ++i) {
                alive -= cnt[i];
                p->tprof[i] = float(alive) / float(n);
            }
        }
        d.lta = T.kt ? upload(p, T.lta) : nullptr;
        d.lt = T.lt_rows ? upload(p, T.lt) : d.lta;
        d.blk = T.blk.empty() ? nullptr : upload(p, T.blk);
        d.ye = d.fs = nullptr;   // per-plan scratch (plan_create)
        d.tw = tk == kFFT ? twiddles_for(device, n) : nullptr;
        d.ralpha = d.tw ? reinterpret_cast<const double *>(d.tw + 2 * (n + 1)) : nullptr;
        d.dense = tk == kDense ? dense_table_for(device, n, pair, forced) : nullptr;
        p->flags = flags;
        d.cyclic = !T.smq.empty();
        d.smq = d.cyclic ? upload(p, T.smq) : nullptr;
        d.cyc = d.cyclic ? upload(p, T.cyc) : nullptr;
        p->sing_modes = T.bad_modes;
        d.nsing = (int)T.bad_modes.size();
        if (d.nsing) {
            std::vector<int> sidx(n, -1);
            for (int i = 0; i < d.nsing; ++i) sidx[T.bad_modes[i]] = i;
            d.sidx = upload(p, sidx);
        }
    } catch (...) {
        cudaDeviceSynchronize();
        for (void *a : p->allocs) dfree(a);
        delete p;
        throw;
    }
    return p;
}

static void free_tables(Plan *p) {
    if (!p) return;
    cudaSetDevice(p->device);
    cudaDeviceSynchronize();
    for (void *a : p->allocs) dfree(a);
    delete p;
}

// Plans are immutable once built, so identical (device, grid, spacing, kappa,
// end modifiers) requests share one set of device tables: the centre and the
// four arms of the BASELINE crosses need one table build instead of five, and
// repeated solves on the same geometry reuse the last few builds (LRU).
namespace {
struct PlanKey {
    int device, m, n, pair, flags;
    double v[5];
    bool operator==(const PlanKey &o) const {
        return device == o.device && m == o.m && n == o.n && pair == o.pair && flags == o.flags &&
               memcmp(v, o.v, sizeof(v)) == 0;
    }
};
constexpr size_t kPlanCache = 8;
std::mutex g_plan_mu;
auto *g_plan_lru = new std::list<std::pair<PlanKey, std::shared_ptr<Plan>>>();   // never destroyed
}  // namespace

Plan *plan_create(int m, int n, double dx, double dy, double kappa, double mod_w, double mod_e,
                  int device, int pair, int flags) {
    PlanKey key{device, m, n, pair, flags, {dx, dy, kappa, mod_w, mod_e}};
    std::shared_ptr<Plan> proto;
    {
        std::lock_guard<std::mutex> g(g_plan_mu);
        for (auto it = g_plan_lru->begin(); it != g_plan_lru->end(); ++it)
            if (it->first == key) {
                g_plan_lru->splice(g_plan_lru->begin(), *g_plan_lru, it);
                proto = g_plan_lru->front().second;
                break;
            }
    }
    if (!proto) {
        proto = std::shared_ptr<Plan>(build_proto(m, n, dx, dy, kappa, mod_w, mod_e, device, pair, flags), free_tables);
        std::lock_guard<std::mutex> g(g_plan_mu);
        g_plan_lru->emplace_front(key, proto);
        if (g_plan_lru->size() > kPlanCache) g_plan_lru->pop_back();
    }
    FD_CUDA(cudaSetDevice(device));
    Plan *p = new Plan();
    p->device = proto->device;
    p->m = proto->m;
    p->n = proto->n;
    p->dx = proto->dx;
    p->dy = proto->dy;
    p->kappa = proto->kappa;
    p->mod_w = proto->mod_w;
    p->mod_e = proto->mod_e;
    p->delta_x = proto->delta_x;
    p->delta_y = proto->delta_y;
    p->transform = proto->transform;
    p->explicit_rows = proto->explicit_rows;
    p->dev = proto->dev;
    p->tprof = proto->tprof;
    p->shared = proto;
    p->flags = proto->flags;
    p->sing_modes = proto->sing_modes;
    p->dev.pinv = nullptr;   // pseudo-inverses are attached per plan (fd_plan_set_pinv)
    p->dev.sf = p->dev.sph = nullptr;
    if (p->transform == kDense || p->transform == kSep) {   // pass-1/carry scratch of the three-kernel solves
        try {
            if (p->dev.nsing) {
                const size_t sb = sizeof(double) * size_t(p->dev.nsing) * m;
                p->dev.sf = static_cast<double *>(dmalloc(sb));
                p->allocs.push_back(p->dev.sf);
                p->dev.sph = static_cast<double *>(dmalloc(sb));
                p->allocs.push_back(p->dev.sph);
            }
            const size_t bytes = sizeof(double) * size_t(p->dev.nb) * n;
            p->dev.ye = static_cast<double *>(dmalloc(bytes));
            p->allocs.push_back(p->dev.ye);
            p->dev.fs = static_cast<double *>(dmalloc(bytes));
            p->allocs.push_back(p->dev.fs);
            FD_CUDA(cudaMemset(p->dev.ye, 0, bytes));
            FD_CUDA(cudaMemset(p->dev.fs, 0, bytes));
        } catch (...) {
            for (void *a : p->allocs) dfree(a);
            delete p;
            throw;
        }
    }
    return p;
}

void plan_destroy(Plan *p) {
    if (!p) return;
    cudaSetDevice(p->device);
    cudaDeviceSynchronize();
    for (void *a : p->allocs) dfree(a);
    delete p;   // drops the shared tables reference
}

// Interface-end pivots of the per-mode sweep systems of a DD line of length L:
// inv[k] = 1 / beta_end,k where beta_end is the last pivot of the reference's
// forward recurrence (end = 1: the interface is the sweep's last row) or of the
// same recurrence run from the far end (end = 0: first row), i.e. the corner
// element of the inverse of tridiag(off, lambda_k + end modifiers, off).
void steklov_pivots(int L, int M, double delta_line, double delta_sweep, double kappa, double mod_lo,
                    double mod_hi, int end, double *inv) {
    const double off = delta_sweep;
    parallel_for(L, [&](int k0, int k1) {
        for (int k = k0; k < k1; ++k) {
            const double lam = eig_dd(k, L, delta_line, delta_sweep, kappa);
            // walk from the far end towards the interface row
            const double m_start = end ? mod_lo : mod_hi, m_end = end ? mod_hi : mod_lo;
            double b = lam;
            if (M == 1) {
                b = lam + mod_lo;
                b = b + mod_hi;
            } else {
                b = lam + m_start;
                bool fixed = false;
                for (int i = 1; i < M; ++i) {
                    const double d = (i == M - 1) ? lam + m_end : lam;
                    if (fixed && i < M - 1) continue;   // bitwise fixed point: rows until the last are equal
                    const double l = off / b;
                    const double nb = d - off * l;
                    if (i < M - 1 && nb == b) fixed = true;
                    b = nb;
                }
            }
            inv[k] = 1.0 / b;
        }
    });
}

void factor_tables_host(int m, int n, double dx, double dy, double kappa, double mod_w,
                        double mod_e, double *beta, double *lower) {
    if (m < 1 || n < 1) FD_FAIL(FD_ERR_VALIDATION, "factor: empty grid");
    const int R = (transform_kind(n) >= 0) ? rows_per_block(n) : 16;
    HostTables T = build_tables(m, n, dx, dy, kappa, mod_w, mod_e, R, true);
    for (int k = 0; k < n; ++k) {
        for (int i = 0; i < m; ++i) {
            const bool ex = i < T.len[k];
            const double *r = &T.ex[4 * size_t(T.off[k] + (ex ? i : 0))];
            double l = ex ? r[0] : T.cv[4 * k + 0];
            double b = (i == m - 1) ? T.last[2 * k] : (ex ? r[2] : T.cv[4 * k + 2]);
            beta[size_t(i) * n + k] = b;
            lower[size_t(i) * n + k] = l;
        }
    }
    if (!T.bad_modes.empty()) FD_FAIL(FD_ERR_SINGULAR, "operator singular");
}

}  // namespace fd
