// Transforms of any length (the reference's transforms.py:74-148 formulations,
// every one a single complex FFT per row) and the rectangle solve built on
// them, for lengths the fused kernels do not take (n + 1 not a power of two
// with n > 2048, NN / PP axes longer than 2048):
//
//   DD   Q = Q^T:  odd extension of length M = 2(n+1), X = -Im(FFT)/2 * s
//                  (transforms.py:74-80); two rows ride in one complex FFT
//                  (Re Z = 2 S_b, Im Z = -2 S_a)
//   NN   Q^T: even extension, M = 2n, X_k = s_k Re(e^{-i pi k/2n} F_k)/2
//                  (dct2, transforms.py:83-89)
//        Q:   z_j = s_j a_j e^{i pi j/2n}, M = 2n, X = Re(inverse DFT)
//                  (dct3, transforms.py:92-97)
//   PP   Q^T: F = FFT_n(v), cosine / sine amplitudes (transforms.py:139-148)
//        Q:   half spectrum -> inverse DFT (transforms.py:114-126)
//
// The complex DFT of length M: 7-smooth M by mixed-radix (4, 2, 3, 5, 7)
// Stockham passes in shared memory (M <= 4096 in one kernel over the row;
// larger M as a four-step P1 x P2 split, lines staged through shared memory
// several at a time so the strided accesses coalesce); any other M by
// Bluestein's chirp-z (X_k = w_k sum_j (x_j w_j) conj(w_{k-j}),
// w_j = e^{-i pi j^2 / M}) as a power-of-two cyclic convolution of length
// P >= 2M - 1.
#include <math.h>

#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "dst_device.cuh"
#include "fd_internal.h"

namespace fd {

// ---------------------------------------------------------------------------
// batched power-of-two FFT of "lines": line l of row r holds element e at
//   base + r * row + l * ls + e * es      (complex units)
struct Lines {
    const double2 *in;
    double2 *out;
    int L, logL;                 // line length 2^logL <= 4096
    int lines;                   // lines per row
    long long rows;
    long long in_row, out_row;
    long long in_ls, in_es, out_ls, out_es;
    const double2 *tw;           // W_L^k = e^{-2 pi i k / L}, k < L
    const double2 *post;         // optional W_P^j, j < P: output (l, k) times W_P^{l k}
    int P;
    int inverse;                 // conjugate twiddles (e^{+2 pi i jk/L}), unnormalised
    int nfac;                    // radix sequence of L (4, 2, 3, 5, 7), product L
    int fac[24];
};

constexpr int kFftThreads = 256;
constexpr int kFftSmemC = 8192;   // complex values per CTA (2 x 64 KB ping-pong)

__device__ __forceinline__ double2 twv(const double2 *tw, int idx, int inverse) {
    const double2 w = __ldg(tw + idx);
    return make_double2(w.x, inverse ? -w.y : w.y);
}

// in-place R-point DFT (R = 2, 3, 4, 5, 7) with roots e^{-+2 pi i / R}
template <int R>
__device__ __forceinline__ void small_dft(double2 (&v)[7], int inverse) {
    if constexpr (R == 2) {
        const double2 a = v[0];
        v[0] = cadd(a, v[1]);
        v[1] = csub(a, v[1]);
    } else if constexpr (R == 4) {
        const double2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]), s13 = cadd(v[1], v[3]), d13 = csub(v[1], v[3]);
        const double2 rd13 = inverse ? make_double2(-d13.y, d13.x) : make_double2(d13.y, -d13.x);
        v[0] = cadd(s02, s13);
        v[1] = cadd(d02, rd13);
        v[2] = csub(s02, s13);
        v[3] = csub(d02, rd13);
    } else {
        // cos / sin (2 pi m / R), m < R
        constexpr double c3[3] = {1.0, -0.5, -0.5}, s3[3] = {0.0, 0.8660254037844386467637, -0.8660254037844386467637};
        constexpr double c5[5] = {1.0, 0.3090169943749474241023, -0.8090169943749474241023, -0.8090169943749474241023,
                                  0.3090169943749474241023};
        constexpr double s5[5] = {0.0, 0.9510565162951535721164, 0.5877852522924731291687, -0.5877852522924731291687,
                                  -0.9510565162951535721164};
        constexpr double c7[7] = {1.0, 0.623489801858733530525, -0.2225209339563144042889, -0.9009688679024191262361,
                                  -0.9009688679024191262361, -0.2225209339563144042889, 0.623489801858733530525};
        constexpr double s7[7] = {0.0, 0.7818314824680298087084, 0.9749279121818236070181, 0.4338837391175581204758,
                                  -0.4338837391175581204758, -0.9749279121818236070181, -0.7818314824680298087084};
        double2 o[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            double2 acc = v[0];
#pragma unroll
            for (int j = 1; j < R; ++j) {
                const int mm = (j * k) % R;
                const double cs = R == 3 ? c3[mm] : R == 5 ? c5[mm] : c7[mm];
                const double sn = R == 3 ? s3[mm] : R == 5 ? s5[mm] : s7[mm];
                acc = cadd(acc, cmul(v[j], make_double2(cs, inverse ? sn : -sn)));
            }
            o[k] = acc;
        }
#pragma unroll
        for (int k = 0; k < R; ++k) v[k] = o[k];
    }
}

template <int R>
__device__ __forceinline__ void stockham_pass(const Lines &s, const double2 *x, double2 *y, int nl, int Ns) {
    const int L = s.L, span = L / R;
    for (int q = threadIdx.x; q < nl * span; q += kFftThreads) {
        const int li = q / span, j = q % span;
        const double2 *xl = x + li * L;
        double2 *yl = y + li * L;
        double2 v[7];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = xl[j + r * span];
        const int k = j % Ns;
        if (k) {
            const int step = L / (R * Ns);   // e^{-2 pi i k r / (R Ns)} = W_L^{k r step}
#pragma unroll
            for (int r = 1; r < R; ++r) v[r] = cmul(v[r], twv(s.tw, (k * r * step) % L, s.inverse));
        }
        small_dft<R>(v, s.inverse);
        const int o = (j / Ns) * Ns * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) yl[o + r * Ns] = v[r];
    }
}

// LB lines of length L per CTA, one Stockham pass per radix of L (natural-order
// output, ping-pong buffers in shared memory)
__global__ void __launch_bounds__(kFftThreads) fft_lines_kernel(const __grid_constant__ Lines s) {
    extern __shared__ __align__(16) double2 fsm[];
    const int L = s.L;
    const int LB = max(1, min(kFftSmemC / 2 / L, 32));
    double2 *x = fsm, *y = fsm + LB * L;
    const long long blocks_per_row = (s.lines + LB - 1) / LB;
    const long long r = blockIdx.x / blocks_per_row;
    const int l0 = int(blockIdx.x % blocks_per_row) * LB;
    const int nl = min(LB, s.lines - l0);
    if (r >= s.rows) return;
    const double2 *in = s.in + r * s.in_row;
    double2 *out = s.out + r * s.out_row;
    const int total = nl * L;
    // load: consecutive threads walk the dimension with unit stride
    const bool line_fast_in = s.in_es != 1;
    for (int q = threadIdx.x; q < total; q += kFftThreads) {
        const int li = line_fast_in ? q % nl : q / L, e = line_fast_in ? q / nl : q % L;
        x[li * L + e] = in[(l0 + li) * s.in_ls + e * s.in_es];
    }
    __syncthreads();
    int Ns = 1;
    for (int f = 0; f < s.nfac; ++f) {
        switch (s.fac[f]) {
            case 4: stockham_pass<4>(s, x, y, nl, Ns); break;
            case 2: stockham_pass<2>(s, x, y, nl, Ns); break;
            case 3: stockham_pass<3>(s, x, y, nl, Ns); break;
            case 5: stockham_pass<5>(s, x, y, nl, Ns); break;
            default: stockham_pass<7>(s, x, y, nl, Ns); break;
        }
        Ns *= s.fac[f];
        __syncthreads();
        double2 *t = x;
        x = y;
        y = t;
    }
    const bool line_fast_out = s.out_es != 1;
    for (int q = threadIdx.x; q < total; q += kFftThreads) {
        const int li = line_fast_out ? q % nl : q / L, e = line_fast_out ? q / nl : q % L;
        double2 v = x[li * L + e];
        if (s.post) v = cmul(v, twv(s.post, int((long long)(l0 + li) * e % s.P), s.inverse));
        out[(l0 + li) * s.out_ls + e * s.out_es] = v;
    }
}

// radix sequence of L (4s first, then 2, 3, 5, 7); false unless L is 7-smooth
static bool factor_smooth(int L, Lines &s) {
    s.nfac = 0;
    int v = L;
    for (int r : {4, 2, 3, 5, 7})
        while (v % r == 0 && s.nfac < 24) {
            s.fac[s.nfac++] = r;
            v /= r;
        }
    return v == 1;
}

static size_t lines_smem() { return size_t(kFftSmemC) * sizeof(double2); }

static void run_lines(const Lines &s, cudaStream_t st) {
    static std::once_flag once;
    std::call_once(once, [] {
        FD_CUDA(cudaFuncSetAttribute(fft_lines_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)lines_smem()));
    });
    const int LB = std::max(1, std::min(kFftSmemC / 2 / s.L, 32));
    const long long blocks = s.rows * ((s.lines + LB - 1) / LB);
    if (blocks == 0) return;
    if (blocks > 0x7fffffffLL) FD_FAIL(FD_ERR_VALIDATION, "fft: too many lines");
    fft_lines_kernel<<<(unsigned)blocks, kFftThreads, lines_smem(), st>>>(s);
    FD_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// per-device tables
static std::mutex g_any_mu;
static std::map<std::pair<int, int>, double2 *> g_pow2_tw;   // (device, P) -> W_P^k

static const double2 *pow2_twiddles(int device, int P) {   // W_P^k, k < P (any P)
    std::lock_guard<std::mutex> g(g_any_mu);
    auto key = std::make_pair(device, P);
    auto it = g_pow2_tw.find(key);
    if (it != g_pow2_tw.end()) return it->second;
    std::vector<double2> h(P);
    const long double PI = 3.141592653589793238462643383279502884L;
    for (int k = 0; k < P; ++k) {
        const long double a = 2.0L * PI * (long double)k / (long double)P;
        h[k] = make_double2((double)cosl(a), (double)(-sinl(a)));
    }
    double2 *d = static_cast<double2 *>(dmalloc(sizeof(double2) * P));
    FD_CUDA(cudaMemcpy(d, h.data(), sizeof(double2) * P, cudaMemcpyHostToDevice));
    g_pow2_tw[key] = d;   // kept for the process lifetime (small)
    return d;
}

static int ilog2(long long v) {
    int l = 0;
    while ((1LL << l) < v) ++l;
    return l;
}

// M = P1 * P2 with both factors <= 4096 (any such split of a 7-smooth M),
// P1 the smallest factor >= sqrt(M); false when there is none
static bool smooth_split(int M, int &P1, int &P2) {
    Lines t{};
    if (!factor_smooth(M, t)) return false;
    for (int a = 1; a <= 4096; ++a) {
        if (M % a || (long long)a * a < M) continue;
        if (M / a <= 4096) {
            P1 = a;
            P2 = M / a;
            return true;
        }
    }
    return false;
}

// rows x P (row stride P) DFT of a 7-smooth length P, in -> out (out may equal
// in for P <= 4096; the four-step split goes through `tmp`, rows x P)
static void fft_smooth(long long rows, int P, const double2 *in, double2 *out, double2 *tmp, int inverse,
                       cudaStream_t st, int device) {
    if (P <= 4096) {
        Lines s{};
        s.in = in;
        s.out = out;
        s.L = P;
        s.lines = 1;
        s.rows = rows;
        s.in_row = s.out_row = P;
        s.in_ls = s.out_ls = P;
        s.in_es = s.out_es = 1;
        s.tw = pow2_twiddles(device, P);
        s.inverse = inverse;
        if (!factor_smooth(P, s)) FD_FAIL(FD_ERR_UNSUPPORTED, "fft: length is not 7-smooth");
        run_lines(s, st);
        return;
    }
    int P1 = 0, P2 = 0;
    if (!smooth_split(P, P1, P2)) FD_FAIL(FD_ERR_UNSUPPORTED, "fft: no four-step split of this length");
    // four-step: x[n2 + P2 n1], X[k1 + P1 k2]
    // A: for each n2, DFT over n1 (stride P2), times W_P^{n2 k1} -> tmp[k1 * P2 + n2]
    Lines a{};
    a.in = in;
    a.out = tmp;
    a.L = P1;
    a.lines = P2;
    a.rows = rows;
    a.in_row = a.out_row = P;
    a.in_ls = 1;
    a.in_es = P2;
    a.out_ls = 1;
    a.out_es = P2;
    a.tw = pow2_twiddles(device, P1);
    a.post = pow2_twiddles(device, P);
    a.P = P;
    a.inverse = inverse;
    factor_smooth(P1, a);
    run_lines(a, st);
    // B: for each k1, DFT over n2 (contiguous in tmp) -> out[k1 + P1 k2]
    Lines b{};
    b.in = tmp;
    b.out = out;
    b.L = P2;
    b.lines = P1;
    b.rows = rows;
    b.in_row = b.out_row = P;
    b.in_ls = P2;
    b.in_es = 1;
    b.out_ls = 1;
    b.out_es = P1;
    b.tw = pow2_twiddles(device, P2);
    b.inverse = inverse;
    factor_smooth(P2, b);
    run_lines(b, st);
}
static void fft_pow2(long long rows, int P, const double2 *in, double2 *out, double2 *tmp, int inverse,
                     cudaStream_t st, int device) {
    if (P > (1 << 18)) FD_FAIL(FD_ERR_UNSUPPORTED, "fft: length above 2^18");
    fft_smooth(rows, P, in, out, tmp, inverse, st, device);
}

// Bluestein data of a length M: chirp w_j = e^{-i pi j^2 / M} (j < M) and the
// power-of-two transform of the convolution kernel b (b_j = conj w_j, wrapped)
struct Chirp {
    int M, P;
    double2 *w;      // [M]
    double2 *bhat;   // [P]
};
static std::map<std::pair<int, int>, Chirp> g_chirp;

// a_j = (conj? conj(x_j) : x_j) w_j, zero-padded to P
__global__ void chirp_mul_kernel(long long rows, int M, int P, const double2 *in, long long in_row, int in_es,
                                 const double2 *w, double2 *out, int conj_in) {
    const long long tot = rows * P;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < tot; q += (long long)gridDim.x * blockDim.x) {
        const long long r = q / P;
        const int j = int(q % P);
        double2 v = make_double2(0.0, 0.0);
        if (j < M) {
            v = in[r * in_row + (long long)j * in_es];
            if (conj_in) v.y = -v.y;
            v = cmul(v, __ldg(w + j));
        }
        out[q] = v;
    }
}
__global__ void spec_mul_kernel(long long rows, int P, double2 *a, const double2 *bhat) {
    const long long tot = rows * P;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < tot; q += (long long)gridDim.x * blockDim.x)
        a[q] = cmul(a[q], __ldg(bhat + q % P));
}
// X_k = w_k * conv_k / P for k < M (the 1/P of the convolution's inverse
// transform), conjugated for an inverse DFT
__global__ void chirp_out_kernel(long long rows, int M, int P, const double2 *conv, const double2 *w, double2 *out,
                                 long long out_row, int conj_out) {
    const long long tot = rows * M;
    const double s = 1.0 / P;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < tot; q += (long long)gridDim.x * blockDim.x) {
        const long long r = q / M;
        const int k = int(q % M);
        const double2 c = cmul(conv[r * P + k], __ldg(w + k));
        out[r * out_row + k] = make_double2(c.x * s, (conj_out ? -c.y : c.y) * s);
    }
}

static int ew_grid(long long n) { return (int)std::min<long long>((n + 255) / 256, 148LL * 16); }

static const Chirp &chirp_for(int device, int M, cudaStream_t st) {
    {
        std::lock_guard<std::mutex> g(g_any_mu);
        auto it = g_chirp.find({device, M});
        if (it != g_chirp.end()) return it->second;
    }
    Chirp c{};
    c.M = M;
    c.P = 1 << ilog2(2LL * M - 1);
    std::vector<double2> w(M), b(c.P, make_double2(0.0, 0.0));
    const long double PI = 3.141592653589793238462643383279502884L;
    for (int j = 0; j < M; ++j) {
        const long long q = (long long)j * j % (2LL * M);   // exact argument reduction
        const long double a = PI * (long double)q / (long double)M;
        w[j] = make_double2((double)cosl(a), (double)(-sinl(a)));
        b[j] = make_double2(w[j].x, -w[j].y);
        if (j) b[c.P - j] = b[j];
    }
    c.w = static_cast<double2 *>(dmalloc(sizeof(double2) * M));
    c.bhat = static_cast<double2 *>(dmalloc(sizeof(double2) * c.P));
    FD_CUDA(cudaMemcpy(c.w, w.data(), sizeof(double2) * M, cudaMemcpyHostToDevice));
    FD_CUDA(cudaMemcpy(c.bhat, b.data(), sizeof(double2) * c.P, cudaMemcpyHostToDevice));
    double2 *tmp = static_cast<double2 *>(dmalloc(sizeof(double2) * c.P));
    fft_pow2(1, c.P, c.bhat, c.bhat, tmp, 0, st, device);
    FD_CUDA(cudaStreamSynchronize(st));
    dfree(tmp);
    std::lock_guard<std::mutex> g(g_any_mu);
    return g_chirp.emplace(std::make_pair(device, M), c).first->second;
}

// grow-only scratch per device (complex)
static std::map<int, Workspace> g_any_ws;
static double2 *any_scratch(int device, size_t count) {
    std::lock_guard<std::mutex> g(g_any_mu);
    return reinterpret_cast<double2 *>(g_any_ws[device].get(2 * count));
}

constexpr long long kDftChunk = 1LL << 24;   // complex values per scratch chunk (256 MB)

// rows x M complex DFT of any length (row stride M): forward e^{-2 pi i jk/M}
// or inverse e^{+2 pi i jk/M}, unnormalised; out may alias in.
void dft_rows(long long rows, int M, const double2 *in, double2 *out, int inverse, cudaStream_t st) {
    if (rows <= 0) return;
    int device = 0;
    FD_CUDA(cudaGetDevice(&device));
    int P1 = 0, P2 = 0;
    if (M <= 4096 ? [&] { Lines t{}; return factor_smooth(M, t); }() : smooth_split(M, P1, P2)) {
        // 7-smooth: mixed-radix Stockham passes (four-step above 4096)
        const long long chunk = std::max<long long>(1, kDftChunk / M);
        double2 *tmp = M > 4096 ? any_scratch(device, size_t(std::min(rows, chunk)) * M) : nullptr;
        for (long long r0 = 0; r0 < rows; r0 += chunk) {
            const long long rr = std::min(chunk, rows - r0);
            fft_smooth(rr, M, in + r0 * M, out + r0 * M, tmp, inverse, st, device);
        }
        return;
    }
    const Chirp &c = chirp_for(device, M, st);
    const int P = c.P;
    const long long chunk = std::max<long long>(1, kDftChunk / (2LL * P));
    const long long rmax = std::min(rows, chunk);
    double2 *a = any_scratch(device, size_t(rmax) * P * 2);
    double2 *t = a + size_t(rmax) * P;
    for (long long r0 = 0; r0 < rows; r0 += chunk) {
        const long long rr = std::min(chunk, rows - r0);
        // the inverse DFT is conj(forward DFT(conj x))
        chirp_mul_kernel<<<ew_grid(rr * P), 256, 0, st>>>(rr, M, P, in + r0 * M, M, 1, c.w, a, inverse);
        FD_CUDA(cudaGetLastError());
        fft_pow2(rr, P, a, a, t, 0, st, device);
        spec_mul_kernel<<<ew_grid(rr * P), 256, 0, st>>>(rr, P, a, c.bhat);
        FD_CUDA(cudaGetLastError());
        fft_pow2(rr, P, a, a, t, 1, st, device);
        chirp_out_kernel<<<ew_grid(rr * M), 256, 0, st>>>(rr, M, P, a, c.w, out + r0 * M, M, inverse);
        FD_CUDA(cudaGetLastError());
    }
}

}  // namespace fd

namespace fd {

// ---------------------------------------------------------------------------
// real row transforms of any length on top of dft_rows
__global__ void dd_pre_kernel(long long pairs, long long rows, int n, const double *in, double2 *z) {
    const int N = n + 1, M = 2 * N;
    const long long tot = pairs * M;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < tot; q += (long long)gridDim.x * blockDim.x) {
        const long long p = q / M;
        const int j = int(q % M);
        const long long ra = 2 * p, rb = 2 * p + 1;
        double a = 0.0, b = 0.0;   // odd extension: x_j, 0 at j = 0, N, -x_{2N-j} above N
        if (j != 0 && j != N) {
            const int src = j < N ? j - 1 : M - j - 1;
            const double sg = j < N ? 1.0 : -1.0;
            a = sg * in[ra * n + src];
            if (rb < rows) b = sg * in[rb * n + src];
        }
        z[q] = make_double2(a, b);
    }
}
// X_a = -Im Z / 2 * s, X_b = Re Z / 2 * s (transforms.py:80, 110-113)
__global__ void dd_post_kernel(long long pairs, long long rows, int n, const double2 *Z, double *out,
                               double alpha, double beta, const double *other) {
    const int M = 2 * (n + 1);
    const double s = sqrt(2.0 / (n + 1));
    const long long tot = pairs * n;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < tot; q += (long long)gridDim.x * blockDim.x) {
        const long long p = q / n;
        const int k = int(q % n);
        const double2 z = Z[p * M + k + 1];
        const double a = -0.5 * z.y * s, b = 0.5 * z.x * s;
        const long long ra = 2 * p, rb = 2 * p + 1;
        double va = alpha * a;
        if (other) va = fma(beta, other[ra * n + k], va);
        out[ra * n + k] = va;
        if (rb < rows) {
            double vb = alpha * b;
            if (other) vb = fma(beta, other[rb * n + k], vb);
            out[rb * n + k] = vb;
        }
    }
}
__device__ __forceinline__ double nn_sc(int k, int n) { return k == 0 ? sqrt(1.0 / n) : sqrt(2.0 / n); }
// Q^T: even extension (transforms.py:83-89) | Q: phase-shifted half spectrum (transforms.py:92-97)
__global__ void nn_pre_kernel(long long rows, int n, int inverse, const double *in, double2 *z) {
    const int M = 2 * n;
    const long long tot = rows * M;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < tot; q += (long long)gridDim.x * blockDim.x) {
        const long long r = q / M;
        const int j = int(q % M);
        if (!inverse) {
            z[q] = make_double2(in[r * n + (j < n ? j : M - 1 - j)], 0.0);
        } else if (j < n) {
            double sn, cs;
            sincospi(double(j) / double(M), &sn, &cs);   // e^{i pi j / 2n}
            const double a = nn_sc(j, n) * in[r * n + j];
            z[q] = make_double2(a * cs, a * sn);
        } else {
            z[q] = make_double2(0.0, 0.0);
        }
    }
}
__global__ void nn_post_kernel(long long rows, int n, int inverse, const double2 *Z, double *out, double alpha,
                               double beta, const double *other) {
    const int M = 2 * n;
    const long long tot = rows * n;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < tot; q += (long long)gridDim.x * blockDim.x) {
        const long long r = q / n;
        const int k = int(q % n);
        const double2 z = Z[r * M + k];
        double v;
        if (!inverse) {   // s_k * 0.5 * Re(e^{-i pi k / 2n} F_k)
            double sn, cs;
            sincospi(double(k) / double(M), &sn, &cs);
            v = nn_sc(k, n) * (0.5 * (cs * z.x + sn * z.y));
        } else {
            v = z.x;
        }
        v *= alpha;
        if (other) v = fma(beta, other[r * n + k], v);
        out[r * n + k] = v;
    }
}
// real Fourier basis, even n (transforms.py:114-126 Q, 139-148 Q^T)
__global__ void pp_pre_kernel(long long rows, int n, int inverse, const double *in, double2 *z) {
    const long long tot = rows * n;
    const double root = sqrt(1.0 / n), amp = sqrt(2.0 / n);
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < tot; q += (long long)gridDim.x * blockDim.x) {
        const long long r = q / n;
        const int k = int(q % n);
        const double v = in[r * n + k];
        if (!inverse) {
            z[q] = make_double2(v, 0.0);
        } else if (k == 0 || k == n / 2) {
            z[q] = make_double2(v * root, 0.0);
        } else if (k < n / 2) {
            z[q] = make_double2(amp * v, 0.0);
        } else {
            z[q] = make_double2(0.0, -amp * v);
        }
    }
}
__global__ void pp_post_kernel(long long rows, int n, int inverse, const double2 *Z, double *out, double alpha,
                               double beta, const double *other) {
    const long long tot = rows * n;
    const double root = sqrt(1.0 / n), amp = sqrt(2.0 / n);
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < tot; q += (long long)gridDim.x * blockDim.x) {
        const long long r = q / n;
        const int k = int(q % n);
        const double2 z = Z[q];
        double v;
        if (inverse) v = z.x;
        else if (k == 0 || k == n / 2) v = z.x * root;
        else if (k < n / 2) v = amp * z.x;
        else v = -amp * z.y;
        v *= alpha;
        if (other) v = fma(beta, other[r * n + k], v);
        out[r * n + k] = v;
    }
}

static std::map<int, Workspace> g_rows_ws;   // complex row buffers of transform_rows_any

// rows x n real rows along the transform axis: out = alpha * T(in) + beta * other
// with T = Q (inverse) or Q^T, out may alias in
void transform_rows_any(long long rows, int n, int pair, int inverse, const double *in, double *out, double alpha,
                        double beta, const double *other, cudaStream_t st) {
    if (rows <= 0) return;
    int device = 0;
    FD_CUDA(cudaGetDevice(&device));
    const int M = pair == kPairDD ? 2 * (n + 1) : pair == kPairNN ? 2 * n : n;
    const bool packed = pair == kPairDD;   // two real rows per complex row
    const long long lines = packed ? (rows + 1) / 2 : rows;
    const long long chunk = std::max<long long>(1, (1LL << 23) / M);   // lines per pass (<= 128 MB)
    double2 *z;
    {
        std::lock_guard<std::mutex> g(g_any_mu);
        z = reinterpret_cast<double2 *>(g_rows_ws[device].get(2 * size_t(std::min(lines, chunk)) * M));
    }
    for (long long l0 = 0; l0 < lines; l0 += chunk) {
        const long long ln = std::min(chunk, lines - l0);
        const long long r0 = packed ? 2 * l0 : l0;
        const long long rn = packed ? std::min(2 * ln, rows - r0) : ln;
        const double *ip = in + r0 * n;
        double *op = out + r0 * n;
        const double *qp = other ? other + r0 * n : nullptr;
        const int g = ew_grid(ln * M);
        if (pair == kPairDD) {
            dd_pre_kernel<<<g, 256, 0, st>>>(ln, rn, n, ip, z);
            FD_CUDA(cudaGetLastError());
            dft_rows(ln, M, z, z, 0, st);
            dd_post_kernel<<<ew_grid(ln * n), 256, 0, st>>>(ln, rn, n, z, op, alpha, beta, qp);
        } else if (pair == kPairNN) {
            nn_pre_kernel<<<g, 256, 0, st>>>(ln, n, inverse, ip, z);
            FD_CUDA(cudaGetLastError());
            dft_rows(ln, M, z, z, inverse, st);
            nn_post_kernel<<<ew_grid(ln * n), 256, 0, st>>>(ln, n, inverse, z, op, alpha, beta, qp);
        } else {
            pp_pre_kernel<<<g, 256, 0, st>>>(ln, n, inverse, ip, z);
            FD_CUDA(cudaGetLastError());
            dft_rows(ln, M, z, z, inverse, st);
            pp_post_kernel<<<ew_grid(ln * n), 256, 0, st>>>(ln, n, inverse, z, op, alpha, beta, qp);
        }
        FD_CUDA(cudaGetLastError());
    }
}

}  // namespace fd
