// Internal structures of libfftddm_b200 (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/fftddm_b200.h"

namespace fd {

// ---------------------------------------------------------------------------
// rank-to-rank transport of the sharded solve (comm.cpp): NCCL or loopback
struct Transport {
    int nranks = 1, rank = 0;
    virtual ~Transport() = default;
    virtual void send(const void *buf, size_t bytes, int peer, cudaStream_t s) = 0;
    virtual void recv(void *buf, size_t bytes, int peer, cudaStream_t s) = 0;
    virtual void group_start() {}
    virtual void group_end() {}
};

// ---------------------------------------------------------------------------
// error plumbing
void set_error(const std::string &msg);
struct Error {
    int code;
    std::string msg;
};
#define FD_CUDA(call)                                                              \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess)                                                     \
            throw ::fd::Error{FD_ERR_CUDA, std::string(#call) + ": " +             \
                                               cudaGetErrorString(e_)};           \
    } while (0)
#define FD_FAIL(code, msg) throw ::fd::Error{(code), (msg)}

// ---------------------------------------------------------------------------
// Device view of one rectangle plan.  Passed by value to kernels.
//
// Layout: field (m, n) fp64 row-major; rows = x-lines = sweep axis, columns =
// y = DST axis.  Rows are grouped into carry blocks of R rows (the last one
// may be short): nb = ceil(m / R).
//
// Factor tables (compressed, ref rectsolver.py:62-77): for mode k the rows
// i < ex_len[k] are stored explicitly at ex_off[k] + i; rows >= ex_len[k]
// (a multiple of R) carry the bitwise fixed point (l_inf, beta_inf).  Row m-1
// always uses last_b (it carries the east end modifier).
constexpr int kLtNarrow = 32;   // modes of the narrow slow-mode table: the sweeps' first warp

struct PlanDev {
    int m, n, R, nb;
    double off;          // delta_x: constant off-diagonal of the sweep system
    double nio;          // -1 / off
    double mod_w, mod_e; // sweep-axis end modifiers on rows 0 and m-1
    double scale;        // sqrt(2/(n+1)): orthonormal DST-I factor
    const int *ex_off;   // [n]
    const int *ex_len;   // [n]
    const double *ex;    // [sum ex_len][4]: l, 1/beta, beta, P(block-relative)
    const double *cv;    // [n][4]: l_inf, 1/beta_inf, beta_inf, 1/(-l_inf)
    const double *last;  // [n][2]: beta_{m-1}, 1/beta_{m-1}
    const double *mode;  // [n][8]: l_inf, 1/b_inf, b_inf, 1/(-l_inf), b_last, lambda, ex_off, fixed-point row (int64 bits)
    int ecap;            // rows [0, ecap) of every mode also stored row-major (coalesced):
    const double *dl, *dib, *db;   // [ecap][n] lower, 1/beta, beta
    // slowly converging modes k < kt (ktp = kt rounded to even): row-major factor tables
    // (l_i, 1/beta_i, -beta_{i-1}/delta).  Row groups starting before lt_need read all kt
    // modes from the wide table; from lt_need on every mode >= kLtNarrow is on its fixed
    // point and only the first kta modes are read, from the narrow table
    int kt, ktp, kta, ktpa;
    int lt_rows, lt_need;
    const double *lt;    // [lt_rows][3][ktp], lt_rows >= lt_need + one group of rows
    const double *lta;   // [m][3][ktpa]
    const double *blk;   // [nb][3][n]: Pe, xi_s, Q per block and mode
    double *ye;          // [nb][n] pass-1 local forward value at block end -> Y carries
    double *fs;          // [nb][n] pass-1 local backward value at block start -> X carries
    const double *dense; // [n][n] sin table (dense transform) or nullptr
    const double2 *tw;   // FFT twiddles e^{-2 pi i t / L}, t < L = 2(n+1), or nullptr
    const double *ralpha;// [n+1] real-DST pre-weights (rsolve.cu), alpha_j = s/2 sin(pi j/N) + s/4
    int tpair;           // transform-axis pair: kPairDD (sine), kPairNN (shifted cosine), kPairPP (real Fourier)
    int tkind;           // Transform of the plan (kFFT, kDense, kSep)
    // periodic sweep axis (rectsolver.py:136-153,202-205): the factors above are
    // those of the rank-one modified system; phat -= q_k (vy_k / denom_k)
    int cyclic;
    const double *smq;   // [m][n] correction solves q_k
    const double *cyc;   // [n][2]: delta/gamma_k, denom_k
    // pin_mean singular modes (rectsolver.py:157-175,206-207): phat_k = M_k^+ fhat_k
    int nsing;
    const int *sidx;     // [n]: index of mode k among the singular modes, -1 otherwise
    const double *pinv;  // [nsing][m][m] pseudo-inverses (caller-attached)
    double *sf, *sph;    // [nsing][m] per-plan scratch: fhat columns, M^+ fhat
};

// plan flags (fd_plan_create_sweep)
constexpr int kPlanCyclic = 1, kPlanPinMean = 2;

// transform-axis BC pairs (reference transforms.BC_PAIRS, transforms.py:24)
enum TransformPair { kPairDD = 0, kPairNN = 1, kPairPP = 2 };

// ---------------------------------------------------------------------------
// Geometry of the real-symmetric persistent solve (rsolve.cu), shared with the
// plan builder (long-transient table cap).  N = n + 1 = 2^NL; one CTA of
// kRsThreads per SM; N/16 threads per row pair; the pair regions, twiddles,
// pre-weights and scan scratch are fixed, the rest of the shared memory holds
// one group's slice of the long-transient table (24 B per row and mode).
constexpr int kRsThreads = 512;
constexpr int kRsMinN = 256, kRsMaxN = 4096;
constexpr size_t kRsSmem = 227 * 1024 - 2048;
#ifndef FD_RS_SMALL_N
#define FD_RS_SMALL_N 0
#endif
// N <= FD_RS_SMALL_N: two CTAs of 256 threads per SM (one CTA's barriers and
// copy waits overlap the other's transforms); larger N: one CTA of 512.
#ifndef FD_RS1024_NT
#define FD_RS1024_NT 576
#endif
// N = 1024: nine row pairs per CTA (576 threads, 96 registers), so that a CTA's ~35 rows of
// the c1 batch are two groups of 18 instead of 16 + 16 + 3
#ifndef FD_RS2048_NT
#define FD_RS2048_NT 512
#endif
constexpr int rs_threads(int N) {
    return N <= FD_RS_SMALL_N ? 256 : (N == 1024 ? FD_RS1024_NT : N == 2048 ? FD_RS2048_NT : kRsThreads);
}
constexpr size_t rs_smem(int N) { return rs_threads(N) == 256 ? size_t(110) * 1024 : kRsSmem; }
constexpr int rs_pairs(int N) { return rs_threads(N) / (N / 16); }
constexpr int rs_rows_per_group(int N) { return 2 * rs_pairs(N); }
constexpr size_t rs_fixed_smem(int N) {
    return size_t(rs_pairs(N)) * size_t(N + N / 16) * 16 + 272 * 16 + size_t(N) * 8 +
           size_t(rs_pairs(N)) * 16 * 8;
}
#ifndef FD_KT_CAP_MAX
#define FD_KT_CAP_MAX (1 << 20)   // test builds lower it to drive modes onto the capped-table paths
#endif
constexpr int rs_kt_cap(int N) {
    const int cap = int((rs_smem(N) - rs_fixed_smem(N)) / (24 * size_t(rs_rows_per_group(N)))) & ~1;
    return cap < FD_KT_CAP_MAX ? cap : FD_KT_CAP_MAX;
}
inline bool rs_supported(int n) {
    const int N = n + 1;
    return N >= kRsMinN && N <= kRsMaxN && (N & (N - 1)) == 0;
}

enum Transform { kDense = 0, kFFT = 1, kSep = 2 };   // kSep: any-length transform passes + sweeps
constexpr int kDenseMax = 2048;   // longest dense periodic-table transform (dst_device.cuh)
constexpr int kSepMax = 65535;    // longest any-length transform (fft_any.cu: power-of-two sizes <= 2^18)

// Device allocations of plans, operators and the Krylov basis come from the
// device's stream-ordered pool with an unbounded release threshold, so the
// gigabytes a c3/c4 solve allocates are recycled by the next solve instead of
// going back to the driver (cudaMalloc + cudaFree of the 6.8 GB basis cost
// ~0.9 s per solve).  dfree() callers synchronise the device first (destroy
// paths), like cudaFree would.
void *dmalloc(size_t bytes);
void dfree(void *p);

// grow-only device scratch (block carries of the persistent solve)
struct Workspace {
    double *ptr = nullptr;
    size_t cap = 0;
    double *get(size_t count) {
        if (count > cap) {
            if (ptr) {
                cudaDeviceSynchronize();
                dfree(ptr);
            }
            ptr = nullptr;
            cap = 0;
            ptr = static_cast<double *>(dmalloc(count * sizeof(double)));
            cap = count;
        }
        return ptr;
    }
    ~Workspace() {
        if (ptr) dfree(ptr);
    }
};

struct Plan {
    int device;
    int m, n;
    double dx, dy, kappa, mod_w, mod_e;
    double delta_x, delta_y;
    int transform;
    long long explicit_rows;
    PlanDev dev;
    std::vector<float> tprof;   // see SolveJob::tprof
    std::vector<void *> allocs;
    Workspace ws;
    std::shared_ptr<Plan> shared;   // immutable device tables shared by identical plans (plan.cpp)
    int flags = 0;                  // kPlanCyclic | kPlanPinMean
    std::vector<int> sing_modes;    // singular spectral modes (pin_mean plans)
    bool pinv_ready = false;
    // transform along x (reference transform_axis == "x"): the tables above are
    // those of the transposed rectangle (m, n) = (user n, user m); user-layout
    // fields are transposed into tws around the solve
    bool transposed = false;
    int um = 0, un = 0;   // user-layout rows (x-lines), columns (y)
    Workspace tws;
};

// one job of a batched rectangle launch
struct SolveJob {
    PlanDev p;
    const double *in;
    double *out;
    // pass-2 epilogue: out = alpha * x + beta * other  (other may be null)
    double alpha, beta;
    const double *other;
    Workspace *ws;   // host-side: scratch owner for the batch (unused on device)
    // host-side cost profile of the sweep rows (row partition of the persistent
    // solves): tprof[i] = fraction of modes still in their transient at row i
    const float *tprof = nullptr;
    int tlen = 0;
};

constexpr int kMaxJobs = 8;
struct JobList {
    int count;
    int block_start[kMaxJobs + 1];  // prefix of CTAs per job
    SolveJob job[kMaxJobs];
};

// kernels / launchers (solve.cu)
int rows_per_block(int n, int pair = kPairDD);
int transform_kind(int n, int pair = kPairDD);
void launch_solve(const std::vector<SolveJob> &jobs, cudaStream_t s);
// any-length transforms (fft_any.cu): complex DFT rows (power of two: Stockham;
// otherwise Bluestein) and the real row transforms of the three pairs
void dft_rows(long long rows, int M, const double2 *in, double2 *out, int inverse, cudaStream_t st);
void transform_rows_any(long long rows, int n, int pair, int inverse, const double *in, double *out, double alpha,
                        double beta, const double *other, cudaStream_t st);
bool launch_persist(const std::vector<SolveJob> &jobs, cudaStream_t s, Workspace &ws);
void launch_transform_rows(int rows, int n, int pair, int inverse, const double *in, double *out,
                           const double *dense, cudaStream_t s);
void launch_dst_rows(int rows, int n, const double *in, double *out, const double2 *tw,
                     const double *dense, cudaStream_t s);
const double2 *twiddles_for(int device, int n);
const double *dense_table_for(int device, int n, int pair = kPairDD, bool force = false);

// vector kernels (ops.cu)
void launch_stencil(int m, int n, double delta_x, double delta_y, double kappa, double mw,
                    double me, double ms, double mn, const double *v, double *out, cudaStream_t s,
                    int ppx = 0, int ppy = 0);
inline void launch_stencil(const Plan &p, double ms, double mn, const double *v, double *out,
                           cudaStream_t s) {
    launch_stencil(p.m, p.n, p.delta_x, p.delta_y, p.kappa, p.mod_w, p.mod_e, ms, mn, v, out, s);
}
void launch_scatter(int len, const int64_t *from, const int64_t *to, double c, const double *src,
                    double *dst, int accumulate, cudaStream_t s);
void launch_assemble(int m, int n, double x0, double y0, double dx, double dy, double kappa, int sol,
                     const double lift[4], double *f, double *exact, cudaStream_t s);
void launch_mul(long long N, const double *x, const double *y, double *out, cudaStream_t s);   // out = x * y
void steklov_pivots(int L, int M, double delta_line, double delta_sweep, double kappa, double mod_lo,
                    double mod_hi, int end, double *inv);
void launch_zero_at(int len, const int64_t *to, double *dst, cudaStream_t s);   // dst[to[t]] = 0
// Several index maps in one launch (one grid row per map).  mode 0: dst[to] =
// c src[from] (maps with distinct destinations); 1: dst[to] += c src[from] by
// atomic add -- only for a zero destination that receives at most two
// contributions per entry, where the result is independent of the order
// (0 + a + b == 0 + b + a bitwise); 2: dst[to] = 0.
constexpr int kMaxScatter = 8;
struct ScatterBatch {
    int count = 0;
    int len[kMaxScatter];
    const int64_t *from[kMaxScatter];
    const int64_t *to[kMaxScatter];
    double c[kMaxScatter];
    const double *src[kMaxScatter];
    double *dst[kMaxScatter];
};
void launch_scatter_batch(const ScatterBatch &b, int mode, cudaStream_t s);
void launch_axpby(long long N, double a, const double *x, double b, const double *y, double *out,
                  cudaStream_t s);
// deterministic reductions: result written to device scalar *out
struct RedWork {
    double *partials;   // [kRedBlocks]
    unsigned int *counter;
};
constexpr int kRedBlocks = 592;  // 4 x 148 SMs
void launch_dot(long long N, const double *x, const double *y, double *out, RedWork w,
                cudaStream_t s);
// fused MGS step: w -= (*h_prev) * vprev (if vprev); *h_out = vi . w   (vi may be null -> ||w||^2)
void launch_mgs(long long N, double *w, const double *vprev, const double *h_prev,
                const double *vi, double *h_out, RedWork wk, cudaStream_t s);
// low-synchronisation MGS Arnoldi (see ops.cu)
constexpr int kMaxArnoldi = 128;           // basis vectors V_0..V_k per step, k + 1 <= 128 (m <= 127)
struct ArnWork {
    double *partials;        // [grid][2 * kMaxArnoldi + 2]
    unsigned int *counter;
    double *G;               // Gram rows: G[i * ldg + j] = V_i . V_j, j < i
    double *out;             // results of the launch
};
constexpr size_t kArnPartials = size_t(148) * 16 * (2 * kMaxArnoldi + 2);
// out[0..k] = h (MGS projections), out[k+1] = ||w||^2 before orthogonalisation; Gram row k stored
void launch_arnoldi_dots(long long N, int k, const double *V, const double *w, ArnWork a, int ldg,
                         cudaStream_t s);
// w -= sum_j h_j V_j (j ascending); out[0] = ||w||^2 after
void launch_arnoldi_update(long long N, int k, const double *V, double *w, const double *h, ArnWork a,
                           cudaStream_t s);
void launch_scale_sqrt(long long N, const double *x, const double *nrm2, double *out, cudaStream_t s);
// out (C x R) = alpha * in^T + beta * other (other may be null); in is R x C
void launch_transpose(int R, int C, const double *in, double *out, double alpha, double beta,
                      const double *other, cudaStream_t s);
void launch_basis_update(long long N, int k, const double *V, const double *y_dev, double *x,
                         cudaStream_t s);
void launch_scale(long long N, const double *x, const double *s_dev, double *out, cudaStream_t s);

}  // namespace fd

struct fd_comm_s {
    std::unique_ptr<fd::Transport> t;
    int device;
};
