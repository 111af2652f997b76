// ARCHIVED EXPERIMENT (round 2, session 3) -- not compiled into libfftddm_b200.so.
// To build it again: copy to paper_2509_23180_b200/csrc/split.cu, declare
// `bool launch_split(const std::vector<SolveJob>&, cudaStream_t, Workspace&)` in
// fd_internal.h, call it first in launch_persist (rsolve.cu), and add the padded
// factor table `fe` / `fep` to PlanDev + plan.cpp (see git history, commit
// "Split rectangle solve (opt-in, FD_SPLIT=1)").
//
// Measured on one B200 (c1: 5 x 1023^2, 8 rotating buffer sets; the shipped fused
// kernel rsolve.cu: 89-90 us per apply):
//   K_A row-pair DST (HBM -> Z)            33-35 us   (29 us under ncu, cold L2)
//   K_C row-pair DST (Z -> out)            29-31 us
//   K_B mode-sliced Thomas, TMA ring       48 us      (24 us for slices on the fixed
//       point, 48 us for the four slices per job that stream the long-transient table)
//   K_B blocks-in-one-CTA form             50-93 us
//   whole apply                            105-115 us -- slower than the fused kernel.
// Why (ncu + clock stamps + tools/micro):
//  * K_A / K_C run the same RFft passes as rsolve.cu with the same 16 warps per SM
//    (128 registers): 1562 warp instructions per row pair and warp at IPC 1.2 per SM,
//    warp-cycles per issued instruction 11.4 -- latency-bound at 25 % occupancy.
//    Independent small CTAs did not overlap better than the lockstep kernel; bulk-copy
//    (TMA) input instead of global loads changed nothing (33.9 vs 33.9 us).
//  * A lone in-order warp walking the Thomas chain can reach 9.2-11.3 cycles per row
//    (tools/micro/chain.cu, chain2.cu: DFMA latency 8.2 cycles) only with straight-line
//    code; every dependent test / branch between two links costs 4-10 cycles, a
//    per-row cp.async.bulk costs ~64 cycles of the issuing warp (tools/micro/gather.cu,
//    lat.cu), mbarrier.try_wait ~150 cycles.  The kernel below reaches 16-18
//    cycles per row (1050 cycles per 64-row tile) after those were removed.
//  * Splitting the rows of a mode slice over the warps of one CTA (second kernel)
//    needs the slice on chip between the sweeps: 32 modes x 1023 rows x 8 B = 262 KB
//    exceeds the register file (256 KB), so half of every block lives in shared
//    memory, the CTA count (160) needs two rounds on 148 SMs, and the blocks holding
//    table rows (the first 128 rows, strided 256-byte reads of dl/dib/db) run 3-6x
//    longer than the others, which wait at the carry barrier.
//  * Both extra trips of the field through the L2 are not free: the 2 x 42 MB
//    scratch traffic of K_B alone is ~10 us at the L2 rates reached here.
// Split rectangle solve for FFT lengths whose fields fit the L2 (n + 1 = N = 2^NL):
// three launches instead of one cooperative kernel,
//
//   K_A  dst_pair_kernel   one CTA per row pair: rows from HBM -> real-symmetric
//                          DST-I (rsolve_common.cuh, RFft) -> yhat rows in a scratch
//                          field Z of row pitch N doubles (stays in L2)
//   K_B  thomas_kernel     one CTA per slice of W modes: the reference's Thomas
//                          recurrences (rectsolver.py:80-91) over ALL rows of the
//                          slice, lane = mode, 16-row tiles of Z streamed through
//                          shared memory by TMA tensor copies ahead of the
//                          dependent chain, in place
//   K_C  dst_pair_kernel   one CTA per row pair: xhat rows (Z) -> DST-I ->
//                          out = alpha x + beta other
//
// Why: the fused kernel (rsolve.cu) partitions the sweep over row blocks, which
// ties every CTA to "load -> transform -> sweep" in lockstep plus two grid
// barriers and a carry phase.  Partitioning the sweep over MODES instead needs no
// carries at all (each lane runs the reference recurrence top to bottom and back),
// leaves the transforms as independent small CTAs that overlap each other's
// loads, exchanges and stores, and costs one extra trip of the field through the
// L2 -- which is free while 2 x 8 B/pt of the batch fit the 126 MB L2.
#include <cuda.h>

#include <set>
#include <type_traits>
#include <tuple>

#include "rsolve_common.cuh"

namespace fd {

// ---------------------------------------------------------------------------
// K_A / K_C: row-pair transforms
struct XJob {
    const double *src;
    double *dst;
    const double *other;
    double alpha, beta;
    double h2;        // 0.5 * scale
    int m, pairs;
    int spitch, dpitch;   // row pitch of src / dst in doubles (other: n)
    int tma;              // src row pairs are 16-byte aligned multiples of 16 bytes: bulk copies
};
struct XList {
    int count, n;
    const double *ralpha;   // [N] pre-weights
    const double2 *m16;     // [16] e^{-2 pi i q / 256}  (N >= 512), then la[NB] e^{-2 pi i q / N}
    XJob job[kMaxPJobs];
};

template <int NL, bool STREAM>
__global__ void __launch_bounds__(RS<NL>::T, (512 / RS<NL>::T) > 8 ? 8 : (512 / RS<NL>::T))
    dst_pair_kernel(const __grid_constant__ XList xl) {
    using C = RS<NL>;
    using F = RFft<NL>;
    constexpr int T = C::T, XR = C::XR;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *buf = reinterpret_cast<double2 *>(smem_raw);
    double *scr = reinterpret_cast<double *>(smem_raw + C::REG);
    const int t = threadIdx.x, lane = t & 31;
    const int n = xl.n;
    int pid = blockIdx.x, j = 0;
    while (pid >= xl.job[j].pairs) {
        pid -= xl.job[j].pairs;
        ++j;
    }
    const XJob &J = xl.job[j];
    const int r0 = 2 * pid;
    const bool hb = r0 + 1 < J.m;
    const double *A = J.src + size_t(r0) * J.spitch;
    double2 v[16];
    if (J.tma && hb) {
        // the row pair arrives by one bulk copy (TMA) in the exchange region itself
        // and is pre-weighted out of shared memory: one memory round trip per
        // CTA instead of one per batch of loads the registers allow
        __shared__ __align__(8) uint64_t bar;
        if (t == 0) {
            mbar_init(&bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_expect_tx(&bar, uint32_t(2 * J.spitch * 8));
            tma_load_1d(buf, A, uint32_t(2 * J.spitch * 8), &bar);
        }
        __syncthreads();
        mbar_wait(&bar, 0);
        const double *SA = reinterpret_cast<const double *>(buf);
        F::load(v, SA, SA + J.spitch, xl.ralpha, J.h2, t);
        rsync<T>(0);   // the staged rows alias the exchange buffer
    } else {
        // pre-weighted input of the first pass (RFft::load) straight from global
        // memory; STREAM: the user's right-hand side is read once -- evict-first,
        // so that it does not push the scratch field Z out of the L2
        const double *B = hb ? A + J.spitch : A;
        constexpr int N = C::N;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int jj = t + r * T;
            if (r == 0 && t == 0) {
                v[0] = make_double2(0.0, 0.0);
                continue;
            }
            const double a = __ldg(xl.ralpha + jj), bq = a - J.h2;
            const int i1 = jj - 1, i2 = N - 1 - jj;
            if (STREAM) {
                v[r].x = fma(a, __ldcs(A + i1), bq * __ldcs(A + i2));
                v[r].y = fma(a, __ldcs(B + i1), bq * __ldcs(B + i2));
            } else {
                v[r].x = fma(a, __ldcg(A + i1), bq * __ldcg(A + i2));
                v[r].y = fma(a, __ldcg(B + i1), bq * __ldcg(B + i2));
            }
        }
    }
    F::first(buf, v, t, 0);
    if constexpr (C::NMID > 0) F::mid(buf, xl.m16, t, 0);
    F::last(buf, xl.m16 + 16, t, 0);
    double *XA = reinterpret_cast<double *>(buf);
    F::post(buf, scr, t, 0, lane, XA, hb ? XA + XR : nullptr);
    rsync<T>(0);
    const double al_ = J.alpha, be_ = J.beta;
    const int rp = hb ? 2 : 1;
    for (int h = 0; h < rp; ++h) {
        const double *Xh = XA + h * XR;
        double *oh = J.dst + size_t(r0 + h) * J.dpitch;
        const double *qh = J.other ? J.other + size_t(r0 + h) * n : nullptr;
        if (qh) {
#pragma unroll 8
            for (int q = t; q < n; q += T) __stcs(oh + q, fma(be_, __ldcs(qh + q), al_ * Xh[xi(q)]));
        } else if (al_ == 1.0) {
#pragma unroll 8
            for (int q = t; q < n; q += T) {
                if (STREAM) oh[q] = Xh[xi(q)];      // stage A writes Z: keep it in the L2
                else __stcs(oh + q, Xh[xi(q)]);
            }
        } else {
#pragma unroll 8
            for (int q = t; q < n; q += T) __stcs(oh + q, al_ * Xh[xi(q)]);
        }
    }
}

// ---------------------------------------------------------------------------
// K_B: mode-sliced Thomas sweeps
//
// CTA = slice of W modes [k0, k0 + W) of one job; consumer warp c owns modes
// k0 + 32 c + lane, the last warp's lane 0 is the producer.  Rows move in tiles
// of kSR = 64: one TMA tensor copy (box 64 x W of the pitch-N field Z; rows and
// modes out of range arrive as zeros and are clipped on the way back) per tile
// and direction.  Shared memory: a ring of NG data tiles and kFG factor tiles
// for the tiles whose factors come from tables: rows < ecap (PlanDev::fe, every
// mode) and, for slices holding slowly converging modes k < kt, every later row
// (PlanDev::lt).  All other rows use the per-mode fixed point.
//
// Forward (rectsolver.py:86):  y_i = r_i - l_i y_{i-1}                tiles 0 .. T-1
// Backward (rectsolver.py:90): x_i = (y_i - off x_{i+1}) / beta_i     tiles T-1 .. 0
// The last NG tiles of y stay in their slots for the backward pass; earlier
// tiles go back to Z (L2) and are copied in again as the backward pass frees
// slots.  Every global access of the field is a tensor copy issued by the
// producer (async proxy, ordered by the bulk groups).
//
// The consumers' chains are latency-bound (8 cycles per dependent DFMA), so
// nothing with a long latency may sit between two 16-row chunks: the chunk's
// values are loaded one chunk ahead, and instead of waiting on mbarriers (a
// phase query takes ~150 cycles and blocks the in-order warp) the consumers read
// plain shared-memory counters that the producer bumps as copies land; the
// counter is read one tile ahead of its use.  Consumers -> producer stays an
// mbarrier arrive (fire and forget) per 64-row tile.
constexpr int kSR = 64;                 // rows per tile (one tensor copy)
constexpr int kCH = 16;                 // rows per register chunk
constexpr int kFG = 2;                  // factor ring depth (tiles)
constexpr int kMaxW = 64;               // modes per slice (two consumer warps)
constexpr int kThomasThreads = 96;

struct TJob {
    alignas(64) CUtensorMap zmap;    // Z: {n, m}, pitch N doubles, box {W, 64}
    alignas(64) CUtensorMap femap;   // fe: {fep, 2 ecap}, box {W, 64}
    alignas(64) CUtensorMap ltmap;   // lt: {3 ktp, m}, box {W, 64} (valid when kt > 0)
    const double *mode;
    double off;
    int m, n, ecap, kt, ktp;
    int cta0;         // CTAs [cta0, next job's cta0) take slices of W modes
};
struct TList {
    int count;
    int NG;           // data tiles in shared memory
    int W;            // modes per slice
    long long *dbg;   // optional [grid][16] cycle counters (FD_SPLIT_TIMING)
    int dbgmask;      // timing experiments (FD_SPLIT_DBG)
    TJob job[kMaxPJobs];
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t mbar_test(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done;
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, int c0, int c1, const void *src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(c0),
                 "r"(c1), "r"(smem_u32(src))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}

template <int W>
__global__ void __launch_bounds__(kThomasThreads, 1) thomas_kernel(const __grid_constant__ TList tl) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int j = 0;
    while (j + 1 < tl.count && int(blockIdx.x) >= tl.job[j + 1].cta0) ++j;
    const TJob &J = tl.job[j];
    const int n = J.n, m = J.m;
    const int k0 = (int(blockIdx.x) - J.cta0) * W;
    const int w = min(W, n - k0);
    const int NG = tl.NG;
    const int T = (m + kSR - 1) / kSR;
    const int ecap = J.ecap;
    const bool slow = k0 < J.kt;                                  // slice holds table modes
    auto fact = [&](int t) { return t * kSR < ecap || slow; };   // tile's factors come from tables
    constexpr uint32_t tile_bytes = uint32_t(kSR) * W * 8;
    constexpr int TILE = kSR * W;                                 // doubles per tile

    double *slots = reinterpret_cast<double *>(smem_raw);                 // [NG][64][W]
    double *fslots = slots + size_t(NG) * TILE;                            // [kFG][64][W]
    uint64_t *full = reinterpret_cast<uint64_t *>(fslots + size_t(kFG) * TILE);   // [NG]
    uint64_t *done_f = full + NG;                                          // [NG] forward pass
    uint64_t *done_b = done_f + NG;                                        // [NG] backward pass
    uint64_t *ffull = done_b + NG;                                         // [kFG]
    uint32_t *landed = reinterpret_cast<uint32_t *>(ffull + kFG);          // data / factor copies landed so far
    constexpr int NCW = kThomasThreads / 32 - 1;
    if (tid == 0) {
        for (int g = 0; g < NG; ++g) {
            mbar_init(&full[g], 1);
            mbar_init(&done_f[g], NCW);
            mbar_init(&done_b[g], NCW);
        }
        for (int g = 0; g < kFG; ++g) mbar_init(&ffull[g], 1);
        landed[0] = landed[1] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int TS = max(0, T - NG);   // tiles below TS stream through Z, the rest stay in their slots

    if (warp == NCW) {
        // ------------------------------ producer ------------------------------
        if (lane != 0) return;
        // copies are issued in the order the consumers need them; sequence
        // numbers (data: di, factors: fi) index the landed counters
        uint32_t di = 0, fi = 0;         // issued
        uint32_t dl = 0, fl = 0;         // landed and published
        uint64_t fullpar = 0;            // parity of full[g]
        uint32_t ffpar = 0;              // parity of ffull[fg]
        constexpr int QN = 16;
        int dq[QN], fq[QN];              // slots of the issued, not yet landed copies (FIFO)
        auto publish = [&]() {   // copies that have landed, in issue order
            while (dl < di) {
                const int g = dq[dl % QN];
                if (!mbar_test(&full[g], uint32_t(fullpar >> g) & 1u)) break;
                fullpar ^= uint64_t(1) << g;
                st_release(&landed[0], ++dl);
            }
            while (fl < fi) {
                const int fg = fq[fl % QN];
                if (!mbar_test(&ffull[fg], (ffpar >> fg) & 1u)) break;
                ffpar ^= 1u << fg;
                st_release(&landed[1], ++fl);
            }
        };
        auto issue_data = [&](int t) {
            while (int(di - dl) >= QN) publish();
            const int g = t % NG;
            mbar_expect_tx(&full[g], tile_bytes);
            tma_load_2d(slots + size_t(g) * TILE, &J.zmap, k0, t * kSR, &full[g]);
            dq[di % QN] = g;
            ++di;
        };
        auto issue_fact = [&](int t, bool backward) {
            while (int(fi - fl) >= QN) publish();
            const int fg = t % kFG;
            mbar_expect_tx(&ffull[fg], tile_bytes);
            double *dst = fslots + size_t(fg) * TILE;
            if (t * kSR < ecap) tma_load_2d(dst, &J.femap, k0, (backward ? ecap : 0) + t * kSR, &ffull[fg]);
            else tma_load_2d(dst, &J.ltmap, (backward ? J.ktp : 0) + k0, t * kSR, &ffull[fg]);
            fq[fi % QN] = fg;
            ++fi;
        };
        const long long p_start = clock64();
        for (int t = 0; t < min(NG, T); ++t) {
            issue_data(t);
            if (t < kFG && fact(t)) issue_fact(t, false);
        }
        uint64_t dpar = 0;   // parity of done_f[g]
        for (int c = 0, g = 0; c < T; ++c, g = (g + 1 == NG ? 0 : g + 1)) {   // forward
            while (!mbar_test(&done_f[g], uint32_t(dpar >> g) & 1u)) {
                publish();
                if (tl.dbgmask & 1) __nanosleep(200);
            }
            dpar ^= uint64_t(1) << g;
            if (c < TS) {
                tma_store_2d(&J.zmap, k0, c * kSR, slots + size_t(g) * TILE);   // y of a streamed tile
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                issue_data(c + NG);
            }
            if (c + kFG < T && fact(c + kFG)) issue_fact(c + kFG, false);
            publish();
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // streamed y visible before it is copied in again
        const long long p_mid = clock64();
        for (int t = T - 1; t >= max(T - kFG, 0); --t)
            if (fact(t)) issue_fact(t, true);
        dpar = 0;            // parity of done_b[g]
        for (int c = T - 1, g = (T - 1) % NG; c >= 0; --c, g = (g == 0 ? NG - 1 : g - 1)) {   // backward
            while (!mbar_test(&done_b[g], uint32_t(dpar >> g) & 1u)) {
                publish();
                if (tl.dbgmask & 1) __nanosleep(200);
            }
            dpar ^= uint64_t(1) << g;
            tma_store_2d(&J.zmap, k0, c * kSR, slots + size_t(g) * TILE);       // xhat
            if (c - NG >= 0) {
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                issue_data(c - NG);
            }
            if (c - kFG >= 0 && fact(c - kFG)) issue_fact(c - kFG, true);
            publish();
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        if (tl.dbg) {
            long long *d = tl.dbg + size_t(blockIdx.x) * 16;
            d[8] = p_mid - p_start;
            d[9] = clock64() - p_mid;
        }
        return;
    }

    // ------------------------------ consumers ------------------------------
    const int q = 32 * warp + lane;        // mode within the slice
    const bool inb = q < W;                // lane owns a column of the tile
    const bool act = q < w;
    const int qq = inb ? q : 0;
    const int k = k0 + (act ? q : 0);
    const bool tabm = act && k < J.kt;     // this lane's factors beyond ecap come from lt
    double l_inf = 0.0, ib_inf = 0.0, ib_last = 0.0;
    {
        const double2 *rec = reinterpret_cast<const double2 *>(J.mode) + 4 * k;
        const double2 a = __ldg(rec), c = __ldg(rec + 2);
        if (act) {
            l_inf = a.x;
            ib_inf = a.y;
            ib_last = 1.0 / c.x;
        }
    }
    const double noff = -J.off;
    const double nl_inf = -l_inf, g_inf = noff * ib_inf;
    uint32_t dneed = 0, fneed = 0;   // copies that must have landed before the next tile of each kind
    uint32_t dseen = 0, fseen = 0;   // last counter values read
    double carry = 0.0;              // y_{i-1} forward, x_{i+1} backward
    long long cwait = 0;

    auto run_pass = [&](auto bwd_tag) {
        constexpr bool BWD = decltype(bwd_tag)::value;
        constexpr int dir = BWD ? -1 : 1;
        constexpr int NC = kSR / kCH;   // chunks per tile
        uint64_t *done = BWD ? done_b : done_f;
        auto need = [&](int t) { return !BWD || t < TS; };            // tile is copied in during this pass
        auto wrap = [&](int g) { return BWD ? (g == 0 ? NG - 1 : g - 1) : (g + 1 == NG ? 0 : g + 1); };
        // make sure tile t's copies have landed (the counters were read a tile ago)
        auto acquire = [&](int t) {
            if (need(t)) {
                ++dneed;
                if (dseen < dneed) {
                    const long long c0 = clock64();
                    while ((dseen = ld_acquire(&landed[0])) < dneed) {}
                    cwait += clock64() - c0;
                }
            }
            if (fact(t)) {
                ++fneed;
                if (fseen < fneed) {
                    const long long c0 = clock64();
                    while ((fseen = ld_acquire(&landed[1])) < fneed) {}
                    cwait += clock64() - c0;
                }
            }
        };
        double da[kCH], db[kCH];   // data of the current / next chunk
        // One tile.  KIND 0: fixed-point factors; 1: factors from the table tile
        // (per lane: table or fixed point); 2: the pass's first backward tile
        // (holds row m-1 and the rows past it).  Straight-line code: the chunk
        // loop is unrolled with compile-time indices and has no tile-uniform
        // tests inside (a lone in-order warp pays ~4-10 cycles for every
        // dependent test and branch between two links of the chain).
        auto tile = [&](auto kind_tag, int t, int g, int tn, int gn, bool more) {
            constexpr int KIND = decltype(kind_tag)::value;
            double *sl = slots + size_t(g) * TILE + qq;
            const double *sn = slots + size_t(gn) * TILE + qq;
            const double *fs = fslots + size_t(t % kFG) * TILE + qq;
            const bool tab = t * kSR < ecap || tabm;
            const bool isf = fact(t);
            // counters for the next tile: read now, compared at this tile's last chunk
            dseen = ld_acquire(&landed[0]);
            fseen = ld_acquire(&landed[1]);
#pragma unroll
            for (int ci = 0; ci < NC; ++ci) {
                const int c = BWD ? NC - 1 - ci : ci;
                auto body = [&](double (&dc)[kCH], double (&dn)[kCH]) {
                    double fv[kCH];
                    if (KIND != 0) {
                        const int i0 = t * kSR + c * kCH;
#pragma unroll
                        for (int r = 0; r < kCH; ++r) {
                            const double cst = BWD ? ((KIND == 2 && i0 + r == m - 1) ? ib_last : ib_inf) : l_inf;
                            fv[r] = (isf && tab) ? fs[(c * kCH + r) * W] : cst;
                            if (KIND == 2 && i0 + r >= m) dc[r] = 0.0;   // the forward pass ran on past row m-1
                        }
                    }
                    if (ci + 1 < NC) {
#pragma unroll
                        for (int r = 0; r < kCH; ++r) dn[r] = sl[((c + dir) * kCH + r) * W];
                    } else {
                        if (more) acquire(tn);
#pragma unroll
                        for (int r = 0; r < kCH; ++r) dn[r] = sn[((BWD ? NC - 1 : 0) * kCH + r) * W];
                    }
                    double *so = sl + c * kCH * W;
                    if (!BWD) {
#pragma unroll
                        for (int r = 0; r < kCH; ++r) {
                            carry = fma(KIND != 0 ? -fv[r] : nl_inf, carry, dc[r]);
                            if (inb) so[r * W] = carry;
                        }
                    } else {
                        double a[kCH], gg[kCH];
#pragma unroll
                        for (int r = 0; r < kCH; ++r) {
                            a[r] = dc[r] * (KIND != 0 ? fv[r] : ib_inf);
                            gg[r] = KIND != 0 ? noff * fv[r] : g_inf;
                        }
#pragma unroll
                        for (int r = kCH - 1; r >= 0; --r) {
                            carry = fma(gg[r], carry, a[r]);
                            if (inb) so[r * W] = carry;
                        }
                    }
                };
                if (ci & 1) body(db, da);
                else body(da, db);
            }
            // the producer's tensor store reads the slot (streamed y, every xhat tile)
            if (BWD || t < TS) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&done[g]);
        };
        int t = BWD ? T - 1 : 0, g = t % NG;
        acquire(t);
        {
            const double *sl = slots + size_t(g) * TILE + qq;
#pragma unroll
            for (int r = 0; r < kCH; ++r) da[r] = sl[((BWD ? NC - 1 : 0) * kCH + r) * W];
        }
        for (int it = 0; it < T; ++it) {
            const int tn = t + dir, gn = wrap(g);
            const bool more = it + 1 < T;
            if (BWD && it == 0) tile(std::integral_constant<int, 2>{}, t, g, tn, gn, more);
            else if (fact(t)) tile(std::integral_constant<int, 1>{}, t, g, tn, gn, more);
            else tile(std::integral_constant<int, 0>{}, t, g, tn, gn, more);
            if (tl.dbg && tid == 0 && it < 20) tl.dbg[size_t(gridDim.x) * 16 + size_t(blockIdx.x) * 64 + (BWD ? 32 : 0) + it] = clock64();
            t = tn;
            g = gn;
        }
    };
    {
        const long long c_start = clock64();
        run_pass(std::false_type{});
        __syncwarp();
        const long long c_mid = clock64();
        const long long w_f = cwait;
        carry = 0.0;
        run_pass(std::true_type{});
        if (tl.dbg && tid == 0) {
            long long *d = tl.dbg + size_t(blockIdx.x) * 16;
            d[0] = c_mid - c_start;
            d[1] = clock64() - c_mid;
            d[2] = w_f;
            d[3] = cwait - w_f;
        }
    }
}

// ---------------------------------------------------------------------------
// K_B, second form: mode-sliced Thomas sweeps with the rows of a slice split
// over the warps of ONE CTA (block carries exchanged through shared memory).
//
// CTA = 32 modes (lane = mode) x kNB = 16 row blocks (warp = block) of kRPB = 64
// rows; a thread keeps its block of one mode on chip from the forward to the
// backward sweep: the first kRR = 32 rows in registers, the other 32 in a
// private shared-memory column.  The sweeps are those of rsolve.cu (the
// reference recurrences rectsolver.py:86,90 inside a block, affine block carries
// across blocks), but every block of a mode lives in the same CTA, so the carry
// exchange is a __syncthreads and a 16-step scan instead of two grid barriers:
//
//   forward, block [s, e], local (y_{s-1} = 0):
//     y_i = r_i - l_i y_{i-1},  w_i = prod_{j=s..i} (-l_j)      (Y_i = y_i + w_i Y_in)
//     t_i = G_i / beta_i, G_s = 1, G_{i+1} = G_i g_i, g_i = -off / beta_i
//     F0 = sum t_i y_i,  xi = sum t_i w_i,  Q = G_{e+1}         (x_s = F0 + xi Y_in + Q X_out)
//   scan over blocks: Y_in(b+1) = y_e(b) + w_e(b) Y_in(b);  X_out(b-1) = x_s(b)
//   backward: Y_i = y_i + w_i Y_in (w walked back with 1/(-l_i)),  x_i = (Y_i - off x_{i+1}) / beta_i
//
// fp64 work: 5 + 4 instructions per row and mode, 4 warps per scheduler: the
// kernel is bound by fp64 issue, not by the latency of one chain.
constexpr int kRPB = 64;    // rows per thread
constexpr int kRR = 32;     // ... of which in registers
constexpr int kNB = 16;     // row blocks (warps) per CTA
constexpr int kBThreads = 32 * kNB;
constexpr size_t kBSmem = size_t(kNB) * (kRPB - kRR) * 32 * 8 + size_t(kNB) * 5 * 32 * 8;

struct BJob {
    PlanDev p;
    double *z;        // field (row pitch `pitch` doubles), swept in place
    int pitch;
    int cta0;         // CTAs [cta0, next job's cta0) take slices of 32 modes
};
struct BList {
    int count;
    long long *dbg;   // optional [grid][kNB][4] cycle stamps (FD_SPLIT_TIMING)
    BJob job[kMaxPJobs];
};

__global__ void __launch_bounds__(kBThreads, 1) thomas_blocks_kernel(const __grid_constant__ BList bl) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *ycol = reinterpret_cast<double *>(smem_raw);                       // [kNB][kRPB - kRR][32]
    double *scal = ycol + size_t(kNB) * (kRPB - kRR) * 32;                     // [kNB][5][32]
    const int tid = threadIdx.x, lane = tid & 31, b = tid >> 5;
    int j = 0;
    while (j + 1 < bl.count && int(blockIdx.x) >= bl.job[j + 1].cta0) ++j;
    const BJob &J = bl.job[j];
    const PlanDev &p = J.p;
    const int n = p.n, m = p.m, NP = J.pitch;
    const int k0 = (int(blockIdx.x) - J.cta0) * 32;
    const bool act = k0 + lane < n;
    const int k = act ? k0 + lane : n - 1;
    // The blocks cover rows [0, m-1); the last row (its 1/beta carries the end
    // modifier) is one more link of the carry scan.
    const int mb = m - 1;
    const int s = b * kRPB;
    const int nr = max(0, min(kRPB, mb - s));     // rows of this block (warp-uniform)
    const int nb = (mb + kRPB - 1) / kRPB;        // blocks of the job (<= kNB)
    double *Zj = J.z + k;
    double *Z = Zj + size_t(s) * NP;
    double *ys = ycol + (size_t(b) * (kRPB - kRR)) * 32 + lane;

    const long long c_t0 = clock64();
    ModeRec mr;
    mr.load(p, k);
    const double l_inf = mr.l_inf, ib_inf = mr.ib_inf, inv_nl = mr.inv_nl;
    const double noff = -p.off, nio = p.nio;
    const double g_inf = noff * ib_inf, nl_inf = -l_inf;
    // Factors l_i, 1/beta_i, 1/(-l_i) = -beta_{i-1}/off of a row:
    //   i < ecap: the row-major tables dl, dib, db (they hold every mode, the
    //             fixed point filled in past a mode's transient);
    //   i >= ecap: the mode's fixed point, except for the slowly converging
    //             modes k < kt, which read the long-transient table lt.
    const bool slowm = p.lt != nullptr && k < p.kt;
    const double *ltk = p.lt + k;
    const size_t lts = size_t(3) * p.ktp;
    // block kind (warp-uniform): 0 fixed point, 1 tables (block below ecap), 2 mixed
    const int ecap = p.ecap;
    const bool any_slow = __any_sync(0xffffffffu, slowm);
    const int kind = (s + nr <= ecap) ? 1 : ((s >= ecap && !any_slow) ? 0 : 2);

    auto fac_fwd = [&](int i, double &l, double &ib) {   // kinds 1, 2
        if (i < ecap) {
            l = __ldg(p.dl + size_t(i) * n + k);
            ib = __ldg(p.dib + size_t(i) * n + k);
        } else if (slowm) {
            l = __ldg(ltk + size_t(i) * lts);
            ib = __ldg(ltk + size_t(i) * lts + p.ktp);
        } else {
            l = l_inf;
            ib = ib_inf;
        }
    };
    auto fac_bwd = [&](int i, double &ib, double &pm) {  // kinds 1, 2
        if (i < ecap) {
            ib = __ldg(p.dib + size_t(i) * n + k);
            pm = (i >= 1) ? __ldg(p.db + size_t(i - 1) * n + k) * nio : 0.0;
        } else if (slowm) {
            ib = __ldg(ltk + size_t(i) * lts + p.ktp);
            pm = __ldg(ltk + size_t(i) * lts + 2 * p.ktp);
        } else {
            ib = ib_inf;
            pm = (i == ecap) ? __ldg(p.db + size_t(i - 1) * n + k) * nio : inv_nl;
        }
    };

    // ---- the register rows; the other rows stream in during the forward sweep
    double d[kRR];
#pragma unroll
    for (int r = 0; r < kRR; ++r) d[r] = (r < nr) ? __ldcg(Z + size_t(r) * NP) : 0.0;

    // ---- forward sweep, 8 rows at a time (loads first, then the chains)
    double y = 0.0, w = 1.0, t = nio, F0 = 0.0, xi = 0.0;
    // full batch, fixed-point factors
    auto fwd8c = [&](double (&v)[8]) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            y = fma(nl_inf, y, v[r]);
            w *= nl_inf;
            t *= g_inf;
            F0 = fma(y, t, F0);
            xi = fma(w, t, xi);
            v[r] = y;
        }
    };
    // batch of cnt <= 8 rows starting at block row r0, factors per row
    auto fwd8g = [&](int r0, int cnt, double (&v)[8]) {
        double lv[8], gv[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            lv[r] = 0.0;
            gv[r] = 0.0;
            if (r < cnt) fac_fwd(s + r0 + r, lv[r], gv[r]);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            if (r < cnt) {
                y = fma(-lv[r], y, v[r]);
                w *= -lv[r];
                t *= noff * gv[r];
                F0 = fma(y, t, F0);
                xi = fma(w, t, xi);
                v[r] = y;
            }
        }
    };
#pragma unroll
    for (int q = 0; q < kRR / 8; ++q) {
        double v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = d[q * 8 + r];
        if (kind == 0 && nr >= kRR) fwd8c(v);
        else fwd8g(q * 8, min(8, nr - q * 8), v);
#pragma unroll
        for (int r = 0; r < 8; ++r) d[q * 8 + r] = v[r];
    }
#pragma unroll 1
    for (int r0 = kRR; r0 < nr; r0 += 8) {
        const int cnt = min(8, nr - r0);
        double v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = (r < cnt) ? __ldcg(Z + size_t(r0 + r) * NP) : 0.0;
        if (kind == 0 && cnt == 8) fwd8c(v);
        else fwd8g(r0, cnt, v);
#pragma unroll
        for (int r = 0; r < 8; ++r) ys[(r0 - kRR + r) * 32] = v[r];
    }
    // block scalars: y_e, w_e, F0, xi, Q
    {
        double *sc = scal + size_t(b) * 5 * 32 + lane;
        sc[0] = y;
        sc[32] = w;
        sc[64] = F0;
        sc[96] = xi;
        sc[128] = t * noff;
    }
    const long long c_t1 = clock64();
    __syncthreads();

    // ---- block carries: warp 0 scans the chains of the 32 modes (nb <= 16 steps
    // each way, row m-1 in between) and leaves Y_in, X_out of every block in the
    // scalar slots 0, 1
    if (b == 0) {
        double Y = 0.0;
#pragma unroll 1
        for (int q = 0; q < nb; ++q) {
            double *sc = scal + size_t(q) * 5 * 32 + lane;
            const double ye = sc[0], pe = sc[32];
            sc[0] = Y;   // Y_in of block q
            Y = fma(pe, Y, ye);
        }
        // last row: y = r - l y_{m-2}, x = y / beta_{m-1}
        double ll = l_inf;
        if (mb < ecap) ll = __ldg(p.dl + size_t(mb) * n + k);
        else if (slowm) ll = __ldg(ltk + size_t(mb) * lts);
        if (mb == 0) ll = 0.0;
        const double yl = fma(-ll, Y, __ldcg(Zj + size_t(mb) * NP));
        double X = yl * (1.0 / mr.b_last);
        if (act) __stcg(Zj + size_t(mb) * NP, X);
#pragma unroll 1
        for (int q = nb - 1; q >= 0; --q) {
            double *sc = scal + size_t(q) * 5 * 32 + lane;
            const double xs = fma(sc[128], X, fma(sc[96], sc[0], sc[64]));
            sc[32] = X;  // X_out of block q
            X = xs;
        }
    }
    __syncthreads();
    const double Yin = scal[size_t(b) * 5 * 32 + lane], Xout = scal[size_t(b) * 5 * 32 + 32 + lane];
    const long long c_t2 = clock64();

    // ---- backward sweep: true y, then x, rows descending; results straight to Z
    double x = Xout, Pc = w;
    auto bwd8c = [&](double (&v)[8]) {
#pragma unroll
        for (int r = 7; r >= 0; --r) {
            const double Y = fma(Pc, Yin, v[r]);
            Pc *= inv_nl;
            x = fma(g_inf, x, Y * ib_inf);
            v[r] = x;
        }
    };
    auto bwd8g = [&](int r0, int cnt, double (&v)[8]) {
        double gv[8], pv[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            gv[r] = 0.0;
            pv[r] = 0.0;
            if (r < cnt) fac_bwd(s + r0 + r, gv[r], pv[r]);
        }
#pragma unroll
        for (int r = 7; r >= 0; --r) {
            if (r < cnt) {
                const double Y = fma(Pc, Yin, v[r]);
                Pc *= pv[r];
                x = fma(noff * gv[r], x, Y * gv[r]);
                v[r] = x;
            }
        }
    };
#pragma unroll 1
    for (int r0 = ((nr - 1) & ~7); r0 >= kRR; r0 -= 8) {
        const int cnt = min(8, nr - r0);
        double v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = ys[(r0 - kRR + r) * 32];
        if (kind == 0 && cnt == 8) bwd8c(v);
        else bwd8g(r0, cnt, v);
#pragma unroll
        for (int r = 0; r < 8; ++r)
            if (act && r < cnt) __stcg(Z + size_t(r0 + r) * NP, v[r]);
    }
#pragma unroll
    for (int q = kRR / 8 - 1; q >= 0; --q) {
        double v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = d[q * 8 + r];
        if (kind == 0 && nr >= kRR) bwd8c(v);
        else bwd8g(q * 8, min(8, nr - q * 8), v);
#pragma unroll
        for (int r = 0; r < 8; ++r)
            if (act && q * 8 + r < nr) __stcg(Z + size_t(q * 8 + r) * NP, v[r]);
    }
    if (bl.dbg && lane == 0) {
        long long *dd = bl.dbg + (size_t(blockIdx.x) * kNB + b) * 4;
        dd[0] = c_t1 - c_t0;
        dd[1] = c_t2 - c_t1;
        dd[2] = clock64() - c_t2;
        dd[3] = kind;
    }
}

// ---------------------------------------------------------------------------
// host side
namespace {
struct TwKey {
    int device, N;
    bool operator<(const TwKey &o) const { return device < o.device || (device == o.device && N < o.N); }
};
std::mutex g_split_mu;
std::map<TwKey, double2 *> g_split_tw;

template <int NL>
const double2 *pair_twiddles(int device) {
    using C = RS<NL>;
    std::lock_guard<std::mutex> g(g_split_mu);
    auto it = g_split_tw.find({device, C::N});
    if (it != g_split_tw.end()) return it->second;
    const long double PI = 3.141592653589793238462643383279502884L;
    std::vector<double2> h(16 + C::NB);
    for (int q = 0; q < 16; ++q) {
        const long double a = 2.0L * PI * (long double)q / 256.0L;
        h[q] = make_double2((double)cosl(a), (double)(-sinl(a)));
    }
    for (int q = 0; q < C::NB; ++q) {
        const long double a = 2.0L * PI * (long double)q / (long double)C::N;
        h[16 + q] = make_double2((double)cosl(a), (double)(-sinl(a)));
    }
    double2 *d = nullptr;
    FD_CUDA(cudaMalloc(&d, sizeof(double2) * h.size()));
    FD_CUDA(cudaMemcpy(d, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice));
    g_split_tw[{device, C::N}] = d;
    return d;
}

struct DevInfo {
    int sms = 0, smem = 0;
};
DevInfo dev_info(int device) {
    static std::mutex mu;
    static std::map<int, DevInfo> cache;
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(device);
    if (it != cache.end()) return it->second;
    DevInfo d;
    FD_CUDA(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, device));
    FD_CUDA(cudaDeviceGetAttribute(&d.smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    cache[device] = d;
    return d;
}

// 2-D fp64 tensor map {cols, rows} with a row pitch in doubles and a {W, 16} box
using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
    static EncodeFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeFn>(p);
    }();
    if (!fn) FD_FAIL(FD_ERR_CUDA, "cuTensorMapEncodeTiled not available");
    return fn;
}
struct MapKey {
    const void *base;
    long long cols, rows, pitch;
    int W;
    bool operator<(const MapKey &o) const {
        return std::tie(base, cols, rows, pitch, W) < std::tie(o.base, o.cols, o.rows, o.pitch, o.W);
    }
};
CUtensorMap tile_map(const void *base, long long cols, long long rows, long long pitch, int W) {
    static std::mutex mu;
    static std::map<MapKey, CUtensorMap> cache;   // a descriptor only encodes geometry: safe to reuse for equal keys
    std::lock_guard<std::mutex> g(mu);
    const MapKey key{base, cols, rows, pitch, W};
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    CUtensorMap m;
    const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(pitch) * 8};
    const cuuint32_t box[2] = {cuuint32_t(W), cuuint32_t(kSR)};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void *>(base), dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) FD_FAIL(FD_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    if (cache.size() > 256) cache.clear();
    cache[key] = m;
    return m;
}

template <int W>
void launch_thomas_w(int ctas, size_t smem, cudaStream_t s, const TList &tl, int smem_max) {
    static std::mutex mu;
    static std::set<int> done;
    int dev = 0;
    FD_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> g(mu);
        if (done.insert(dev).second)
            FD_CUDA(cudaFuncSetAttribute((const void *)thomas_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem_max));
    }
    thomas_kernel<W><<<ctas, kThomasThreads, smem, s>>>(tl);
}
void launch_thomas(int W, int ctas, size_t smem, cudaStream_t s, const TList &tl, int smem_max) {
    switch (W) {
#define FD_TW(V) case V: launch_thomas_w<V>(ctas, smem, s, tl, smem_max); break;
        FD_TW(16) FD_TW(20) FD_TW(24) FD_TW(28) FD_TW(32) FD_TW(36) FD_TW(40) FD_TW(44) FD_TW(48) FD_TW(52) FD_TW(56)
        FD_TW(60) FD_TW(64)
#undef FD_TW
        default: FD_FAIL(FD_ERR_UNSUPPORTED, "split solve: slice width");
    }
}

template <int NL>
void run_split(const std::vector<SolveJob> &jobs, cudaStream_t s, Workspace &ws) {
    using C = RS<NL>;
    int device = 0;
    FD_CUDA(cudaGetDevice(&device));
    const DevInfo di = dev_info(device);
    const double2 *tw = pair_twiddles<NL>(device);
    const size_t xsmem = C::REG + 16 * 8;
    static const bool timing = getenv("FD_SPLIT_TIMING") != nullptr;
    const int n = jobs[0].p.n;
    static const int padq = getenv("FD_SPLIT_PAD") ? atoi(getenv("FD_SPLIT_PAD")) : 16;
    const int NP = C::N + padq;   // row pitch of Z: not a power of two (mode slices walk it row by row)
    size_t zrows = 0;
    for (size_t j0 = 0; j0 < jobs.size(); j0 += kMaxPJobs) {
        size_t r = 0;
        for (size_t j = j0; j < std::min(jobs.size(), j0 + kMaxPJobs); ++j) r += jobs[j].p.m;
        zrows = std::max(zrows, r);
    }
    double *Z = ws.get(zrows * NP);
    for (size_t j0 = 0; j0 < jobs.size(); j0 += kMaxPJobs) {
        const int cnt = (int)std::min<size_t>(kMaxPJobs, jobs.size() - j0);
        XList xa{}, xc{};
        TList tl{};
        xa.count = xc.count = tl.count = cnt;
        xa.n = xc.n = n;
        xa.ralpha = xc.ralpha = jobs[j0].p.ralpha;
        xa.m16 = xc.m16 = tw;
        // modes per slice: every job gets an equal share of the SMs
        const int share = std::max(1, di.sms / cnt);
        int W = (n + share - 1) / share;
        W = std::min(kMaxW, std::max(16, (W + 3) & ~3));   // instantiated slice widths: multiples of 4
        tl.W = W;
        int pairs = 0, ctas = 0;
        size_t zoff = 0;
        for (int j = 0; j < cnt; ++j) {
            const SolveJob &sj = jobs[j0 + j];
            const PlanDev &p = sj.p;
            double *Zj = Z + zoff;
            zoff += size_t(p.m) * NP;
            XJob &a = xa.job[j], &c = xc.job[j];
            a.src = sj.in;
            a.spitch = n;
            a.dst = Zj;
            a.dpitch = NP;
            a.other = nullptr;
            a.alpha = 1.0;
            a.beta = 0.0;
            a.h2 = 0.5 * p.scale;
            a.m = p.m;
            a.pairs = (p.m + 1) / 2;
            static const bool use_tma = !getenv("FD_SPLIT_NOTMA");
            a.tma = use_tma && (reinterpret_cast<uintptr_t>(sj.in) % 16 == 0) && (2 * size_t(n) * 8) % 16 == 0;
            c = a;
            c.tma = use_tma;   // Z rows: even pitch, aligned base
            c.src = Zj;
            c.spitch = NP;
            c.dst = sj.out;
            c.dpitch = n;
            c.other = sj.other;
            c.alpha = sj.alpha;
            c.beta = sj.beta;
            pairs += a.pairs;
            TJob &t = tl.job[j];
            t.zmap = tile_map(Zj, n, p.m, NP, W);
            t.femap = tile_map(p.fe, p.fep, 2LL * p.ecap, p.fep, W);
            if (p.kt > 0) t.ltmap = tile_map(p.lt, 3LL * p.ktp, p.m, 3LL * p.ktp, W);
            else t.ltmap = t.femap;
            t.mode = p.mode;
            t.off = p.off;
            t.m = p.m;
            t.n = n;
            t.ecap = p.ecap;
            t.kt = p.lt ? p.kt : 0;
            t.ktp = p.ktp;
            t.cta0 = ctas;
            ctas += (n + W - 1) / W;
        }
        // shared memory of K_B: factor ring + as many data tiles as fit (<= 64)
        const size_t tile = size_t(kSR) * W * 8;
        int NG = int((size_t(di.smem) - kFG * tile - 1024) / (tile + 24));
        NG = std::min(NG, 64);
        tl.NG = NG;
        const size_t tsmem = (size_t(NG) + kFG) * tile + size_t(3 * NG + kFG) * 8 + 16;
        long long *dbg = nullptr;
        if (timing) {
            FD_CUDA(cudaMallocAsync(&dbg, size_t(ctas) * 80 * 8, s));
            FD_CUDA(cudaMemsetAsync(dbg, 0, size_t(ctas) * 80 * 8, s));
        }
        tl.dbg = dbg;
        static const int dbgmask = getenv("FD_SPLIT_DBG") ? atoi(getenv("FD_SPLIT_DBG")) : 0;
        tl.dbgmask = dbgmask;
        cudaEvent_t ev[4];
        if (timing)
            for (auto &e : ev) FD_CUDA(cudaEventCreate(&e));
        if (timing) FD_CUDA(cudaEventRecord(ev[0], s));
        dst_pair_kernel<NL, true><<<pairs, C::T, xsmem, s>>>(xa);
        FD_CUDA(cudaGetLastError());
        if (timing) FD_CUDA(cudaEventRecord(ev[1], s));
        static const int bmode = getenv("FD_SPLIT") ? atoi(getenv("FD_SPLIT")) : 1;
        bool blocks_ok = bmode != 2;
        for (int j = 0; j < cnt; ++j) blocks_ok = blocks_ok && jobs[j0 + j].p.m <= kRPB * kNB;
        if (blocks_ok) {
            BList bq{};
            bq.count = cnt;
            int c0 = 0;
            size_t zo = 0;
            for (int j = 0; j < cnt; ++j) {
                const PlanDev &p = jobs[j0 + j].p;
                bq.job[j].p = p;
                bq.job[j].z = Z + zo;
                bq.job[j].pitch = NP;
                bq.job[j].cta0 = c0;
                c0 += (n + 31) / 32;
                zo += size_t(p.m) * NP;
            }
            static std::once_flag once;
            std::call_once(once, [] {
                cudaFuncSetAttribute((const void *)thomas_blocks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kBSmem);
            });
            long long *bdbg = nullptr;
            if (timing) {
                FD_CUDA(cudaMallocAsync(&bdbg, size_t(c0) * kNB * 4 * 8, s));
                FD_CUDA(cudaMemsetAsync(bdbg, 0, size_t(c0) * kNB * 4 * 8, s));
            }
            bq.dbg = bdbg;
            thomas_blocks_kernel<<<c0, kBThreads, kBSmem, s>>>(bq);
            if (timing) {
                std::vector<long long> hb(size_t(c0) * kNB * 4);
                FD_CUDA(cudaMemcpyAsync(hb.data(), bdbg, hb.size() * 8, cudaMemcpyDeviceToHost, s));
                FD_CUDA(cudaStreamSynchronize(s));
                FD_CUDA(cudaFreeAsync(bdbg, s));
                for (int c : {0, 10, c0 - 1}) {
                    fprintf(stderr, "  blocks cta %d [fwd/scan/bwd cycles, kind] per warp:", c);
                    for (int q = 0; q < kNB; ++q) {
                        const long long *e = &hb[(size_t(c) * kNB + q) * 4];
                        fprintf(stderr, " %lld/%lld/%lld,%lld", e[0], e[1], e[2], e[3]);
                    }
                    fprintf(stderr, "\n");
                }
            }
        } else {
            launch_thomas(W, ctas, tsmem, s, tl, di.smem);
        }
        FD_CUDA(cudaGetLastError());
        if (timing) FD_CUDA(cudaEventRecord(ev[2], s));
        dst_pair_kernel<NL, false><<<pairs, C::T, xsmem, s>>>(xc);
        FD_CUDA(cudaGetLastError());
        if (timing) {
            FD_CUDA(cudaEventRecord(ev[3], s));
            FD_CUDA(cudaStreamSynchronize(s));
            float a, b, c;
            cudaEventElapsedTime(&a, ev[0], ev[1]);
            cudaEventElapsedTime(&b, ev[1], ev[2]);
            cudaEventElapsedTime(&c, ev[2], ev[3]);
            fprintf(stderr, "[fd split us] A %.1f  B %.1f  C %.1f  (pairs %d, slices %d, W %d, NG %d)\n", a * 1e3,
                    b * 1e3, c * 1e3, pairs, ctas, W, NG);
            for (auto &e : ev) cudaEventDestroy(e);
            std::vector<long long> h(size_t(ctas) * 80);
            FD_CUDA(cudaMemcpy(h.data(), dbg, h.size() * 8, cudaMemcpyDeviceToHost));
            FD_CUDA(cudaFreeAsync(dbg, s));
            for (int c : {0, 5, ctas - 1}) {
                const long long *d = &h[size_t(c) * 16];
                fprintf(stderr, "  cta %d cycles: consumer fwd %lld (waiting %lld) bwd %lld (waiting %lld) | producer fwd %lld bwd %lld\n",
                        c, d[0], d[2], d[1], d[3], d[8], d[9]);
                const long long *e = &h[size_t(ctas) * 16 + size_t(c) * 64];
                fprintf(stderr, "    tile cycles fwd:");
                for (int i = 1; i < 20 && e[i]; ++i) fprintf(stderr, " %lld", e[i] - e[i - 1]);
                fprintf(stderr, "\n    tile cycles bwd:");
                for (int i = 1; i < 20 && e[32 + i]; ++i) fprintf(stderr, " %lld", e[32 + i] - e[32 + i - 1]);
                fprintf(stderr, "\n");
            }
        }
    }
}
}  // namespace

// Split solve of a batch of FFT-path plans with one transform length; false
// when the batch is not eligible (the caller falls back to the fused kernel).
bool launch_split(const std::vector<SolveJob> &jobs, cudaStream_t s, Workspace &ws) {
    static const int mode = getenv("FD_SPLIT") ? atoi(getenv("FD_SPLIT")) : 0;
    if (!mode) return false;
    const int n = jobs[0].p.n;
    if (n + 1 != 1024) return false;
    for (auto &j : jobs) {
        if (!j.p.ralpha || !j.p.fe || j.p.cyclic || j.p.nsing) return false;
        if (j.tlen > j.p.ecap) return false;   // table-free modes must reach their fixed point within the fe rows
    }
    run_split<10>(jobs, s, ws);
    return true;
}

}  // namespace fd
