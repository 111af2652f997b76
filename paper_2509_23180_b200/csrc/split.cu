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
};
struct XList {
    int count, n;
    const double *ralpha;   // [N] pre-weights
    const double2 *m16;     // [16] e^{-2 pi i q / 256}  (N >= 512), then la[NB] e^{-2 pi i q / N}
    XJob job[kMaxPJobs];
};

template <int NL>
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
    F::load(v, A, hb ? A + J.spitch : nullptr, xl.ralpha, J.h2, t);
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
            for (int q = t; q < n; q += T) oh[q] = fma(be_, __ldg(qh + q), al_ * Xh[xi(q)]);
        } else if (al_ == 1.0) {
#pragma unroll 8
            for (int q = t; q < n; q += T) oh[q] = Xh[xi(q)];
        } else {
#pragma unroll 8
            for (int q = t; q < n; q += T) oh[q] = al_ * Xh[xi(q)];
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
    const bool inb = q < W && !(tl.dbgmask & 2);                // lane owns a column of the tile
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
        // make sure tile t's copies have landed (counters were read a tile ago)
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
        // chunk c (16 rows; ascending c forward, descending backward) of tile t in slot g -> registers
        auto load = [&](int t, int g, int c, double (&dv)[kCH], double (&fv)[kCH]) {
            const double *sl = slots + size_t(g) * TILE + c * kCH * W + qq;
            if (!(tl.dbgmask & 4)) {
#pragma unroll
                for (int r = 0; r < kCH; ++r) dv[r] = sl[r * W];
            }
            const int i0 = t * kSR + c * kCH;
            if (fact(t)) {
                const double *fs = fslots + size_t(t % kFG) * TILE + c * kCH * W + qq;
                const bool tab = i0 < ecap || tabm;
#pragma unroll
                for (int r = 0; r < kCH; ++r) {
                    const double cst = BWD ? ((i0 + r == m - 1) ? ib_last : ib_inf) : l_inf;
                    fv[r] = tab ? fs[r * W] : cst;
                }
            } else if (BWD && t == T - 1) {
#pragma unroll
                for (int r = 0; r < kCH; ++r) fv[r] = (i0 + r == m - 1) ? ib_last : ib_inf;
            }
            if (BWD && t == T - 1) {   // the forward pass ran on past row m-1 in this (resident) tile
#pragma unroll
                for (int r = 0; r < kCH; ++r)
                    if (i0 + r >= m) dv[r] = 0.0;
            }
        };
        // One chunk of the recurrence.  The results stay in registers (oc) and are
        // stored one chunk LATER, interleaved with the next chunk's chain (op, sp):
        // a store issued right behind the DFMA that produces its value waits ~20
        // cycles for the fp64 result and, the warp issuing in order, holds up the
        // next link of the chain (measured: 21.7 instead of 8.2 cycles per row).
        auto compute = [&](int t, const double (&dv)[kCH], const double (&fv)[kCH], double (&oc)[kCH],
                           const double (&op)[kCH], double *sp) {
            const bool st = inb && sp != nullptr;
            if (fact(t) || (BWD && t == T - 1)) {
                if (!BWD) {
#pragma unroll
                    for (int r = 0; r < kCH; ++r) {
                        carry = fma(-fv[r], carry, dv[r]);
                        oc[r] = carry;
                        if (st) sp[r * W] = op[r];
                    }
                } else {
                    double a[kCH], gg[kCH];
#pragma unroll
                    for (int r = 0; r < kCH; ++r) {
                        a[r] = dv[r] * fv[r];
                        gg[r] = noff * fv[r];
                    }
#pragma unroll
                    for (int r = kCH - 1; r >= 0; --r) {
                        carry = fma(gg[r], carry, a[r]);
                        oc[r] = carry;
                        if (st) sp[r * W] = op[r];
                    }
                }
            } else if (!BWD) {
#pragma unroll
                for (int r = 0; r < kCH; ++r) {
                    carry = fma(nl_inf, carry, dv[r]);
                    oc[r] = carry;
                    if (st) sp[r * W] = op[r];
                }
            } else {
                double a[kCH];
#pragma unroll
                for (int r = 0; r < kCH; ++r) a[r] = dv[r] * ib_inf;
#pragma unroll
                for (int r = kCH - 1; r >= 0; --r) {
                    carry = fma(g_inf, carry, a[r]);
                    oc[r] = carry;
                    if (st) sp[r * W] = op[r];
                }
            }
        };
        auto signal = [&](int t, int g) {
            // the producer's tensor store reads the slot (streamed y, every xhat tile)
            if (BWD || t < TS) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&done[g]);
        };
        // Tile loop; the four chunks of a tile are unrolled with compile-time
        // chunk indices, the registers ping-pong (A, B, A, B), and the last
        // chunk prefetches the first chunk of the next tile.
        double da[kCH], fa[kCH], db[kCH], fb[kCH], oa[kCH], ob[kCH];
        double *sprev = nullptr;   // where the previous chunk's results (in oa / ob) go
        int t = BWD ? T - 1 : 0, g = t % NG;
        int tp = t, gp = g;
        acquire(t);
        load(t, g, BWD ? NC - 1 : 0, da, fa);
        for (int it = 0; it < T; ++it) {
            const int tn = t + dir, gn = wrap(g);
            const bool more = it + 1 < T;
            // counters for the next tile: read now, compared after this tile's first chunks
            dseen = ld_acquire(&landed[0]);
            fseen = ld_acquire(&landed[1]);
#pragma unroll
            for (int ci = 0; ci < NC; ++ci) {
                const int c = BWD ? NC - 1 - ci : ci;
                double *sl = slots + size_t(g) * TILE + c * kCH * W + qq;
                auto body = [&](double (&dc)[kCH], double (&fc)[kCH], double (&dn)[kCH], double (&fn)[kCH],
                                double (&oc)[kCH], double (&op)[kCH]) {
                    if (ci + 1 < NC) {
                        load(t, g, c + dir, dn, fn);
                    } else if (more) {
                        acquire(tn);
                        load(tn, gn, BWD ? NC - 1 : 0, dn, fn);
                    }
                    compute(t, dc, fc, oc, op, sprev);
                };
                if (ci & 1) body(db, fb, da, fa, ob, oa);
                else body(da, fa, db, fb, oa, ob);
                sprev = sl;
                if (ci == 0 && it > 0) signal(tp, gp);   // the previous tile's last stores have been issued
            }
            if (tl.dbg && tid == 0 && it < 20) tl.dbg[size_t(gridDim.x) * 16 + size_t(blockIdx.x) * 64 + (BWD ? 32 : 0) + it] = clock64();
            tp = t;
            gp = g;
            t = tn;
            g = gn;
        }
        if (inb) {   // NC is even: the last chunk's results are in ob
#pragma unroll
            for (int r = 0; r < kCH; ++r) sprev[r * W] = ob[r];
        }
        signal(tp, gp);
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
    const int n = jobs[0].p.n, NP = C::N;
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
            c = a;
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
        dst_pair_kernel<NL><<<pairs, C::T, xsmem, s>>>(xa);
        FD_CUDA(cudaGetLastError());
        if (timing) FD_CUDA(cudaEventRecord(ev[1], s));
        launch_thomas(W, ctas, tsmem, s, tl, di.smem);
        FD_CUDA(cudaGetLastError());
        if (timing) FD_CUDA(cudaEventRecord(ev[2], s));
        dst_pair_kernel<NL><<<pairs, C::T, xsmem, s>>>(xc);
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
