// Shared pieces of the persistent fused-solve kernels (rsolve.cu, rsws.cu,
// persist.cu): job/segment descriptors, TMA bulk-copy + mbarrier helpers,
// per-mode factor access, and the host-side cooperative launcher.
#pragma once
#include <cooperative_groups.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "dst_device.cuh"
#include "fd_internal.h"

namespace fd {
namespace cg = cooperative_groups;

struct PJob {
    PlanDev p;
    const double *in;
    double *out;
    double alpha, beta;
    const double *other;
    long long row0;   // first global row of the job
    int c_first;      // first virtual range touching the job
    int nblk;         // carry blocks of the job
    int blk_base;     // global index of its first block
};

constexpr int kMaxPJobs = 8;
constexpr int kMaxSegs = 48;
constexpr int kMaxRowsPerBlock = 256;   // keeps block products P_e far from underflow
constexpr int kCarryVals = 7;           // yhat_e, F_s, P_e, xi_s, Q, Y, X
constexpr int kMaxV = 512;              // virtual row ranges per launch

struct PList {
    int count;
    int V;               // virtual row ranges (carry blocks)
    long long total_rows;
    double *carry;       // [total_blocks][kCarryVals][cn]
    int n;
    int cn;              // even row pitch of the carry rows (n rounded up): 16-byte aligned rows for bulk copies
    unsigned long long *tstamp;   // optional [gridDim][8] phase timestamps (FD_PHASE_TIMING)
    unsigned long long *trace;    // optional per-item timeline of one CTA (FD_TRACE=cta)
    int trace_cta;
    int dbg;             // FD_DBG experiment bits (timing studies only; 0 in production)
    double *bsave;       // [gridDim][bstride][n] beta checkpoints (phase 1 -> phase 3)
    int bstride;
    PJob job[kMaxPJobs];
    int vstart[kMaxV + 1];   // global first row of virtual range v (cost-balanced)
};

struct Seg {
    int job, s, e, blk, ngroups, item0;
};

// --- TMA bulk copy + mbarrier helpers --------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Issue the copy of rows [g0, g0+rows) of an (m, n) array into `stg`; the data
// lands at stg + off where off = (address mod 16) / 8.  The bulk copy is
// widened to 16-byte boundaries; only the last group of an array, whose end may
// be the end of the allocation, leaves an 8-byte tail that thread 0 fetches
// into a register (returned) and stores once the copy has landed.
struct Tail {
    double v;
    int idx;   // -1: none
};
// The table slice (lt != null) is counted in the same expect_tx; with
// defer_lt its copy is left to issue_lt(), so the slice buffer can still be
// read by the current group (the mbarrier phase completes only when both
// copies have landed).
__device__ __forceinline__ void issue_lt(double *ltstg, const double *lt, int g0, int rows, int ktp,
                                         uint64_t *bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tma_load_1d(ltstg, lt + size_t(g0) * 3 * ktp, uint32_t(rows) * 3u * uint32_t(ktp) * 8u, bar);
}
__device__ __forceinline__ Tail issue_rows(double *stg, const double *base, int g0, int rows, int n,
                                           int m, uint64_t *bar, double *ltstg = nullptr,
                                           const double *lt = nullptr, int ktp = 0,
                                           bool defer_lt = false) {
    const uintptr_t start = reinterpret_cast<uintptr_t>(base + size_t(g0) * n);
    const uintptr_t end = start + uintptr_t(rows) * n * sizeof(double);
    const uintptr_t a = start & ~uintptr_t(15);
    const bool last = (g0 + rows >= m);
    const uintptr_t e = last ? (end & ~uintptr_t(15)) : ((end + 15) & ~uintptr_t(15));
    const uint32_t bytes = uint32_t(e - a);
    const uint32_t ltbytes = lt ? uint32_t(rows) * 3u * uint32_t(ktp) * 8u : 0u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, bytes + ltbytes);
    tma_load_1d(stg, reinterpret_cast<const void *>(a), bytes, bar);
    if (ltbytes && !defer_lt) tma_load_1d(ltstg, lt + size_t(g0) * 3 * ktp, ltbytes, bar);
    Tail t{0.0, -1};
    if (end != e) {
        t.v = __ldcg(reinterpret_cast<const double *>(e));
        t.idx = int((e - a) / 8);
    }
    return t;
}
// true when the group's copy leaves a tail (identical on every thread)
__device__ __forceinline__ bool has_tail(const double *base, int g0, int rows, int n, int m) {
    const uintptr_t end = reinterpret_cast<uintptr_t>(base + size_t(g0 + rows) * n);
    return (g0 + rows >= m) && (end & 15);
}

__device__ __forceinline__ int stg_off(const double *base, int g0, int n) {
    return int((reinterpret_cast<uintptr_t>(base + size_t(g0) * n) & 15) >> 3);
}

// Per-mode record (PlanDev::mode, 64 B): l_inf, 1/beta_inf, beta_inf,
// 1/(-l_inf), beta_{m-1}, lambda_k, explicit offset, explicit length.
struct ModeRec {
    double l_inf, ib_inf, b_inf, inv_nl, b_last, lam;
    int off, len;
    __device__ void load(const PlanDev &p, int k) {
        const double2 *r = reinterpret_cast<const double2 *>(p.mode) + 4 * k;
        const double2 a = __ldg(r), b = __ldg(r + 1), c = __ldg(r + 2), d = __ldg(r + 3);
        l_inf = a.x;
        ib_inf = a.y;
        b_inf = b.x;
        inv_nl = b.y;
        b_last = c.x;
        lam = c.y;
        off = int(__double_as_longlong(d.x));
        len = int(__double_as_longlong(d.y));
    }
};

__device__ __forceinline__ double mode_lam(const PlanDev &p, int k) { return __ldg(p.mode + 8 * size_t(k) + 5); }
__device__ __forceinline__ double mode_blast(const PlanDev &p, int k) { return __ldg(p.mode + 8 * size_t(k) + 4); }
__device__ __forceinline__ double mode_binf(const PlanDev &p, int k) { return __ldg(p.mode + 8 * size_t(k) + 2); }

// beta_i of mode k from the plan's tables (used once per segment start)
__device__ __forceinline__ double beta_at(const PlanDev &p, const ModeRec &c, int k, int i) {
    if (i == p.m - 1) return c.b_last;
    if (i < p.ecap) return __ldg(p.db + size_t(i) * p.n + k);
    if (i < c.len) return __ldg(p.ex + 4 * (size_t(c.off) + i) + 2);
    return c.b_inf;
}

// Diagonal of row i: lambda (+ west modifier on row 0) (+ east on row m-1),
// summed in the reference's order (rectsolver.py:125,132-133).
__device__ __forceinline__ double diag_at(const PlanDev &p, double lam, int i) {
    double d = lam;
    if (i == 0) d = __dadd_rn(d, p.mod_w);
    if (i == p.m - 1) d = __dadd_rn(d, p.mod_e);
    return d;
}

// ---------------------------------------------------------------------------
// host launcher
// K: kernel traits with static members NT (threads), G (rows per item),
// SMEM (dynamic shared bytes) and fn() (the __global__ entry point).
template <class K>
static int persist_grid(int device) {
    static std::mutex mu;
    static std::map<int, int> cache;
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(device);
    if (it != cache.end()) return it->second;
    FD_CUDA(cudaFuncSetAttribute(K::fn(), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM));
    int per_sm = 0, sms = 0;
    FD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, K::fn(), K::NT, K::SMEM));
    FD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    if (per_sm < 1) FD_FAIL(FD_ERR_CUDA, "persistent solve kernel cannot be resident");
    cache[device] = per_sm * sms;
    return per_sm * sms;
}

template <class K>
static void run_persist(const std::vector<SolveJob> &jobs, cudaStream_t s, Workspace &ws) {
    using C = K;
    int device = 0;
    FD_CUDA(cudaGetDevice(&device));
    const int grid = persist_grid<K>(device);
    for (size_t j0 = 0; j0 < jobs.size(); j0 += kMaxPJobs) {
        PList pl{};
        pl.count = (int)std::min<size_t>(kMaxPJobs, jobs.size() - j0);
        pl.n = jobs[j0].p.n;
        long long total = 0;
        for (int j = 0; j < pl.count; ++j) total += jobs[j0 + j].p.m;
        pl.total_rows = total;
        long long V = std::max<long long>(grid, (total + kMaxRowsPerBlock - 1) / kMaxRowsPerBlock);
        // more ranges than CTAs (long batches, rows-per-block cap): a whole number of
        // ranges per CTA, or some CTAs would sweep one range more than the others
        if (V > grid && (V + grid - 1) / grid * grid <= kMaxV) V = (V + grid - 1) / grid * grid;
        V = std::min<long long>(std::min<long long>(V, total), kMaxV);
        pl.V = (int)V;
        // Cost-balanced ranges: a row weighs 1 + tau1 * (fraction of modes in
        // their transient at that row); a subdomain's first row carries the
        // extra group/segment set-up (tau0 rows).
        // Group quantisation: a range one row longer than a whole number of row groups
        // pays a whole extra group in both phases.  When the average range fits k
        // groups, the transient weights are backed off (x 2/3, 1/3, 0) until no range
        // of one subdomain is longer than k groups.
        const long long cap = ((total + V - 1) / V + K::G - 1) / K::G * K::G;
        for (int attempt = 0; attempt < 4; ++attempt) {
            static const double tau1_ = getenv("FD_TAU1") ? atof(getenv("FD_TAU1")) : 1.2;
            static const double tau0_ = getenv("FD_TAU0") ? atof(getenv("FD_TAU0")) : 4.0;
            // a row with any sizeable set of modes in their transient pays the divergent
            // transient path in every warp that holds one of them (step term)
            static const double tau2_ = getenv("FD_TAU2") ? atof(getenv("FD_TAU2")) : 0.3;
            const double back = double(3 - attempt) / 3.0;
            const double tau1 = tau1_ * back, tau0 = tau0_ * back, tau2 = tau2_ * back;
            struct JW {
                long long r0;
                int m, t;
                double start;
                std::vector<double> pre;   // cumulative weight of rows [0, i), i <= t
            };
            std::vector<JW> jw(pl.count);
            double W = 0.0;
            long long r0 = 0;
            for (int j = 0; j < pl.count; ++j) {
                const SolveJob &sj = jobs[j0 + j];
                JW &q = jw[j];
                q.r0 = r0;
                q.m = sj.p.m;
                q.t = std::min(sj.tlen, q.m);
                q.start = W;
                q.pre.assign(q.t + 1, 0.0);
                for (int i = 0; i < q.t; ++i)
                    q.pre[i + 1] = q.pre[i] + 1.0 + tau1 * sj.tprof[i] + (sj.tprof[i] > 0.02f ? tau2 : 0.0) +
                                   (i == 0 ? tau0 : 0.0);
                const double wj = (q.t > 0 ? q.pre[q.t] : tau0) + double(q.m - q.t);
                W += wj;
                r0 += q.m;
            }
            auto row_at = [&](double target) -> long long {   // first row whose cumulative weight reaches target
                int j = 0;
                while (j + 1 < pl.count && jw[j + 1].start <= target) ++j;
                const JW &q = jw[j];
                double x = target - q.start;
                if (q.t > 0 && x <= q.pre[q.t]) {
                    const int i = int(std::lower_bound(q.pre.begin(), q.pre.end(), x) - q.pre.begin());
                    return q.r0 + std::min(i, q.m);
                }
                x -= (q.t > 0 ? q.pre[q.t] : tau0);
                return q.r0 + std::min<long long>(q.m, q.t + (long long)std::ceil(x));
            };
            pl.vstart[0] = 0;
            static const long long snap = getenv("FD_SNAP") ? atoll(getenv("FD_SNAP")) : 3;
            for (long long v = 1; v < V; ++v) {
                long long r = row_at(W * double(v) / double(V));
                // snap to a subdomain start within 3 rows: no tiny extra segment
                for (int j = 1; j < pl.count; ++j)
                    if (std::llabs(r - jw[j].r0) <= snap) r = jw[j].r0;
                r = std::max<long long>(r, pl.vstart[v - 1] + 1);             // non-empty ranges
                r = std::min<long long>(r, total - (V - v));
                pl.vstart[v] = (int)r;
            }
            pl.vstart[V] = (int)total;
            bool over = false;
            for (long long v = 0; v < V && !over; ++v) {
                if (pl.vstart[v + 1] - pl.vstart[v] <= cap) continue;
                bool one_job = false;   // ranges across a subdomain start have their own group structure
                for (int j = 0; j < pl.count; ++j)
                    one_job = one_job || (pl.vstart[v] >= jw[j].r0 && pl.vstart[v + 1] <= jw[j].r0 + jw[j].m);
                over = one_job;
            }
            if (!over) break;
        }
        auto lo = [&](long long v) { return (long long)pl.vstart[v]; };
        auto range_of = [&](long long r) {   // largest v with lo(v) <= r
            return (long long)(std::upper_bound(pl.vstart, pl.vstart + V + 1, (int)r) - pl.vstart) - 1;
        };
        long long row0 = 0;
        int blocks = 0;
        for (int j = 0; j < pl.count; ++j) {
            const SolveJob &sj = jobs[j0 + j];
            PJob &pj = pl.job[j];
            pj.p = sj.p;
            pj.in = sj.in;
            pj.out = sj.out;
            pj.alpha = sj.alpha;
            pj.beta = sj.beta;
            pj.other = sj.other;
            pj.row0 = row0;
            const long long cf = range_of(row0), cl = range_of(row0 + sj.p.m - 1);
            pj.c_first = (int)cf;
            pj.nblk = (int)(cl - cf + 1);
            pj.blk_base = blocks;
            blocks += pj.nblk;
            row0 += sj.p.m;
        }
        pl.cn = (pl.n + 1) & ~1;
        const size_t carry_sz = size_t(blocks) * kCarryVals * pl.cn;
        pl.carry = ws.get(carry_sz);
        pl.bsave = nullptr;
        pl.bstride = 0;
        static const bool timing = getenv("FD_PHASE_TIMING") != nullptr;
        unsigned long long *ts = nullptr;
        if (timing) FD_CUDA(cudaMallocAsync(&ts, sizeof(unsigned long long) * 8 * grid, s));
        pl.tstamp = ts;

        static const bool tracing = getenv("FD_TRACE") != nullptr;
        unsigned long long *tr = nullptr;
        if (tracing) {
            FD_CUDA(cudaMallocAsync(&tr, sizeof(unsigned long long) * (16 * 64 * 2 + 64), s));
            FD_CUDA(cudaMemsetAsync(tr, 0, sizeof(unsigned long long) * (16 * 64 * 2 + 64), s));
        }
        pl.trace = tr;
        pl.trace_cta = tracing ? atoi(getenv("FD_TRACE")) : 0;
        static const int dbg = getenv("FD_DBG") ? atoi(getenv("FD_DBG")) : 0;
        pl.dbg = dbg;
        void *args[] = {(void *)&pl};
        FD_CUDA(cudaLaunchCooperativeKernel(K::fn(), dim3(grid), dim3(C::NT), args, C::SMEM, s));
        if (tracing) {
            std::vector<unsigned long long> h(16 * 64 * 2 + 64);
            FD_CUDA(cudaMemcpyAsync(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost, s));
            FD_CUDA(cudaStreamSynchronize(s));
            FD_CUDA(cudaFreeAsync(tr, s));
            unsigned long long t0 = ~0ull;
            for (auto v : h)
                if (v) t0 = std::min(t0, v);
            if (pl.dbg & 4) {   // per-pass cycle stamps of pair 0 (rsolve)
                for (int it = 0; it < 8; ++it) {   // phase 1 items 0-3, then phase 3 items 0-3
                    const long long *c = reinterpret_cast<const long long *>(h.data()) + 2048 + it * 8;
                    if (!c[0]) continue;
                    fprintf(stderr, "[fft cycles p%d it %d] load %lld first %lld mid %lld last %lld post %lld\n",
                            it < 4 ? 1 : 3, it & 3, c[1] - c[0], c[2] - c[1], c[3] - c[2], c[4] - c[3], c[5] - c[4]);
                }
            }
            for (int role = 0; role < 16; ++role) {
                bool any = false;
                for (int it = 0; it < 64; ++it)
                    if (h[(role * 64 + it) * 2] || h[(role * 64 + it) * 2 + 1]) any = true;
                if (!any) continue;
                fprintf(stderr, "[trace role %2d]", role);
                for (int it = 0; it < 64; ++it) {
                    const auto a = h[(role * 64 + it) * 2], b = h[(role * 64 + it) * 2 + 1];
                    if (a || b) fprintf(stderr, " %.1f/%.1f", a ? (a - t0) * 1e-3 : -1.0, b ? (b - t0) * 1e-3 : -1.0);
                }
                fprintf(stderr, "\n");
            }
        }
        if (timing) {
            std::vector<unsigned long long> h(8 * grid);
            FD_CUDA(cudaMemcpyAsync(h.data(), ts, h.size() * 8, cudaMemcpyDeviceToHost, s));
            FD_CUDA(cudaStreamSynchronize(s));
            FD_CUDA(cudaFreeAsync(ts, s));
            unsigned long long t0 = ~0ull;
            for (int c = 0; c < grid; ++c) t0 = std::min(t0, h[8 * c]);
            double mx[6] = {0}, mn[6] = {1e30, 1e30, 1e30, 1e30, 1e30, 1e30};
            for (int c = 0; c < grid; ++c)
                for (int k = 0; k < 6; ++k) {
                    double v = (h[8 * c + k] - t0) * 1e-3;
                    mx[k] = std::max(mx[k], v);
                    mn[k] = std::min(mn[k], v);
                }
            if (getenv("FD_PHASE_TIMING_CTA")) {
                // slowest CTAs of phase 1 and of phase 3
                for (int ph = 0; ph < 3; ++ph) {
                    std::vector<std::pair<double, int>> d;
                    const int s0 = ph == 0 ? 0 : ph == 1 ? 2 : 4;
                    for (int c = 0; c < grid; ++c) d.push_back({(h[8 * c + s0 + 1] - h[8 * c + s0]) * 1e-3, c});
                    std::sort(d.rbegin(), d.rend());
                    fprintf(stderr, "  slowest p%d:", ph + 1);
                    for (int q = 0; q < 12 && q < (int)d.size(); ++q)
                        fprintf(stderr, " cta%d[%d,%d)=%.1f", d[q].second, pl.vstart[d[q].second],
                                pl.vstart[d[q].second + 1], d[q].first);
                    fprintf(stderr, "  median %.1f\n", d[d.size() / 2].first);
                }
            }
            if (getenv("FD_PHASE_TIMING_ALL")) {   // every CTA: SM id, row range, phase-1 and phase-3 durations
                for (int c = 0; c < grid; ++c)
                    fprintf(stderr, "  cta %3d sm %3llu [%d,%d) p1 %.1f p3 %.1f\n", c, h[8 * c + 6], pl.vstart[c],
                            pl.vstart[c + 1], (h[8 * c + 1] - h[8 * c]) * 1e-3, (h[8 * c + 5] - h[8 * c + 4]) * 1e-3);
            }
            fprintf(stderr, "[fd phase us] start %.1f-%.1f p1end %.1f-%.1f sync1 %.1f-%.1f p2end %.1f-%.1f sync2 %.1f-%.1f end %.1f-%.1f (grid %d, V %d, rows %lld)\n",
                    mn[0], mx[0], mn[1], mx[1], mn[2], mx[2], mn[3], mx[3], mn[4], mx[4], mn[5], mx[5], grid, pl.V, total);
        }
    }
}


}  // namespace fd
