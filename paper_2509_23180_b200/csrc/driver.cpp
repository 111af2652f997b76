// Host orchestration + C ABI: Schur operator (ddm.py:94-136), restarted GMRES
// with device-resident Krylov basis (krylov.py:61-165), Algorithm 1
// (ddm.py:210-270).  Scalars of the Hessenberg/Givens recurrences live on the
// host in fp64 with -ffp-contract=off, so the least-squares arithmetic rounds
// like the reference's numpy scalars; every vector-sized operation runs in a
// kernel on the caller's stream.
#include <math.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <chrono>
#include <map>
#include <unordered_map>
#include <mutex>
#include <set>
#include <thread>
#include <sstream>
#include <tuple>

#include <nvtx3/nvToolsExt.h>

#include "fd_internal.h"

namespace fd {

Plan *plan_create(int m, int n, double dx, double dy, double kappa, double mod_w, double mod_e,
                  int device, int pair = kPairDD, int flags = 0);
void plan_destroy(Plan *p);
void factor_tables_host(int m, int n, double dx, double dy, double kappa, double mod_w,
                        double mod_e, double *beta, double *lower);

void *dmalloc(size_t bytes) {
    static std::mutex mu;
    static std::set<int> configured;
    int dev = 0;
    FD_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> g(mu);
        if (configured.insert(dev).second) {
            cudaMemPool_t pool;
            FD_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
            uint64_t keep = UINT64_MAX;
            FD_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        }
    }
    void *p = nullptr;
    FD_CUDA(cudaMallocAsync(&p, std::max<size_t>(bytes, 16), 0));
    FD_CUDA(cudaStreamSynchronize(0));
    return p;
}
void dfree(void *p) {
    if (p) cudaFreeAsync(p, 0);
}

// FD_HOST_TIMING=1: host-side phase times of the drivers on stderr (diagnostics)
// NVTX range of a host-side phase (header-only NVTX 3: a no-op unless a
// profiler is attached); the ranges name the phases of Algorithm 1 in nsys /
// ncu timelines: ddm_solve > presolves | gmres (> cycle) | backsub, schur_apply,
// rect_solve_batched.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

struct HostTimer {
    const char *name;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    bool on;
    explicit HostTimer(const char *n) : name(n) {
        static const int env = getenv("FD_HOST_TIMING") ? atoi(getenv("FD_HOST_TIMING")) : 0;
        on = env != 0;
        nosync = env == 2;   // 2: host clock only, no stream synchronisation
    }
    bool nosync = false;
    void mark(const char *what, cudaStream_t s = 0, bool sync = true) {
        if (!on) return;
        if (sync && !nosync) cudaStreamSynchronize(s);
        const auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "[fd host] %s %s %.3f ms\n", name, what,
                std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    }
};

static thread_local std::string g_last_error;
void set_error(const std::string &msg) { g_last_error = msg; }

// ---------------------------------------------------------------------------
// per-device scratch for reductions (used by the generic Arnoldi entry points)
struct Scratch {
    RedWork red;
    double *dval;      // device scalars
    double *hval;      // pinned host mirror
    int cap;
};
// Pinned host mirrors for the per-iteration scalar read-backs: page-locked
// allocations cost milliseconds, so released blocks are kept for reuse (one
// size class; the few blocks a process needs are never returned to the OS).
static std::mutex g_pin_mu;
static std::multimap<size_t, void *> *g_pin_free = new std::multimap<size_t, void *>();   // never destroyed
static std::map<void *, size_t> *g_pin_size = new std::map<void *, size_t>();
constexpr size_t kPinBytes = 8192;
static void *pinned_get(size_t bytes) {
    bytes = std::max(bytes, kPinBytes);
    {
        std::lock_guard<std::mutex> g(g_pin_mu);
        auto it = g_pin_free->lower_bound(bytes);
        if (it != g_pin_free->end()) {
            void *p = it->second;
            g_pin_free->erase(it);
            return p;
        }
    }
    void *p = nullptr;
    FD_CUDA(cudaMallocHost(&p, bytes));
    std::lock_guard<std::mutex> g(g_pin_mu);
    (*g_pin_size)[p] = bytes;
    return p;
}
static void pinned_put(void *p) {
    if (!p) return;
    std::lock_guard<std::mutex> g(g_pin_mu);
    g_pin_free->emplace((*g_pin_size)[p], p);
}

static Scratch make_scratch(int cap) {
    Scratch s{};
    s.red.partials = (double *)dmalloc(sizeof(double) * kRedBlocks);
    s.red.counter = (unsigned int *)dmalloc(sizeof(unsigned int));
    FD_CUDA(cudaMemset(s.red.counter, 0, sizeof(unsigned int)));
    s.dval = (double *)dmalloc(sizeof(double) * cap);
    s.hval = (double *)pinned_get(sizeof(double) * cap);
    s.cap = cap;
    return s;
}
static void free_scratch(Scratch &s) {   // callers synchronise the device first
    dfree(s.red.partials);
    dfree(s.red.counter);
    dfree(s.dval);
    pinned_put(s.hval);
}
// One scratch per (device, stream, host thread): calls on different streams
// or from different host threads never share a counter, partials or the
// pinned mirror.  Capacity grows with the request (restart length + 3).
static std::mutex g_scr_mu;
static std::map<std::tuple<int, cudaStream_t, std::thread::id>, Scratch> g_scratch;
static Scratch &device_scratch(cudaStream_t s, int need = 64) {
    int dev = 0;
    FD_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(g_scr_mu);
    auto key = std::make_tuple(dev, s, std::this_thread::get_id());
    auto it = g_scratch.find(key);
    if (it != g_scratch.end() && it->second.cap < need) {
        FD_CUDA(cudaStreamSynchronize(s));
        free_scratch(it->second);
        g_scratch.erase(it);
        it = g_scratch.end();
    }
    if (it == g_scratch.end()) it = g_scratch.emplace(key, make_scratch(std::max(need, 64))).first;
    return it->second;
}

// ---------------------------------------------------------------------------
// Arnoldi step (krylov.py:105-111): w_norm = ||w||; MGS against V[0..k];
// h[0..k] projections, h[k+1] = ||w|| after.  h, w_norm are host outputs.
static void arnoldi_step(long long N, int k, const double *V, double *w, double *h, double *w_norm,
                         Scratch &sc, cudaStream_t s) {
    if (k + 3 > sc.cap) FD_FAIL(FD_ERR_VALIDATION, "arnoldi: restart length too large");
    double *d = sc.dval;   // d[0] = ||w||^2, d[1..k+1] = h_0..h_k, d[k+2] = ||w_orth||^2
    launch_dot(N, w, w, d, sc.red, s);
    for (int i = 0; i <= k; ++i)
        launch_mgs(N, w, i ? V + (long long)(i - 1) * N : nullptr, i ? d + i : nullptr,
                   V + (long long)i * N, d + 1 + i, sc.red, s);
    launch_mgs(N, w, V + (long long)k * N, d + 1 + k, nullptr, d + k + 2, sc.red, s);
    FD_CUDA(cudaMemcpyAsync(sc.hval, d, sizeof(double) * (k + 3), cudaMemcpyDeviceToHost, s));
    FD_CUDA(cudaStreamSynchronize(s));
    *w_norm = sqrt(sc.hval[0]);
    for (int i = 0; i <= k; ++i) h[i] = sc.hval[1 + i];
    h[k + 1] = sqrt(sc.hval[k + 2]);
}

static double norm2(long long N, const double *x, Scratch &sc, cudaStream_t s) {
    launch_dot(N, x, x, sc.dval, sc.red, s);
    FD_CUDA(cudaMemcpyAsync(sc.hval, sc.dval, sizeof(double), cudaMemcpyDeviceToHost, s));
    FD_CUDA(cudaStreamSynchronize(s));
    return sqrt(sc.hval[0]);
}

// ---------------------------------------------------------------------------
// Schur operator
struct Coupling {
    int len;
    int64_t *from, *to;   // device, in the plans' internal layouts
    double c;
    int64_t *from_user;   // R_ci only: neighbour indices in the user layout (== from unless transposed)
};

}  // namespace fd

struct fd_plan_s {
    fd::Plan *p;
};

struct fd_schur_s {
    int device;
    fd::Plan *center;
    double mod_s, mod_n;
    std::vector<fd::Plan *> nb;
    std::vector<fd::Coupling> to_c, from_c;   // R_ci, R_ic per neighbour
    std::vector<double *> nbf;                // neighbour work fields (solve outputs)
    std::vector<double *> nbin;               // neighbour inputs: zero except the interface line
    double *tmp = nullptr, *tmp2 = nullptr;   // centre-sized work vectors
    // GMRES workspace
    double *V = nullptr;
    int vcap = 0;
    double *w = nullptr, *r = nullptr, *ydev = nullptr;
    int ycap = 0;
    fd::Scratch sc{};
    // low-synchronisation Arnoldi: Gram rows, partials, results (device) + pinned mirror
    fd::ArnWork arn{};
    double *arn_out = nullptr, *arn_host = nullptr;   // arn_host: two slots of kArnSlot
    cudaEvent_t arn_ev[2] = {nullptr, nullptr};        // a slot's results have landed
    // interface-only (Steklov) neighbour applies: per arm the
    // line positions of the R_ic / R_ci entries and the interface-end inverse
    // pivots; line buffers [arms][L]
    struct Steklov {
        int L = 0;
        int64_t *pos_in = nullptr, *pos_out = nullptr;   // device, per coupling entry
        double *invpiv = nullptr;                        // device [L]
    };
    std::vector<Steklov> stk;
    bool steklov = false;
    // the R_ci scatter-adds of all neighbours in one atomic launch: every centre
    // entry receives at most two contributions (checked at create), so the sum
    // onto the zero vector does not depend on their order
    bool fused_add = false;
    // small problems: the preconditioned apply (a dozen short launches) replayed
    // as one CUDA graph on a fixed input buffer (0 untried, 2 warmed, 1 ready, -1 off)
    int graph_state = 0;
    cudaGraphExec_t pgraph = nullptr;
    cudaStream_t gstream = nullptr;
    double *gin = nullptr;
    double *lines = nullptr, *lines_hat = nullptr;
    // sharded solve: arm i is solved on rank owner[i]; rank 0 holds
    // the centre, the Krylov basis and drives the protocol; every rank holds
    // the same operator object (plans, couplings, work fields of its arms)
    // the centre operator A_c in the caller's layout (unprecond_apply); set by
    // fd_schur_set_stencil, else taken from the centre plan
    struct Stencil {
        int m = 0, n = 0, px = 0, py = 0;
        double dx = 0, dy = 0, kappa = 0, mw = 0, me = 0, ms = 0, mn = 0;
    } stencil;
    bool stencil_set = false;
    fd_comm_s *comm = nullptr;
    std::vector<int> owner;
    int64_t *iota = nullptr;                  // 0 .. max line length - 1
    std::vector<double *> sline, rline;       // per arm: line out / line back (device)
    long long *cmd = nullptr;                 // device command word
    long long *cmd_host = nullptr;            // pinned mirror
    std::vector<void *> allocs;
    bool remote(size_t i) const { return comm && owner[i] != comm->t->rank; }
    bool dist() const { return comm && comm->t->nranks > 1; }
};

namespace fd {

static void *dalloc(fd_schur_s *op, size_t bytes) {
    void *d = nullptr;
    d = dmalloc(bytes);
    op->allocs.push_back(d);
    return d;
}

static void solve_batch(const std::vector<SolveJob> &jobs, cudaStream_t s) {
    // group by transform length (one pipeline launch per length)
    // by (transform length, pair, dense path): a periodic-sweep or pin_mean plan
    // of an FFT length runs the dense three-kernel solve
    std::map<std::tuple<int, int, bool>, std::vector<SolveJob>> groups;
    for (const auto &j : jobs) groups[{j.p.n, j.p.tpair, j.p.dense != nullptr}].push_back(j);
    for (auto &g : groups) launch_solve(g.second, s);
}

static SolveJob job_of(const Plan *p, const double *in, double *out) {
    SolveJob j{};
    j.p = p->dev;
    j.in = in;
    j.out = out;
    j.alpha = 1.0;
    j.beta = 0.0;
    j.other = nullptr;
    j.ws = const_cast<Workspace *>(&p->ws);
    j.tprof = p->tprof.data();
    j.tlen = (int)p->tprof.size();
    return j;
}

// Solves on fields in the caller's layout.  Plans with a transposed transform
// axis get their field transposed into the plan's scratch, solved in place
// there and transposed back with the epilogue out = alpha x + beta other.
struct UJob {
    Plan *p;
    const double *in;
    double *out;
    double alpha = 1.0, beta = 0.0;
    const double *other = nullptr;
};
static void solve_user(const std::vector<UJob> &uj, cudaStream_t s) {
    std::vector<SolveJob> jobs;
    std::vector<size_t> tr;
    for (size_t i = 0; i < uj.size(); ++i) {
        Plan *p = uj[i].p;
        if (!p->transposed) {
            SolveJob j = job_of(p, uj[i].in, uj[i].out);
            j.alpha = uj[i].alpha;
            j.beta = uj[i].beta;
            j.other = uj[i].other;
            jobs.push_back(j);
            continue;
        }
        for (size_t q : tr)
            if (uj[q].p == p) {   // one scratch per plan: a repeated plan runs on its own
                for (const UJob &u : uj) solve_user({u}, s);
                return;
            }
        const size_t cnt = size_t(p->m) * p->n;
        double *t = p->tws.get(cnt);
        launch_transpose(p->um, p->un, uj[i].in, t, 1.0, 0.0, nullptr, s);
        jobs.push_back(job_of(p, t, t));
        tr.push_back(i);
    }
    solve_batch(jobs, s);
    for (size_t i : tr) {
        Plan *p = uj[i].p;
        launch_transpose(p->m, p->n, p->tws.ptr, uj[i].out, uj[i].alpha, uj[i].beta, uj[i].other, s);
    }
}

// Interface-only form of the same sum: for a DD line of length L adjacent to an
// interface end of the sweep, R_ci A_i^{-1} R_ic restricted to that line is
// c_ci c_ic Q diag(1 / beta_end) Q^T (Q the orthonormal DST-I of the line): the
// neighbour's field is zero except on the line, so the forward elimination is
// y = r on the line row and the back-substitution's interface value is
// y / beta_end -- the arm's full solve yields exactly these values there.
// O(L log L) per arm instead of a full arm solve.
// R_ci parts of every neighbour added into out (zero): one atomic launch when
// fused_add holds, else one ordered launch per neighbour (ddm.py:120-122)
static void scatter_add_parts(fd_schur_s *op, const std::vector<const int64_t *> &from,
                              const std::vector<const double *> &src, double *out, cudaStream_t s) {
    const size_t nnb = op->nb.size();
    if (op->fused_add) {
        ScatterBatch b{};
        b.count = (int)nnb;
        for (size_t i = 0; i < nnb; ++i) {
            const Coupling &c = op->to_c[i];
            b.len[i] = c.len;
            b.from[i] = from[i];
            b.to[i] = c.to;
            b.c[i] = c.c;
            b.src[i] = src[i];
            b.dst[i] = out;
        }
        launch_scatter_batch(b, 1, s);
        return;
    }
    for (size_t i = 0; i < nnb; ++i) {
        const Coupling &c = op->to_c[i];
        launch_scatter(c.len, from[i], c.to, c.c, src[i], out, 1, s);
    }
}

// Interface-only form of the same sum: for a DD line of length L adjacent to an
// interface end of the sweep, R_ci A_i^{-1} R_ic restricted to that line is
// c_ci c_ic Q diag(1 / beta_end) Q^T (Q the orthonormal DST-I of the line): the
// neighbour's field is zero except on the line, so the forward elimination is
// y = r on the line row and the back-substitution's interface value is
// y / beta_end -- the arm's full solve yields exactly these values there.
// O(L log L) per arm instead of a full arm solve.  out_zero: out is already
// zero (the operator's own centre vector), no field-sized memset.
static void schur_apply_steklov(fd_schur_s *op, const double *p, double *out, bool out_zero, cudaStream_t s) {
    const size_t nnb = op->nb.size();
    const int L = op->stk[0].L;
    FD_CUDA(cudaMemsetAsync(op->lines, 0, sizeof(double) * nnb * L, s));
    for (size_t i = 0; i < nnb; ++i) {
        const Coupling &c = op->from_c[i];   // centre line -> the arm's interface line
        launch_scatter(c.len, c.from, op->stk[i].pos_in, c.c, p, op->lines + i * L, 0, s);
    }
    launch_dst_rows((int)nnb, L, op->lines, op->lines_hat, twiddles_for(op->device, L),
                    dense_table_for(op->device, L), s);
    for (size_t i = 0; i < nnb; ++i)
        launch_mul(L, op->lines_hat + i * L, op->stk[i].invpiv, op->lines_hat + i * L, s);
    launch_dst_rows((int)nnb, L, op->lines_hat, op->lines, twiddles_for(op->device, L),
                    dense_table_for(op->device, L), s);
    const Plan *cp = op->center;
    if (!out_zero) FD_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * cp->m * cp->n, s));
    std::vector<const int64_t *> from(nnb);
    std::vector<const double *> src(nnb);
    for (size_t i = 0; i < nnb; ++i) {
        from[i] = op->stk[i].pos_out;
        src[i] = op->lines + i * L;
    }
    scatter_add_parts(op, from, src, out, s);
}

// command words of the sharded protocol (rank 0 -> arm owners)
enum : long long { kCmdDone = 0, kCmdApply = 1, kCmdBacksub = 2 };

static void send_command(fd_schur_s *op, long long cmd, cudaStream_t s) {
    Transport &t = *op->comm->t;
    *op->cmd_host = cmd;
    FD_CUDA(cudaMemcpyAsync(op->cmd, op->cmd_host, sizeof(long long), cudaMemcpyHostToDevice, s));
    t.group_start();
    for (int r = 1; r < t.nranks; ++r) t.send(op->cmd, sizeof(long long), r, s);
    t.group_end();
    // the pinned word is rewritten by the next command: wait for this copy
    FD_CUDA(cudaStreamSynchronize(s));
}

// rank 0: R_ic lines of the remote arms to their owners (c_ic p[from])
static void send_lines(fd_schur_s *op, const double *p, cudaStream_t s) {
    Transport &t = *op->comm->t;
    for (size_t i = 0; i < op->nb.size(); ++i)
        if (op->remote(i)) {
            const Coupling &c = op->from_c[i];
            launch_scatter(c.len, c.from, op->iota, c.c, p, op->sline[i], 0, s);
        }
    t.group_start();
    for (size_t i = 0; i < op->nb.size(); ++i)
        if (op->remote(i)) t.send(op->sline[i], sizeof(double) * op->from_c[i].len, op->owner[i], s);
    t.group_end();
}

// out = sum_i R_ci A_i^{-1} R_ic p   (ddm.py:108-123).  The neighbour inputs
// stay zero between applies: the interface lines are gathered in (one launch),
// solved out of place and cleared again (one launch).  Sharded: the remote
// arms' lines go to their owners first, the local arms are solved meanwhile,
// and the returned R_ci lines are added in neighbour order with the local ones.
static void schur_apply(fd_schur_s *op, const double *p, double *out, cudaStream_t s, bool out_zero = false) {
    if (op->steklov) {
        schur_apply_steklov(op, p, out, out_zero, s);
        return;
    }
    if (op->dist()) {
        Transport &t = *op->comm->t;
        send_command(op, kCmdApply, s);
        send_lines(op, p, s);
        std::vector<SolveJob> jobs;
        for (size_t i = 0; i < op->nb.size(); ++i) {
            if (op->remote(i)) continue;
            const Coupling &c = op->from_c[i];
            launch_scatter(c.len, c.from, c.to, c.c, p, op->nbin[i], 0, s);
            jobs.push_back(job_of(op->nb[i], op->nbin[i], op->nbf[i]));
        }
        if (!jobs.empty()) solve_batch(jobs, s);
        for (size_t i = 0; i < op->nb.size(); ++i)
            if (!op->remote(i)) launch_zero_at(op->from_c[i].len, op->from_c[i].to, op->nbin[i], s);
        t.group_start();
        for (size_t i = 0; i < op->nb.size(); ++i)
            if (op->remote(i)) t.recv(op->rline[i], sizeof(double) * op->to_c[i].len, op->owner[i], s);
        t.group_end();
        const Plan *cp = op->center;
        if (!out_zero) FD_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * cp->m * cp->n, s));
        // R_ci parts in neighbour order (remote parts arrive already scaled by c_ci)
        for (size_t i = 0; i < op->nb.size(); ++i) {
            const Coupling &c = op->to_c[i];
            if (op->remote(i)) launch_scatter(c.len, op->iota, c.to, 1.0, op->rline[i], out, 1, s);
            else launch_scatter(c.len, c.from, c.to, c.c, op->nbf[i], out, 1, s);
        }
        return;
    }
    const size_t nnb = op->nb.size();
    const bool batch = nnb <= (size_t)kMaxScatter;
    std::vector<SolveJob> jobs;
    ScatterBatch g{}, z{};
    g.count = z.count = batch ? (int)nnb : 0;
    for (size_t i = 0; i < nnb; ++i) {
        const Plan *q = op->nb[i];
        const Coupling &c = op->from_c[i];
        if (batch) {   // R_ic p into a zero field
            g.len[i] = z.len[i] = c.len;
            g.from[i] = z.from[i] = c.from;
            g.to[i] = z.to[i] = c.to;
            g.c[i] = z.c[i] = c.c;
            g.src[i] = z.src[i] = p;
            g.dst[i] = z.dst[i] = op->nbin[i];
        } else {
            launch_scatter(c.len, c.from, c.to, c.c, p, op->nbin[i], 0, s);
        }
        jobs.push_back(job_of(q, op->nbin[i], op->nbf[i]));
    }
    if (batch) launch_scatter_batch(g, 0, s);
    solve_batch(jobs, s);
    if (batch)
        launch_scatter_batch(z, 2, s);
    else
        for (size_t i = 0; i < nnb; ++i) launch_zero_at(op->from_c[i].len, op->from_c[i].to, op->nbin[i], s);
    const Plan *cp = op->center;
    if (!out_zero) FD_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * cp->m * cp->n, s));
    std::vector<const int64_t *> from(nnb);
    std::vector<const double *> src(nnb);
    for (size_t i = 0; i < nnb; ++i) {
        from[i] = op->to_c[i].from;
        src[i] = op->nbf[i];
    }
    scatter_add_parts(op, from, src, out, s);
}

// out = alpha * A_c^{-1} r + beta * other
static void center_solve(fd_schur_s *op, const double *r, double *out, double alpha, double beta,
                         const double *other, cudaStream_t s) {
    UJob j{op->center, r, out, alpha, beta, other};
    solve_user({j}, s);
}

// (I - A_c^{-1} S) p   (ddm.py:133-136); out must not alias p
// op->tmp is kept zero outside this function: only the interface lines are
// written and cleared again.
static void precond_apply(fd_schur_s *op, const double *p, double *out, cudaStream_t s) {
    schur_apply(op, p, op->tmp, s, true);
    center_solve(op, op->tmp, out, -1.0, 1.0, p, s);
    const size_t nnb = op->nb.size();
    if (nnb <= (size_t)kMaxScatter) {
        ScatterBatch z{};
        z.count = (int)nnb;
        for (size_t i = 0; i < nnb; ++i) {
            z.len[i] = op->to_c[i].len;
            z.to[i] = op->to_c[i].to;
            z.dst[i] = op->tmp;
        }
        launch_scatter_batch(z, 2, s);
    } else {
        for (size_t i = 0; i < nnb; ++i) launch_zero_at(op->to_c[i].len, op->to_c[i].to, op->tmp, s);
    }
}

static void drop_graph(fd_schur_s *op) {
    if (op->pgraph) cudaGraphExecDestroy(op->pgraph);
    op->pgraph = nullptr;
    op->graph_state = 0;
}

// precond_apply(op, p, op->w) for the GMRES loop.  Problems with only dense
// (three-kernel) solves and at most 2^18 centre points are launch-bound: after
// one warm-up apply the sequence is captured once into a graph that reads a
// fixed input copy, and every later apply is one copy + one graph launch.
static void precond_apply_loop(fd_schur_s *op, const double *p, cudaStream_t s) {
    const long long N = (long long)op->center->m * op->center->n;
    if (op->graph_state == 0) {
        bool ok = N <= (1LL << 18) && op->center->transform == kDense && !op->dist();
        for (const Plan *q : op->nb) ok = ok && (op->steklov || q->transform == kDense);
        op->graph_state = ok ? 2 : -1;
        precond_apply(op, p, op->w, s);
        return;
    }
    if (op->graph_state == 2) {
        op->graph_state = -1;   // unless the capture below succeeds
        try {
            if (!op->gin) op->gin = (double *)dalloc(op, sizeof(double) * N);
            if (!op->gstream) FD_CUDA(cudaStreamCreateWithFlags(&op->gstream, cudaStreamNonBlocking));
            FD_CUDA(cudaStreamBeginCapture(op->gstream, cudaStreamCaptureModeThreadLocal));
            cudaGraph_t g = nullptr;
            try {
                precond_apply(op, op->gin, op->w, op->gstream);
            } catch (...) {
                cudaStreamEndCapture(op->gstream, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            FD_CUDA(cudaStreamEndCapture(op->gstream, &g));
            const cudaError_t e = cudaGraphInstantiate(&op->pgraph, g, 0);
            cudaGraphDestroy(g);
            if (e == cudaSuccess) op->graph_state = 1;
        } catch (...) {
            op->pgraph = nullptr;
        }
        cudaGetLastError();   // a refused capture leaves no sticky error
    }
    if (op->graph_state == 1) {
        FD_CUDA(cudaMemcpyAsync(op->gin, p, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
        FD_CUDA(cudaGraphLaunch(op->pgraph, s));
    } else {
        precond_apply(op, p, op->w, s);
    }
}

// (A_c - S) p   (ddm.py:128-131)
static void unprecond_apply(fd_schur_s *op, const double *p, double *out, cudaStream_t s) {
    if (op->stencil_set) {
        const auto &t = op->stencil;
        launch_stencil(t.m, t.n, t.dx, t.dy, t.kappa, t.mw, t.me, t.ms, t.mn, p, op->tmp2, s, t.px, t.py);
    } else {
        launch_stencil(*op->center, op->mod_s, op->mod_n, p, op->tmp2, s);
    }
    schur_apply(op, p, out, s);
    const long long N = (long long)op->center->m * op->center->n;
    launch_axpby(N, 1.0, op->tmp2, -1.0, out, out, s);
}

constexpr size_t kArnSlot = 2 * kMaxArnoldi + 4;   // doubles per host result slot

static void ensure_arnoldi(fd_schur_s *op) {
    if (op->arn.partials) return;
    op->arn.partials = (double *)dalloc(op, sizeof(double) * kArnPartials);
    op->arn.counter = (unsigned int *)dalloc(op, sizeof(unsigned int));
    FD_CUDA(cudaMemset(op->arn.counter, 0, sizeof(unsigned int)));
    op->arn.G = (double *)dalloc(op, sizeof(double) * kMaxArnoldi * kMaxArnoldi);
    op->arn_out = (double *)dalloc(op, sizeof(double) * (2 * kMaxArnoldi + 4));
    op->arn_host = (double *)pinned_get(sizeof(double) * 2 * kArnSlot);
    for (auto &e : op->arn_ev) FD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

// Arnoldi step on the operator's basis with the low-synchronisation MGS of
// ops.cu (two passes over V instead of k + 1): h[0..k] projections, h[k+1] =
// ||w|| after, *w_norm = ||w|| before; V[k+1] = w / h[k+1] is formed on the
// device (unused by the caller on breakdown, like the reference).
//
// Split in two so the GMRES loop can pipeline: arnoldi_enqueue puts step k's
// operator apply, both passes, the normalisation and the copy of its results
// into host slot k % 2 on the stream; arnoldi_collect waits for that slot.
// Step k + 1 only needs V[k+1], which the device forms itself, so the loop
// enqueues it before it reads step k's column: the host round trip (copy,
// wake-up, Givens, the next launches) no longer leaves the GPU idle.
static void arnoldi_enqueue(fd_schur_s *op, long long N, int k, cudaStream_t s) {
    precond_apply_loop(op, op->V + (long long)k * N, s);   // -> w
    ArnWork a = op->arn;
    a.out = op->arn_out;
    launch_arnoldi_dots(N, k, op->V, op->w, a, kMaxArnoldi, s);
    ArnWork b = op->arn;
    b.out = op->arn_out + kMaxArnoldi + 2;
    launch_arnoldi_update(N, k, op->V, op->w, a.out, b, s);
    launch_scale_sqrt(N, op->w, b.out, op->V + (long long)(k + 1) * N, s);
    FD_CUDA(cudaMemcpyAsync(op->arn_host + (k & 1) * kArnSlot, op->arn_out, sizeof(double) * (kMaxArnoldi + 3),
                            cudaMemcpyDeviceToHost, s));
    FD_CUDA(cudaEventRecord(op->arn_ev[k & 1], s));
}
static void arnoldi_collect(fd_schur_s *op, int k, double *h, double *w_norm) {
    FD_CUDA(cudaEventSynchronize(op->arn_ev[k & 1]));
    const double *o = op->arn_host + (k & 1) * kArnSlot;
    for (int i = 0; i <= k; ++i) h[i] = o[i];
    *w_norm = sqrt(o[k + 1]);
    h[k + 1] = sqrt(o[kMaxArnoldi + 2]);
}

static void ensure_basis(fd_schur_s *op, int m) {
    ensure_arnoldi(op);
    if (op->ycap < m + 1) {   // back-solve coefficients y (k_used <= m)
        if (op->ydev) {
            FD_CUDA(cudaDeviceSynchronize());
            dfree(op->ydev);
        }
        op->ydev = (double *)dmalloc(sizeof(double) * (m + 1));
        op->ycap = m + 1;
    }
    if (op->vcap >= m + 1) return;
    if (op->V) {
        FD_CUDA(cudaDeviceSynchronize());
        dfree(op->V);
    }
    const long long N = (long long)op->center->m * op->center->n;
    op->V = (double *)dmalloc(sizeof(double) * N * (m + 1));
    op->vcap = m + 1;
    if (op->sc.cap < m + 8) {
        if (op->sc.cap) free_scratch(op->sc);
        op->sc = make_scratch(std::max(m + 8, 64));
    }
}

// Restarted GMRES on op.preconditioned (krylov.py:61-165).  x holds x0 (or is
// zeroed when x_is_zero).  Returns FD_OK or FD_ERR_NOT_CONVERGED.
static int gmres_precond(fd_schur_s *op, const double *rhs, double *x, int x_is_zero, int mcfg,
                         double tol, int max_restarts, std::vector<double> &hist, fd_report *rep,
                         cudaStream_t s) {
    const auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&] {
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    const long long N = (long long)op->center->m * op->center->n;
    const int m = (int)std::min<long long>(mcfg, N);
    ensure_basis(op, m);
    const bool lowsync = m + 1 <= kMaxArnoldi;   // else classic (k+1)-pass MGS
    Scratch &sc = op->sc;
    double *r = op->r, *w = op->w;
    if (x_is_zero) {
        FD_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * N, s));
        FD_CUDA(cudaMemcpyAsync(r, rhs, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    } else {
        precond_apply(op, x, w, s);
        launch_axpby(N, 1.0, rhs, -1.0, w, r, s);
    }
    const double r0 = norm2(N, r, sc, s);
    hist.clear();
    memset(rep, 0, sizeof(*rep));
    if (r0 == 0.0) {
        hist.push_back(0.0);
        rep->converged = 1;
        rep->wall_time = elapsed();
        return FD_OK;
    }
    hist.push_back(1.0);
    int total = 0, cycles = 0;
    std::vector<double> H((m + 1) * (size_t)m), g(m + 1), cs(m), sn(m), hcol(m + 2), y(m);
    auto Hat = [&](int i, int k) -> double & { return H[(size_t)i * m + k]; };
    for (int cyc = 0; cyc < max_restarts; ++cyc) {
        const double beta = norm2(N, r, sc, s);
        if (beta / r0 <= tol) break;
        ++cycles;
        NvtxRange nvtx_cycle("fd:gmres_cycle");
        std::fill(H.begin(), H.end(), 0.0);
        std::fill(g.begin(), g.end(), 0.0);
        std::fill(cs.begin(), cs.end(), 0.0);
        std::fill(sn.begin(), sn.end(), 0.0);
        sc.hval[0] = beta;
        FD_CUDA(cudaMemcpyAsync(sc.dval, sc.hval, sizeof(double), cudaMemcpyHostToDevice, s));
        launch_scale(N, r, sc.dval, op->V, s);   // V[0] = r / beta
        g[0] = beta;
        int k_used = 0;
        bool breakdown = false;
        if (lowsync) arnoldi_enqueue(op, N, 0, s);
        for (int k = 0; k < m; ++k) {
            double w_norm = 0.0;
            if (lowsync) {
                // step k + 1 is enqueued before step k's column is read; if step k
                // ends the cycle (breakdown, convergence) that work is discarded:
                // it touches only w, V[k+2], the Gram row k+1 and the other slot
                if (k + 1 < m) arnoldi_enqueue(op, N, k + 1, s);
                arnoldi_collect(op, k, hcol.data(), &w_norm);
            } else {
                precond_apply_loop(op, op->V + (long long)k * N, s);   // -> w
                arnoldi_step(N, k, op->V, w, hcol.data(), &w_norm, sc, s);
            }
            for (int i = 0; i <= k; ++i) Hat(i, k) = hcol[i];
            const double h_next = hcol[k + 1];
            Hat(k + 1, k) = h_next;
            for (int i = 0; i < k; ++i) {   // krylov.py:114-117
                const double t = cs[i] * Hat(i, k) + sn[i] * Hat(i + 1, k);
                Hat(i + 1, k) = -sn[i] * Hat(i, k) + cs[i] * Hat(i + 1, k);
                Hat(i, k) = t;
            }
            const double rho = hypot(Hat(k, k), Hat(k + 1, k));   // krylov.py:118-124
            cs[k] = rho != 0.0 ? Hat(k, k) / rho : 1.0;
            sn[k] = rho != 0.0 ? Hat(k + 1, k) / rho : 0.0;
            Hat(k, k) = rho;
            Hat(k + 1, k) = 0.0;
            g[k + 1] = -sn[k] * g[k];
            g[k] = cs[k] * g[k];
            ++total;
            k_used = k + 1;
            hist.push_back(fabs(g[k + 1]) / r0);
            if (h_next <= 1e-14 * w_norm || h_next == 0.0) {   // krylov.py:130-132
                breakdown = true;
                break;
            }
            if (!lowsync) {
                sc.hval[0] = h_next;
                FD_CUDA(cudaMemcpyAsync(sc.dval, sc.hval, sizeof(double), cudaMemcpyHostToDevice, s));
                launch_scale(N, w, sc.dval, op->V + (long long)(k + 1) * N, s);
            }
            if (hist.back() <= tol) break;
        }
        for (int i = k_used - 1; i >= 0; --i) {   // krylov.py:138-140
            double acc = 0.0;
            for (int j = i + 1; j < k_used; ++j) acc += Hat(i, j) * y[j];
            y[i] = (g[i] - acc) / Hat(i, i);
        }
        FD_CUDA(cudaMemcpyAsync(op->ydev, y.data(), sizeof(double) * k_used, cudaMemcpyHostToDevice, s));
        launch_basis_update(N, k_used, op->V, op->ydev, x, s);   // krylov.py:141
        precond_apply(op, x, w, s);
        launch_axpby(N, 1.0, rhs, -1.0, w, r, s);                // krylov.py:143
        const double rn = norm2(N, r, sc, s);
        const double rel = rn / r0;
        if (rel <= tol || (breakdown && hist.back() <= tol)) {
            hist.back() = rel;
            rep->converged = 1;
            rep->iterations = total;
            rep->restarts = cycles;
            rep->true_residual = rn;
            rep->wall_time = elapsed();
            return FD_OK;
        }
        if (breakdown) break;
    }
    precond_apply(op, x, w, s);
    launch_axpby(N, 1.0, rhs, -1.0, w, r, s);
    rep->converged = 0;
    rep->iterations = total;
    rep->restarts = cycles;
    rep->true_residual = norm2(N, r, sc, s);
    rep->wall_time = elapsed();
    return FD_ERR_NOT_CONVERGED;
}

static void copy_hist(const std::vector<double> &h, double *out, int cap, fd_report *rep) {
    const int n = (int)std::min<size_t>(h.size(), cap > 0 ? (size_t)cap : 0);
    if (out && n > 0) memcpy(out, h.data(), sizeof(double) * n);
    rep->hist_len = (int)h.size();
}

}  // namespace fd

// ===========================================================================
// C ABI
using namespace fd;

#define FD_API_BEGIN try {
#define FD_API_END                                        \
    }                                                     \
    catch (const fd::Error &e) {                          \
        fd::set_error(e.msg);                             \
        return e.code;                                    \
    }                                                     \
    catch (const std::exception &e) {                     \
        fd::set_error(std::string("internal: ") + e.what()); \
        return FD_ERR_CUDA;                               \
    }                                                     \
    return FD_OK;

static cudaStream_t S(void *s) { return (cudaStream_t)s; }

extern "C" {

const char *fd_last_error(void) { return g_last_error.c_str(); }
int fd_version(void) { return 100; }

int fd_plan_create(fd_plan *out, int m, int n, double dx, double dy, double kappa, double mod_west,
                   double mod_east, int device) {
    FD_API_BEGIN
    if (!out) FD_FAIL(FD_ERR_VALIDATION, "null output handle");
    *out = nullptr;
    Plan *p = plan_create(m, n, dx, dy, kappa, mod_west, mod_east, device);
    p->um = m;
    p->un = n;
    *out = new fd_plan_s{p};
    FD_API_END
}

int fd_plan_create_sweep(fd_plan *out, int m, int n, double dx, double dy, double kappa,
                         double mod_west, double mod_east, double mod_south, double mod_north,
                         int transform_axis, int transform_pair, int sweep_cyclic, int pin_mean,
                         int device) {
    FD_API_BEGIN
    if (!out) FD_FAIL(FD_ERR_VALIDATION, "null output handle");
    *out = nullptr;
    if (transform_pair != kPairDD && transform_pair != kPairNN && transform_pair != kPairPP)
        FD_FAIL(FD_ERR_UNSUPPORTED, "transform pair must be DD (0), NN (1) or PP (2)");
    // a DD transform axis must carry ghost-node ends (no half-cell modifier,
    // rectsolver.py:24-29); an NN axis's Neumann ends are part of its basis
    const bool dd = transform_pair == kPairDD;
    const int flags = (sweep_cyclic ? kPlanCyclic : 0) | (pin_mean ? kPlanPinMean : 0);
    Plan *p = nullptr;
    if (transform_axis == 0) {
        if (dd && (mod_south != 0.0 || mod_north != 0.0))
            FD_FAIL(FD_ERR_UNSUPPORTED, "DD transform along y needs ghost-node ends on south/north");
        // a periodic sweep axis has no end modifiers (rectsolver.py:127-134)
        p = plan_create(m, n, dx, dy, kappa, sweep_cyclic ? 0.0 : mod_west, sweep_cyclic ? 0.0 : mod_east,
                        device, transform_pair, flags);
    } else if (transform_axis == 1) {
        if (dd && (mod_west != 0.0 || mod_east != 0.0))
            FD_FAIL(FD_ERR_UNSUPPORTED, "DD transform along x needs ghost-node ends on west/east");
        p = plan_create(n, m, dy, dx, kappa, sweep_cyclic ? 0.0 : mod_south, sweep_cyclic ? 0.0 : mod_north,
                        device, transform_pair, flags);
        p->transposed = true;
    } else {
        FD_FAIL(FD_ERR_VALIDATION, "transform_axis must be 0 (y) or 1 (x)");
    }
    p->um = m;
    p->un = n;
    *out = new fd_plan_s{p};
    FD_API_END
}

int fd_plan_create_ex(fd_plan *out, int m, int n, double dx, double dy, double kappa, double mod_west,
                      double mod_east, double mod_south, double mod_north, int transform_axis,
                      int transform_pair, int device) {
    return fd_plan_create_sweep(out, m, n, dx, dy, kappa, mod_west, mod_east, mod_south, mod_north,
                                transform_axis, transform_pair, 0, 0, device);
}

int fd_plan_singular_modes(fd_plan plan, int *modes, int cap, int *count) {
    FD_API_BEGIN
    if (!plan || !count) FD_FAIL(FD_ERR_VALIDATION, "null argument");
    const auto &sm = plan->p->sing_modes;
    *count = (int)sm.size();
    for (int i = 0; i < (int)sm.size() && i < cap && modes; ++i) modes[i] = sm[i];
    FD_API_END
}

int fd_plan_set_pinv(fd_plan plan, int count, const double *pinv) {
    FD_API_BEGIN
    if (!plan || (count && !pinv)) FD_FAIL(FD_ERR_VALIDATION, "null argument");
    Plan *p = plan->p;
    if (!(p->flags & kPlanPinMean)) FD_FAIL(FD_ERR_VALIDATION, "plan was not created with pin_mean");
    if (count != p->dev.nsing) FD_FAIL(FD_ERR_VALIDATION, "pseudo-inverse count != singular modes");
    if (!count) return FD_OK;
    const int m = p->dev.m;
    std::vector<double> t(size_t(count) * m * m);   // transposed per mode: [j][i]
    for (int c = 0; c < count; ++c)
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j)
                t[(size_t(c) * m + j) * m + i] = pinv[(size_t(c) * m + i) * m + j];
    FD_CUDA(cudaSetDevice(p->device));
    double *d = static_cast<double *>(dmalloc(sizeof(double) * t.size()));
    p->allocs.push_back(d);
    FD_CUDA(cudaMemcpy(d, t.data(), sizeof(double) * t.size(), cudaMemcpyHostToDevice));
    p->dev.pinv = d;
    p->pinv_ready = true;
    FD_API_END
}

int fd_plan_create_axis(fd_plan *out, int m, int n, double dx, double dy, double kappa,
                        double mod_west, double mod_east, double mod_south, double mod_north,
                        int transform_axis, int device) {
    return fd_plan_create_ex(out, m, n, dx, dy, kappa, mod_west, mod_east, mod_south, mod_north,
                             transform_axis, kPairDD, device);
}

int fd_transform_kind_pair(int n, int pair) { return transform_kind(n, pair); }

int fd_transform_kind(int n) { return transform_kind(n); }

int fd_plan_destroy(fd_plan plan) {
    FD_API_BEGIN
    if (plan) {
        plan_destroy(plan->p);
        delete plan;
    }
    FD_API_END
}

int fd_plan_info(fd_plan plan, int *block_rows, long long *explicit_rows, int *transform) {
    FD_API_BEGIN
    if (!plan) FD_FAIL(FD_ERR_VALIDATION, "null plan");
    if (block_rows) *block_rows = plan->p->dev.R;
    if (explicit_rows) *explicit_rows = plan->p->explicit_rows;
    if (transform) *transform = plan->p->transform;
    FD_API_END
}

int fd_factor_tables_host(int m, int n, double dx, double dy, double kappa, double mod_west,
                          double mod_east, double *beta, double *lower) {
    FD_API_BEGIN
    factor_tables_host(m, n, dx, dy, kappa, mod_west, mod_east, beta, lower);
    FD_API_END
}

int fd_rect_solve(fd_plan plan, const double *f, double *out, void *stream) {
    FD_API_BEGIN
    if (!plan || !f || !out) FD_FAIL(FD_ERR_VALIDATION, "null argument");
    solve_user({UJob{plan->p, f, out}}, S(stream));
    FD_API_END
}

int fd_rect_solve_batched(int count, const fd_plan *plans, const double *const *f, double *const *out,
                          void *stream) {
    FD_API_BEGIN
    NvtxRange nvtx("fd:rect_solve_batched");
    std::vector<UJob> jobs;
    for (int i = 0; i < count; ++i) {
        if (!plans[i] || !f[i] || !out[i]) FD_FAIL(FD_ERR_VALIDATION, "null argument");
        jobs.push_back(UJob{plans[i]->p, f[i], out[i]});
    }
    solve_user(jobs, S(stream));
    FD_API_END
}

int fd_dst_rows(int rows, int n, const double *in, double *out, int device, void *stream) {
    FD_API_BEGIN
    if (transform_kind(n) < 0) FD_FAIL(FD_ERR_UNSUPPORTED, "no GPU transform for this length");
    FD_CUDA(cudaSetDevice(device));
    launch_dst_rows(rows, n, in, out, twiddles_for(device, n), dense_table_for(device, n), S(stream));
    FD_API_END
}

int fd_transform_rows(int rows, int n, int pair, int inverse, const double *in, double *out, int device,
                      void *stream) {
    FD_API_BEGIN
    if (rows < 0 || n < 1 || !in || !out) FD_FAIL(FD_ERR_VALIDATION, "bad transform arguments");
    if (pair != kPairDD && pair != kPairNN && pair != kPairPP) FD_FAIL(FD_ERR_UNSUPPORTED, "unknown transform pair");
    const int tk = transform_kind(n, pair);
    if (tk < 0) FD_FAIL(FD_ERR_UNSUPPORTED, "no GPU transform for this length and pair");
    FD_CUDA(cudaSetDevice(device));
    if (tk == kFFT)   // DD: Q = Q^T
        launch_dst_rows(rows, n, in, out, twiddles_for(device, n), nullptr, S(stream));
    else
        launch_transform_rows(rows, n, pair, inverse, in, out, dense_table_for(device, n, pair), S(stream));
    FD_API_END
}

int fd_assemble_rhs(int m, int n, double x0, double y0, double dx, double dy, double kappa, int solution,
                    double lift_west, double lift_east, double lift_south, double lift_north, double *f,
                    double *exact, void *stream) {
    FD_API_BEGIN
    if (m < 1 || n < 1 || !f || (solution != 0 && solution != 1)) FD_FAIL(FD_ERR_VALIDATION, "bad assembly arguments");
    const double lift[4] = {lift_west, lift_east, lift_south, lift_north};
    launch_assemble(m, n, x0, y0, dx, dy, kappa, solution, lift, f, exact, S(stream));
    FD_API_END
}

int fd_stencil_apply(int m, int n, double delta_x, double delta_y, double kappa, double mod_west,
                     double mod_east, double mod_south, double mod_north, const double *v,
                     double *out, void *stream) {
    FD_API_BEGIN
    if (m < 1 || n < 1 || !v || !out) FD_FAIL(FD_ERR_VALIDATION, "bad stencil arguments");
    launch_stencil(m, n, delta_x, delta_y, kappa, mod_west, mod_east, mod_south, mod_north, v, out,
                   S(stream));
    FD_API_END
}

int fd_stencil_apply_ex(int m, int n, double delta_x, double delta_y, double kappa, double mod_west,
                        double mod_east, double mod_south, double mod_north, int periodic_x,
                        int periodic_y, const double *v, double *out, void *stream) {
    FD_API_BEGIN
    if (m < 1 || n < 1 || !v || !out) FD_FAIL(FD_ERR_VALIDATION, "bad stencil arguments");
    launch_stencil(m, n, delta_x, delta_y, kappa, mod_west, mod_east, mod_south, mod_north, v, out,
                   S(stream), periodic_x, periodic_y);
    FD_API_END
}

int fd_schur_create(fd_schur *out, fd_plan center, double center_mod_south, double center_mod_north,
                    int n_nb, const fd_plan *nb, const int *line_len,
                    const int64_t *const *to_c_from, const int64_t *const *to_c_to,
                    const double *to_c_coupling, const int64_t *const *from_c_from,
                    const int64_t *const *from_c_to, const double *from_c_coupling) {
    FD_API_BEGIN
    if (!out || !center) FD_FAIL(FD_ERR_VALIDATION, "null argument");
    *out = nullptr;
    fd_schur_s *op = new fd_schur_s();
    try {
        op->device = center->p->device;
        FD_CUDA(cudaSetDevice(op->device));
        op->center = center->p;
        op->mod_s = center_mod_south;
        op->mod_n = center_mod_north;
        const long long Nc = (long long)center->p->m * center->p->n;
        for (int i = 0; i < n_nb; ++i) {
            Plan *q = nb[i]->p;
            op->nb.push_back(q);
            auto up = [&](const int64_t *h, int len) {
                int64_t *d = (int64_t *)dalloc(op, sizeof(int64_t) * std::max(len, 1));
                FD_CUDA(cudaMemcpy(d, h, sizeof(int64_t) * len, cudaMemcpyHostToDevice));
                return d;
            };
            const int len = line_len[i];
            // neighbour-side indices in the plan's internal layout (transposed axis)
            auto internal = [&](const int64_t *h) {
                std::vector<int64_t> v(h, h + len);
                if (q->transposed)
                    for (auto &x : v) x = (x % q->un) * q->um + x / q->un;
                return v;
            };
            const std::vector<int64_t> tcf = internal(to_c_from[i]), fct = internal(from_c_to[i]);
            int64_t *tcf_user = up(to_c_from[i], len);
            op->to_c.push_back(Coupling{len, q->transposed ? up(tcf.data(), len) : tcf_user, up(to_c_to[i], len),
                                        to_c_coupling[i], tcf_user});
            op->from_c.push_back(Coupling{len, up(from_c_from[i], len), up(fct.data(), len),
                                          from_c_coupling[i], nullptr});
            op->nbf.push_back((double *)dalloc(op, sizeof(double) * q->m * q->n));
            op->nbin.push_back((double *)dalloc(op, sizeof(double) * q->m * q->n));
            FD_CUDA(cudaMemset(op->nbin.back(), 0, sizeof(double) * q->m * q->n));
        }
        {   // at most two R_ci contributions per centre entry: one atomic scatter-add
            std::unordered_map<int64_t, int> mult;
            int mx = 0;
            for (int i = 0; i < n_nb; ++i)
                for (int t = 0; t < line_len[i]; ++t) mx = std::max(mx, ++mult[to_c_to[i][t]]);
            op->fused_add = n_nb <= kMaxScatter && mx <= 2;
        }
        op->tmp = (double *)dalloc(op, sizeof(double) * Nc);
        FD_CUDA(cudaMemset(op->tmp, 0, sizeof(double) * Nc));
        op->tmp2 = (double *)dalloc(op, sizeof(double) * Nc);
        op->w = (double *)dalloc(op, sizeof(double) * Nc);
        op->r = (double *)dalloc(op, sizeof(double) * Nc);
        op->sc = make_scratch(128);
    } catch (...) {
        cudaDeviceSynchronize();
        for (void *a : op->allocs) dfree(a);
        delete op;
        throw;
    }
    *out = op;
    FD_API_END
}

int fd_schur_set_stencil(fd_schur op, int m, int n, double delta_x, double delta_y, double kappa, double mod_west,
                         double mod_east, double mod_south, double mod_north, int periodic_x, int periodic_y) {
    FD_API_BEGIN
    if (!op) FD_FAIL(FD_ERR_VALIDATION, "null operator");
    if ((long long)m * n != (long long)op->center->m * op->center->n)
        FD_FAIL(FD_ERR_VALIDATION, "stencil grid does not match the centre plan");
    auto &t = op->stencil;
    t.m = m;
    t.n = n;
    t.dx = delta_x;
    t.dy = delta_y;
    t.kappa = kappa;
    t.mw = mod_west;
    t.me = mod_east;
    t.ms = mod_south;
    t.mn = mod_north;
    t.px = periodic_x;
    t.py = periodic_y;
    op->stencil_set = true;
    FD_API_END
}

int fd_schur_set_steklov(fd_schur op, int i, int line_len, int sweep_len, double delta_line,
                         double delta_sweep, double kappa, double mod_lo, double mod_hi, int end,
                         const int64_t *pos_in, const int64_t *pos_out) {
    FD_API_BEGIN
    if (!op || i < 0 || i >= (int)op->nb.size()) FD_FAIL(FD_ERR_VALIDATION, "steklov: bad neighbour index");
    if (line_len < 1 || sweep_len < 1 || (end != 0 && end != 1)) FD_FAIL(FD_ERR_VALIDATION, "steklov: bad line");
    if (transform_kind(line_len) < 0) FD_FAIL(FD_ERR_UNSUPPORTED, "steklov: no GPU transform for the line length");
    FD_CUDA(cudaSetDevice(op->device));
    if (op->stk.size() != op->nb.size()) op->stk.resize(op->nb.size());
    auto &k = op->stk[i];
    k.L = line_len;
    const int len = op->from_c[i].len;
    std::vector<double> inv(line_len);
    steklov_pivots(line_len, sweep_len, delta_line, delta_sweep, kappa, mod_lo, mod_hi, end, inv.data());
    k.invpiv = (double *)dalloc(op, sizeof(double) * line_len);
    FD_CUDA(cudaMemcpy(k.invpiv, inv.data(), sizeof(double) * line_len, cudaMemcpyHostToDevice));
    k.pos_in = (int64_t *)dalloc(op, sizeof(int64_t) * std::max(len, 1));
    k.pos_out = (int64_t *)dalloc(op, sizeof(int64_t) * std::max(op->to_c[i].len, 1));
    FD_CUDA(cudaMemcpy(k.pos_in, pos_in, sizeof(int64_t) * len, cudaMemcpyHostToDevice));
    FD_CUDA(cudaMemcpy(k.pos_out, pos_out, sizeof(int64_t) * op->to_c[i].len, cudaMemcpyHostToDevice));
    FD_API_END
}

int fd_schur_use_steklov(fd_schur op, int enable) {
    FD_API_BEGIN
    if (!op) FD_FAIL(FD_ERR_VALIDATION, "null operator");
    if (!enable) {
        op->steklov = false;
    } else {
        if (op->stk.size() != op->nb.size() || op->nb.empty())
            FD_FAIL(FD_ERR_VALIDATION, "steklov: describe every neighbour first");
        for (auto &k : op->stk)
            if (!k.invpiv || k.L != op->stk[0].L)
                FD_FAIL(FD_ERR_UNSUPPORTED, "steklov: every neighbour needs a described line of one length");
        if (!op->lines) {
            op->lines = (double *)dalloc(op, sizeof(double) * op->nb.size() * op->stk[0].L);
            op->lines_hat = (double *)dalloc(op, sizeof(double) * op->nb.size() * op->stk[0].L);
        }
        op->steklov = true;
    }
    drop_graph(op);   // the captured apply no longer matches
    FD_API_END
}

int fd_schur_destroy(fd_schur op) {
    FD_API_BEGIN
    if (op) {
        HostTimer ht("schur_destroy");
        cudaSetDevice(op->device);
        cudaDeviceSynchronize();
        drop_graph(op);
        if (op->gstream) cudaStreamDestroy(op->gstream);
        for (void *a : op->allocs) dfree(a);
        if (op->V) dfree(op->V);
        if (op->ydev) dfree(op->ydev);
        if (op->sc.cap) free_scratch(op->sc);
        pinned_put(op->arn_host);
        for (auto e : op->arn_ev)
            if (e) cudaEventDestroy(e);
        delete op;
        ht.mark("done", 0, false);
    }
    FD_API_END
}

int fd_schur_apply(fd_schur op, const double *p, double *out, void *stream) {
    FD_API_BEGIN
    schur_apply(op, p, out, S(stream));
    FD_API_END
}

int fd_center_solve(fd_schur op, const double *r, double *out, void *stream) {
    FD_API_BEGIN
    center_solve(op, r, out, 1.0, 0.0, nullptr, S(stream));
    FD_API_END
}

int fd_precond_apply(fd_schur op, const double *p, double *out, void *stream) {
    FD_API_BEGIN
    NvtxRange nvtx("fd:precond_apply");
    precond_apply(op, p, out, S(stream));
    FD_API_END
}

int fd_unprecond_apply(fd_schur op, const double *p, double *out, void *stream) {
    FD_API_BEGIN
    unprecond_apply(op, p, out, S(stream));
    FD_API_END
}

int fd_gmres_precond(fd_schur op, const double *rhs, double *x, int x_is_zero, int m, double tol,
                     int max_restarts, double *history, int hist_cap, fd_report *rep,
                     void *stream) {
    FD_API_BEGIN
    if (!op || !rhs || !x || !rep) FD_FAIL(FD_ERR_VALIDATION, "null argument");
    if (m < 1 || !(tol > 0) || max_restarts < 1) FD_FAIL(FD_ERR_VALIDATION, "bad GMRES config");
    std::vector<double> hist;
    const int st = gmres_precond(op, rhs, x, x_is_zero, m, tol, max_restarts, hist, rep, S(stream));
    copy_hist(hist, history, hist_cap, rep);
    if (st != FD_OK) {
        std::ostringstream os;
        os << "GMRES did not reach tol=" << tol << " in " << rep->iterations << " iterations";
        FD_FAIL(st, os.str());
    }
    FD_API_END
}

int fd_ddm_solve(fd_schur op, const double *f_center, const double *const *f_nb, double *p_center,
                 double *const *p_nb, int m, double tol, int max_restarts, double *history,
                 int hist_cap, fd_report *rep, void *stream) {
    FD_API_BEGIN
    if (!op || !f_center || !p_center || !rep) FD_FAIL(FD_ERR_VALIDATION, "null argument");
    if (m < 1 || !(tol > 0) || max_restarts < 1) FD_FAIL(FD_ERR_VALIDATION, "bad GMRES config");
    cudaStream_t s = S(stream);
    HostTimer ht("ddm_solve");
    ht.mark("entry", s, false);
    NvtxRange nvtx_solve("fd:ddm_solve");
    nvtxRangePushA("fd:presolves");
    const size_t nnb = op->nb.size();
    const long long Nc = (long long)op->center->m * op->center->n;
    // pre-solves q_i = A_i^{-1} f_i into the caller's output fields (ddm.py:249-250)
    std::vector<UJob> ujobs;
    for (size_t i = 0; i < nnb; ++i) ujobs.push_back(UJob{op->nb[i], f_nb[i], p_nb[i]});
    solve_user(ujobs, s);
    // f' = f_c - sum_i R_ci q_i  (ddm.py:252-254) in a buffer of its own:
    // unprecond_apply (the true residual below) uses tmp2 as scratch
    double *fp = nullptr;
    FD_CUDA(cudaMallocAsync(&fp, sizeof(double) * Nc, s));
    FD_CUDA(cudaMemcpyAsync(fp, f_center, sizeof(double) * Nc, cudaMemcpyDeviceToDevice, s));
    for (size_t i = 0; i < nnb; ++i) {
        const Coupling &c = op->to_c[i];
        // fp[to] = fp[to] - c * q[from]
        launch_scatter(c.len, c.from_user, c.to, -c.c, p_nb[i], fp, 1, s);
    }
    // solve_coupled fft branch: rhs = A_c^{-1} f'; GMRES on the preconditioned system
    // (krylov.py:176-187); fp must survive, so rhs goes to a fresh buffer
    double *rhs = nullptr;
    FD_CUDA(cudaMallocAsync(&rhs, sizeof(double) * Nc, s));
    center_solve(op, fp, rhs, 1.0, 0.0, nullptr, s);
    ht.mark("presolves+rhs", s);
    nvtxRangePop();
    std::vector<double> hist;
    int st;
    {
        NvtxRange nvtx_gmres("fd:gmres");
        st = gmres_precond(op, rhs, p_center, 1, m, tol, max_restarts, hist, rep, s);
    }
    ht.mark("gmres", s);
    NvtxRange nvtx_back("fd:residual+backsub");
    copy_hist(hist, history, hist_cap, rep);
    // true residual ||(A_c - S) x - f'|| (krylov.py:189); rhs buffer reused
    unprecond_apply(op, p_center, rhs, s);
    launch_axpby(Nc, 1.0, rhs, -1.0, fp, rhs, s);
    rep->true_residual = norm2(Nc, rhs, op->sc, s);
    FD_CUDA(cudaFreeAsync(rhs, s));
    FD_CUDA(cudaFreeAsync(fp, s));
    // back-substitution p_i = q_i - A_i^{-1} R_ic p_c (ddm.py:259-269)
    std::vector<SolveJob> jobs;
    for (size_t i = 0; i < nnb; ++i) {
        const Plan *q = op->nb[i];
        const Coupling &c = op->from_c[i];
        launch_scatter(c.len, c.from, c.to, c.c, p_center, op->nbin[i], 0, s);
        jobs.push_back(job_of(q, op->nbin[i], op->nbf[i]));
    }
    solve_batch(jobs, s);
    for (size_t i = 0; i < nnb; ++i) launch_zero_at(op->from_c[i].len, op->from_c[i].to, op->nbin[i], s);
    for (size_t i = 0; i < nnb; ++i) {
        const Plan *q = op->nb[i];
        if (q->transposed)
            launch_transpose(q->m, q->n, op->nbf[i], p_nb[i], -1.0, 1.0, p_nb[i], s);
        else
            launch_axpby((long long)q->m * q->n, 1.0, p_nb[i], -1.0, op->nbf[i], p_nb[i], s);
    }
    ht.mark("residual+backsub", s);
    if (st != FD_OK) {
        std::ostringstream os;
        os << "GMRES did not reach tol=" << tol << " in " << rep->iterations << " iterations";
        FD_FAIL(st, os.str());
    }
    FD_API_END
}

int fd_schur_set_comm(fd_schur op, fd_comm comm, const int *owner) {
    FD_API_BEGIN
    if (!op || !comm || !owner) FD_FAIL(FD_ERR_VALIDATION, "null argument");
    const int nr = comm->t->nranks;
    FD_CUDA(cudaSetDevice(op->device));
    op->owner.assign(owner, owner + op->nb.size());
    for (int o : op->owner)
        if (o < 0 || o >= nr) FD_FAIL(FD_ERR_VALIDATION, "arm owner outside the communicator");
    int lmax = 1;
    for (size_t i = 0; i < op->nb.size(); ++i) lmax = std::max(lmax, std::max(op->from_c[i].len, op->to_c[i].len));
    if (!op->iota) {
        std::vector<int64_t> h(lmax);
        for (int t = 0; t < lmax; ++t) h[t] = t;
        op->iota = (int64_t *)dalloc(op, sizeof(int64_t) * lmax);
        FD_CUDA(cudaMemcpy(op->iota, h.data(), sizeof(int64_t) * lmax, cudaMemcpyHostToDevice));
        for (size_t i = 0; i < op->nb.size(); ++i) {
            op->sline.push_back((double *)dalloc(op, sizeof(double) * lmax));
            op->rline.push_back((double *)dalloc(op, sizeof(double) * lmax));
        }
        op->cmd = (long long *)dalloc(op, sizeof(long long));
        op->cmd_host = (long long *)pinned_get(sizeof(long long));
    }
    op->comm = comm;
    drop_graph(op);
    FD_API_END
}

// Algorithm 1 sharded over the communicator's ranks: rank 0 owns
// the centre, runs GMRES and drives every operator application; an arm owner
// pre-solves its arms, then serves commands (apply: solve the received R_ic
// line and return R_ci of the result; back-substitution: finish its fields).
// Arguments as fd_ddm_solve; on rank r only the owned arms' f_nb / p_nb (and
// on rank 0 f_center / p_center) are read or written.
int fd_ddm_solve_dist(fd_schur op, const double *f_center, const double *const *f_nb, double *p_center,
                      double *const *p_nb, int m, double tol, int max_restarts, double *history, int hist_cap,
                      fd_report *rep, void *stream) {
    FD_API_BEGIN
    if (!op || !rep || !op->comm) FD_FAIL(FD_ERR_VALIDATION, "sharded solve: operator without communicator");
    cudaStream_t s = S(stream);
    Transport &t = *op->comm->t;
    const int rank = t.rank;
    const size_t nnb = op->nb.size();
    memset(rep, 0, sizeof(*rep));
    // pre-solves q_i = A_i^{-1} f_i of the owned arms (ddm.py:249-250)
    std::vector<UJob> ujobs;
    for (size_t i = 0; i < nnb; ++i)
        if (!op->remote(i)) {
            if (!f_nb[i] || !p_nb[i]) FD_FAIL(FD_ERR_VALIDATION, "sharded solve: owned arm without fields");
            ujobs.push_back(UJob{op->nb[i], f_nb[i], p_nb[i]});
        }
    solve_user(ujobs, s);
    if (rank != 0) {
        // R_ci q_i lines to rank 0, then serve commands
        t.group_start();
        for (size_t i = 0; i < nnb; ++i)
            if (!op->remote(i)) {
                const Coupling &c = op->to_c[i];
                launch_scatter(c.len, c.from_user, op->iota, c.c, p_nb[i], op->sline[i], 0, s);
                t.send(op->sline[i], sizeof(double) * c.len, 0, s);
            }
        t.group_end();
        for (;;) {
            t.recv(op->cmd, sizeof(long long), 0, s);
            FD_CUDA(cudaMemcpyAsync(op->cmd_host, op->cmd, sizeof(long long), cudaMemcpyDeviceToHost, s));
            FD_CUDA(cudaStreamSynchronize(s));
            const long long cmd = *op->cmd_host;
            if (cmd == kCmdDone) break;
            std::vector<SolveJob> jobs;
            t.group_start();
            for (size_t i = 0; i < nnb; ++i)
                if (!op->remote(i)) t.recv(op->rline[i], sizeof(double) * op->from_c[i].len, 0, s);
            t.group_end();
            for (size_t i = 0; i < nnb; ++i)
                if (!op->remote(i)) {
                    const Coupling &c = op->from_c[i];
                    launch_scatter(c.len, op->iota, c.to, 1.0, op->rline[i], op->nbin[i], 0, s);
                    jobs.push_back(job_of(op->nb[i], op->nbin[i], op->nbf[i]));
                }
            solve_batch(jobs, s);
            for (size_t i = 0; i < nnb; ++i)
                if (!op->remote(i)) launch_zero_at(op->from_c[i].len, op->from_c[i].to, op->nbin[i], s);
            if (cmd == kCmdApply) {
                t.group_start();
                for (size_t i = 0; i < nnb; ++i)
                    if (!op->remote(i)) {
                        const Coupling &c = op->to_c[i];
                        launch_scatter(c.len, c.from, op->iota, c.c, op->nbf[i], op->sline[i], 0, s);
                        t.send(op->sline[i], sizeof(double) * c.len, 0, s);
                    }
                t.group_end();
            } else {   // back-substitution p_i = q_i - A_i^{-1} R_ic p_c (ddm.py:259-269)
                for (size_t i = 0; i < nnb; ++i) {
                    if (op->remote(i)) continue;
                    const Plan *q = op->nb[i];
                    if (q->transposed)
                        launch_transpose(q->m, q->n, op->nbf[i], p_nb[i], -1.0, 1.0, p_nb[i], s);
                    else
                        launch_axpby((long long)q->m * q->n, 1.0, p_nb[i], -1.0, op->nbf[i], p_nb[i], s);
                }
            }
        }
        FD_CUDA(cudaStreamSynchronize(s));
        return FD_OK;
    }
    // ---- rank 0
    if (!f_center || !p_center) FD_FAIL(FD_ERR_VALIDATION, "sharded solve: rank 0 needs the centre fields");
    const long long Nc = (long long)op->center->m * op->center->n;
    int st = FD_OK;
    std::string err;
    double *fp = nullptr, *rhs = nullptr;
    bool done_sent = false;
    try {
        FD_CUDA(cudaMallocAsync(&fp, sizeof(double) * Nc, s));
        FD_CUDA(cudaMallocAsync(&rhs, sizeof(double) * Nc, s));
        FD_CUDA(cudaMemcpyAsync(fp, f_center, sizeof(double) * Nc, cudaMemcpyDeviceToDevice, s));
        t.group_start();
        for (size_t i = 0; i < nnb; ++i)
            if (op->remote(i)) t.recv(op->rline[i], sizeof(double) * op->to_c[i].len, op->owner[i], s);
        t.group_end();
        for (size_t i = 0; i < nnb; ++i) {   // f' = f_c - sum_i R_ci q_i, neighbour order (ddm.py:252-254)
            const Coupling &c = op->to_c[i];
            if (op->remote(i)) launch_scatter(c.len, op->iota, c.to, -1.0, op->rline[i], fp, 1, s);
            else launch_scatter(c.len, c.from_user, c.to, -c.c, p_nb[i], fp, 1, s);
        }
        center_solve(op, fp, rhs, 1.0, 0.0, nullptr, s);
        std::vector<double> hist;
        st = gmres_precond(op, rhs, p_center, 1, m, tol, max_restarts, hist, rep, s);
        copy_hist(hist, history, hist_cap, rep);
        unprecond_apply(op, p_center, rhs, s);   // true residual ||(A_c - S) x - f'|| (krylov.py:189)
        launch_axpby(Nc, 1.0, rhs, -1.0, fp, rhs, s);
        rep->true_residual = norm2(Nc, rhs, op->sc, s);
        // back-substitution: remote arms by their owners, local arms here
        send_command(op, kCmdBacksub, s);
        send_lines(op, p_center, s);
        std::vector<SolveJob> jobs;
        for (size_t i = 0; i < nnb; ++i) {
            if (op->remote(i)) continue;
            const Coupling &c = op->from_c[i];
            launch_scatter(c.len, c.from, c.to, c.c, p_center, op->nbin[i], 0, s);
            jobs.push_back(job_of(op->nb[i], op->nbin[i], op->nbf[i]));
        }
        if (!jobs.empty()) solve_batch(jobs, s);
        for (size_t i = 0; i < nnb; ++i) {
            if (op->remote(i)) continue;
            launch_zero_at(op->from_c[i].len, op->from_c[i].to, op->nbin[i], s);
            const Plan *q = op->nb[i];
            if (q->transposed)
                launch_transpose(q->m, q->n, op->nbf[i], p_nb[i], -1.0, 1.0, p_nb[i], s);
            else
                launch_axpby((long long)q->m * q->n, 1.0, p_nb[i], -1.0, op->nbf[i], p_nb[i], s);
        }
        send_command(op, kCmdDone, s);
        done_sent = true;
    } catch (const Error &e) {
        st = e.code;
        err = e.msg;
    }
    if (!done_sent) {   // release the arm owners whatever happened here
        try {
            send_command(op, kCmdDone, s);
        } catch (...) {
        }
    }
    if (fp) cudaFreeAsync(fp, s);
    if (rhs) cudaFreeAsync(rhs, s);
    if (!err.empty()) FD_FAIL(st, err);
    if (st != FD_OK) {
        std::ostringstream os;
        os << "GMRES did not reach tol=" << tol << " in " << rep->iterations << " iterations";
        FD_FAIL(st, os.str());
    }
    FD_API_END
}

int fd_arnoldi_step(int N, int k, const double *V, double *w, double *h, double *w_norm,
                    void *stream) {
    FD_API_BEGIN
    if (k < 0) FD_FAIL(FD_ERR_VALIDATION, "arnoldi: negative step");
    arnoldi_step(N, k, V, w, h, w_norm, device_scratch(S(stream), k + 3), S(stream));
    FD_API_END
}

int fd_basis_update(int N, int k, const double *V, const double *y, double *x, void *stream) {
    FD_API_BEGIN
    if (k < 0) FD_FAIL(FD_ERR_VALIDATION, "basis update: negative k");
    Scratch &sc = device_scratch(S(stream), k);
    memcpy(sc.hval, y, sizeof(double) * k);
    FD_CUDA(cudaMemcpyAsync(sc.dval, sc.hval, sizeof(double) * k, cudaMemcpyHostToDevice, S(stream)));
    launch_basis_update(N, k, V, sc.dval, x, S(stream));
    FD_CUDA(cudaStreamSynchronize(S(stream)));
    FD_API_END
}

int fd_axpby(int N, double a, const double *x, double b, const double *y, double *out, void *stream) {
    FD_API_BEGIN
    launch_axpby(N, a, x, b, y, out, S(stream));
    FD_API_END
}

int fd_norm(int N, const double *x, double *result, void *stream) {
    FD_API_BEGIN
    *result = norm2(N, x, device_scratch(S(stream)), S(stream));
    FD_API_END
}

int fd_dot(int N, const double *x, const double *y, double *result, void *stream) {
    FD_API_BEGIN
    Scratch &sc = device_scratch(S(stream));
    launch_dot(N, x, y, sc.dval, sc.red, S(stream));
    FD_CUDA(cudaMemcpyAsync(sc.hval, sc.dval, sizeof(double), cudaMemcpyDeviceToHost, S(stream)));
    FD_CUDA(cudaStreamSynchronize(S(stream)));
    *result = sc.hval[0];
    FD_API_END
}

}  // extern "C"
