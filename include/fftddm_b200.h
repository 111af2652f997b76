/*
 * fftddm_b200.h -- C ABI of the B200-native hot path of the FFT-preconditioned
 * Schur/GMRES solver (arXiv 2509.23180, reference package `fftddm`).
 *
 * Plain C types only: sizes are ints, fields are fp64 DEVICE pointers in the
 * x-line-major layout of the reference (node (i,j) at (i-1)*n + (j-1),
 * fftddm/geometry.py:3-8,142-148), streams are `cudaStream_t` passed as void*.
 * Every entry point returns an FD_* status; on failure fd_last_error() holds a
 * thread-local message.  The Python shim (paper_2509_23180_b200/_native.py)
 * maps the codes onto the reference's exception classes
 * (fftddm/errors.py:1-24).
 *
 * Ownership: the caller owns every field buffer it passes; the library owns the
 * opaque handles (plans, Schur operators, GMRES workspace incl. the Krylov
 * basis) from *_create to *_destroy.  No hidden host<->device copies happen in
 * the solve/apply calls.  One handle is used by one stream at a time.
 */
#ifndef FFTDDM_B200_H
#define FFTDDM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* status codes ------------------------------------------------------------- */
#define FD_OK 0
#define FD_ERR_VALIDATION 1     /* ValidationError / ValueError (shape, ids)   */
#define FD_ERR_SINGULAR 2       /* SingularOperatorError (rectsolver.py:156-163) */
#define FD_ERR_NOT_CONVERGED 3  /* ConvergenceError (krylov.py:156-165)         */
#define FD_ERR_CUDA 4           /* CUDA runtime failure                        */
#define FD_ERR_UNSUPPORTED 5    /* outside the GPU path's scope (NN/PP axes)   */

typedef struct fd_plan_s *fd_plan;
typedef struct fd_schur_s *fd_schur;
typedef struct fd_comm_s *fd_comm;

/* GMRES report; replaces krylov.SolveReport (krylov.py:52-58). */
typedef struct {
    int converged;
    int iterations;
    int restarts;          /* restart cycles run                               */
    int hist_len;          /* entries written to the caller's history buffer   */
    double wall_time;      /* seconds, host clock around the device loop       */
    double true_residual;  /* ||rhs - op(x)||, or the solve_coupled residual   */
} fd_report;

const char *fd_last_error(void);
int fd_version(void);

/* --- rectangle plan: replaces rectsolver.plan_rect (rectsolver.py:94-180) ---
 * DD transform along y (the contiguous axis), per-end diagonal modifiers on
 * the sweep axis (end_modifier west/east, geometry.py:118-128).  Builds the
 * eigenvalues (transforms.py:26-31), the per-mode LU of the sweep system with
 * the reference's recurrence (rectsolver.py:62-77) and the block-carry tables
 * of the two-pass Thomas solve.  FD_ERR_SINGULAR on a zero pivot. */
int fd_plan_create(fd_plan *out, int m, int n, double dx, double dy, double kappa,
                   double mod_west, double mod_east, int device);
/* Same with the transform axis chosen by the caller (reference
 * rectsolver.plan_rect, rectsolver.py:102-123): transform_axis 0 = y (as
 * fd_plan_create; south/north must be ghost-node ends), 1 = x (west/east must
 * be ghost-node ends; the sweep runs along y with the south/north modifiers).
 * Fields passed to the solves stay in the user's x-line-major layout; an
 * x-axis plan transposes them on the device around the fused solve
 * (rectsolver.py:198-199,211-212). */
int fd_plan_create_axis(fd_plan *out, int m, int n, double dx, double dy, double kappa,
                        double mod_west, double mod_east, double mod_south, double mod_north,
                        int transform_axis, int device);
/* General form: transform_pair 0 = DD (sine basis, DST-I), 1 = NN (shifted
 * cosine basis, DCT-II/III; transforms.py:32-33,83-98,106-134), 2 = PP (real
 * Fourier basis, even n; transforms.py:34-35,114-126,139-148).  A DD axis
 * needs ghost-node ends; NN/PP ends belong to the basis.  NN and PP run on
 * the dense periodic-table transform (n <= 2048); a periodic sweep axis
 * needs fd_plan_create_sweep. */
int fd_plan_create_ex(fd_plan *out, int m, int n, double dx, double dy, double kappa,
                      double mod_west, double mod_east, double mod_south, double mod_north,
                      int transform_axis, int transform_pair, int device);
/* Full plan_rect (rectsolver.py:94-180): as fd_plan_create_ex plus
 *  - sweep_cyclic: the sweep axis is periodic (PP, even count).  The per-mode
 *    system is solved as the reference does -- Thomas on the rank-one modified
 *    matrix, then the Sherman-Morrison correction (rectsolver.py:136-153,
 *    202-205); with two rows the wrap doubles the coupling.  End modifiers of
 *    the sweep axis are ignored.
 *  - pin_mean: singular spectral modes (all-Neumann / periodic, kappa = 0) do
 *    not fail the plan; they are solved in the minimum-norm sense
 *    (rectsolver.py:157-175,206-207).  The caller lists them with
 *    fd_plan_singular_modes and attaches each mode's sweep-matrix
 *    pseudo-inverse with fd_plan_set_pinv before the first solve (a solve
 *    before that returns FD_ERR_SINGULAR).
 * Periodic-sweep and pin_mean plans run the dense-transform solve (n <= 2048). */
int fd_plan_create_sweep(fd_plan *out, int m, int n, double dx, double dy, double kappa,
                         double mod_west, double mod_east, double mod_south, double mod_north,
                         int transform_axis, int transform_pair, int sweep_cyclic, int pin_mean,
                         int device);
/* singular spectral modes of a pin_mean plan (indices along the transform
 * axis, ascending); *count receives the total, at most cap are written. */
int fd_plan_singular_modes(fd_plan plan, int *modes, int cap, int *count);
/* attach the pseudo-inverses of the singular modes' sweep matrices, host
 * memory, count x ms x ms row-major (ms = sweep length: m for a y transform,
 * n for an x transform), in fd_plan_singular_modes order. */
int fd_plan_set_pinv(fd_plan plan, int count, const double *pinv);
/* GPU transform for length n: 1 = fused real-symmetric FFT solve (DD,
 * n+1 = 2^p in 256..4096), 0 = dense periodic table (n <= 2048), 2 = any-length
 * mixed-radix / Bluestein passes + separate sweeps (n <= 65535), -1 = none
 * (PP with odd n).  DD pair; fd_transform_kind_pair for NN (1) / PP (2). */
int fd_transform_kind(int n);
int fd_transform_kind_pair(int n, int pair);
int fd_plan_destroy(fd_plan plan);
/* rows per carry block, explicit factor rows, transform kind (0 dense, 1 fft) */
int fd_plan_info(fd_plan plan, int *block_rows, long long *explicit_rows, int *transform);

/* Host-only restatement of the factor tables for testing without a GPU:
 * writes the full (m, n) beta and lower arrays rebuilt from the compressed
 * per-mode tables the device uses. */
int fd_factor_tables_host(int m, int n, double dx, double dy, double kappa,
                          double mod_west, double mod_east, double *beta, double *lower);

/* --- rectangle solve: replaces rectsolver.solve_rect (rectsolver.py:183-213)
 * out = A^{-1} f.  f and out may alias.  Batched form solves `count`
 * independent rectangles in one pipeline (DST-I -> Thomas -> DST-I). */
int fd_rect_solve(fd_plan plan, const double *f, double *out, void *stream);
int fd_rect_solve_batched(int count, const fd_plan *plans, const double *const *f,
                          double *const *out, void *stream);

/* --- transforms.apply_Q / apply_Qt for the DD pair (transforms.py:106-136):
 * out[r, :] = sqrt(2/(n+1)) DST-I(in[r, :]), rows x n, may alias; any n up to
 * 65535 (see fd_transform_rows). */
int fd_dst_rows(int rows, int n, const double *in, double *out, int device, void *stream);

/* apply_Q (inverse = 1) / apply_Qt (inverse = 0) of any pair along rows of
 * length n (transforms.py:106-148): DD on the real-symmetric FFT kernel
 * (n + 1 = 2^p in [256, 4096]) or the dense periodic-table transform
 * (n <= 2048), NN and PP (even n) on the dense table up to 2048, every other
 * length on the mixed-radix / Bluestein passes (n <= 65535). */
int fd_transform_rows(int rows, int n, int pair, int inverse, const double *in, double *out, int device,
                      void *stream);

/* Device-side problem assembly: f = lap p + kappa p at the
 * cell-centred nodes (origin + (i - 1/2) h, geometry.py:82-86) of an m x n
 * rectangle, minus lift_e * delta * p(ghost) on the line next to each edge
 * with a nonzero lift factor (1 ghost-node, 2 half-cell Dirichlet;
 * rectsolver.py:292-313); exact (optional) = p.  solution 0: sin(pi x)
 * sin(pi y) + e^(x+y)/e^2, 1: sin(pi x) sin(pi y). */
int fd_assemble_rhs(int m, int n, double x0, double y0, double dx, double dy, double kappa, int solution,
                    double lift_west, double lift_east, double lift_south, double lift_north, double *f,
                    double *exact, void *stream);

/* --- rectsolver.apply_rect_operator (rectsolver.py:264-289), non-periodic:
 * out = 5-point stencil of v on an m x n grid, delta = 1/h^2, end modifiers
 * mod_* on the four boundary-adjacent lines (geometry.py:118-128). */
int fd_stencil_apply(int m, int n, double delta_x, double delta_y, double kappa,
                     double mod_west, double mod_east, double mod_south, double mod_north,
                     const double *v, double *out, void *stream);
/* Same with periodic axes (wrap-around neighbours instead of end modifiers,
 * rectsolver.py:274-285). */
int fd_stencil_apply_ex(int m, int n, double delta_x, double delta_y, double kappa,
                        double mod_west, double mod_east, double mod_south, double mod_north,
                        int periodic_x, int periodic_y, const double *v, double *out, void *stream);

/* --- ddm.build_schur_operator (ddm.py:182-201).  For neighbour i:
 * to_center maps its line into the centre  (R_ci, ddm.py:85),
 * from_center maps the centre line into it (R_ic, ddm.py:86).
 * Index arrays are HOST int64 of length line_len[i]; they are copied. */
int fd_schur_create(fd_schur *out, fd_plan center, double center_mod_south,
                    double center_mod_north, int n_nb, const fd_plan *nb,
                    const int *line_len,
                    const int64_t *const *to_c_from, const int64_t *const *to_c_to,
                    const double *to_c_coupling,
                    const int64_t *const *from_c_from, const int64_t *const *from_c_to,
                    const double *from_c_coupling);
/* The centre operator A_c of (A_c - S) (fd_unprecond_apply, the true
 * residual) in the caller's layout: grid, 1/h^2, kappa, end modifiers and
 * periodic axes of the coupled subdomain (rectsolver.py:264-289) -- needed
 * for a transposed or periodic centre; default: from the centre plan. */
int fd_schur_set_stencil(fd_schur op, int m, int n, double delta_x, double delta_y, double kappa, double mod_west,
                         double mod_east, double mod_south, double mod_north, int periodic_x, int periodic_y);
/* Interface-only (Steklov) neighbour applies -- SURVEY 8f row 2, an opt-in
 * variant of SchurOperator.schur (ddm.py:108-123) with the same result up to
 * rounding: neighbour i's interface line (length line_len, a DD pair with
 * ghost-node ends along the line) sits at the first (end 0) or last (end 1)
 * row of its sweep (sweep_len rows, end modifiers mod_lo/mod_hi); pos_in[j] /
 * pos_out[j] are the line positions of entry j of its R_ic / R_ci maps.  Then
 * R_ci A_i^{-1} R_ic = c_ci c_ic Q diag(1/beta_end) Q^T on the line, O(L log L)
 * per apply.  Full solves stay in the pre-solves and the back-substitution. */
int fd_schur_set_steklov(fd_schur op, int i, int line_len, int sweep_len, double delta_line,
                         double delta_sweep, double kappa, double mod_lo, double mod_hi, int end,
                         const int64_t *pos_in, const int64_t *pos_out);
int fd_schur_use_steklov(fd_schur op, int enable);
int fd_schur_destroy(fd_schur op);
/* SchurOperator.schur / center_solve / preconditioned / unpreconditioned
 * (ddm.py:112-136); p, out are centre-sized device vectors, may not alias. */
int fd_schur_apply(fd_schur op, const double *p, double *out, void *stream);
int fd_center_solve(fd_schur op, const double *r, double *out, void *stream);
int fd_precond_apply(fd_schur op, const double *p, double *out, void *stream);
int fd_unprecond_apply(fd_schur op, const double *p, double *out, void *stream);

/* --- krylov.gmres(op.preconditioned, rhs) (krylov.py:61-165), x0 = 0 when
 * x_is_zero, else x holds x0.  history (host, capacity hist_cap) receives
 * |g_{k+1}|/||r0|| per step with the reference's final overwrite.
 * FD_ERR_NOT_CONVERGED leaves the last iterate in x and fills *rep. */
int fd_gmres_precond(fd_schur op, const double *rhs, double *x, int x_is_zero,
                     int m, double tol, int max_restarts, double *history,
                     int hist_cap, fd_report *rep, void *stream);

/* --- ddm.ddm_solve for a star composite (ddm.py:210-270 with
 * krylov.solve_coupled's fft branch, krylov.py:168-195): f_center/f_nb are
 * device right-hand sides, p_center/p_nb receive the solution. */
int fd_ddm_solve(fd_schur op, const double *f_center, const double *const *f_nb,
                 double *p_center, double *const *p_nb, int m, double tol,
                 int max_restarts, double *history, int hist_cap, fd_report *rep,
                 void *stream);

/* --- Arnoldi building blocks (krylov.py:105-111,141) for GMRES driven by a
 * caller-supplied operator.  V is a device array of >= k+2 rows of length N
 * (row stride N).  fd_arnoldi_step: MGS of w against V[0..k], writes
 * h[0..k+1] (host) and *w_norm (||w|| before orthogonalisation) and leaves the
 * orthogonalised w in place (not normalised). */
int fd_arnoldi_step(int N, int k, const double *V, double *w, double *h,
                    double *w_norm, void *stream);
/* x += V[0..k-1]^T y  (y host, length k) */
int fd_basis_update(int N, int k, const double *V, const double *y, double *x, void *stream);
/* out = a * x (+ b * y if y) ; y may be NULL */
int fd_axpby(int N, double a, const double *x, double b, const double *y, double *out,
             void *stream);
/* host result: ||x||_2 with the library's deterministic reduction order */
int fd_norm(int N, const double *x, double *result, void *stream);
int fd_dot(int N, const double *x, const double *y, double *result, void *stream);

/* --- subdomain-sharded solve (replaces the reference's thread
 * pool over neighbour solves, ddm.py:112-123,241-261, by one process per GPU).
 * fd_comm_unique_id: 128-byte NCCL id on rank 0 (broadcast it out of band);
 * fd_comm_init: NCCL communicator of this rank over NVLink/NVSwitch (libnccl
 * opened at run time).  fd_comm_init_loopback: nranks in-process ranks (host
 * threads) on one device, the test transport of the protocol. */
int fd_comm_unique_id(char *id128);
int fd_comm_init(fd_comm *out, int nranks, int rank, const char *id128, int device);
int fd_comm_init_loopback(fd_comm *outs, int nranks, int device);
int fd_comm_rank(fd_comm comm, int *rank, int *nranks);
int fd_comm_destroy(fd_comm comm);
/* Attach a communicator to an operator built identically on every rank:
 * owner[i] = rank that solves neighbour i (rank 0 holds the centre). */
int fd_schur_set_comm(fd_schur op, fd_comm comm, const int *owner);
/* fd_ddm_solve over the ranks: every rank calls it; rank 0 runs GMRES and
 * drives the interface-line exchange of each operator application (two
 * point-to-point messages of <= 32 KB per remote arm), arm owners pre-solve,
 * serve the applies and back-substitute their own fields.  f_nb / p_nb are
 * read / written for owned arms only; rep / history are filled on rank 0. */
int fd_ddm_solve_dist(fd_schur op, const double *f_center, const double *const *f_nb, double *p_center,
                      double *const *p_nb, int m, double tol, int max_restarts, double *history,
                      int hist_cap, fd_report *rep, void *stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* FFTDDM_B200_H */
