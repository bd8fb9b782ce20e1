/*
 * bq.h — C ABI of the B200-native BQNPM hot path (libbq.so).
 *
 * Plain C: no torch, numpy or C++ types cross this boundary.  Every device
 * buffer is owned by the caller (a torch tensor on the Python side) and is
 * passed as a raw device pointer plus sizes; streams are passed as the raw
 * cudaStream_t value (void*).  Every entry point returns an int status:
 * 0 = ok, <0 = error (BQ_E*), with the text available from bq_last_error()
 * (thread-local).  Nothing throws or exits across the ABI.  All calls are
 * stream-ordered and asynchronous unless stated otherwise.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/tvqn/):
 *   bq_wtv_prox          dual_tv_solver.py:161-250  solve(prob, eps, max_iter, accelerated)
 *                        (with w_of_p :119-123, _prox_of :126-135, dual_step_size :155-158,
 *                         tv_ops.py:107-180 stencils/projection, wpm.py:145-253 wpm_box)
 *   bq_wpm_box           wpm.py:234-253             wpm_box(x, w, box, beta0, eps, max_iter)
 *   bq_metric_gram       wpm.py:50-56               DiagPlusLowRank.__post_init__ (I +/- U^T U / tau)
 *   bq_metric_apply      wpm.py:81-89               apply_metric(w, x)
 *   bq_metric_inverse    wpm.py:92-106              apply_metric_inverse(w, x)
 *   bq_sr1               hessian_sr1.py:52-101      estimate_sr1(s, m, gamma, alpha_fallback)
 *   bq_vk                solvers.py:80-89           compute_v_k(slots, w, step)
 *   bq_dot               (reduction helper used by the host mirrors; fixed-order, deterministic)
 *   bq_tv_value          tv_ops.py:162-167          tv_value(grid, x, mode)
 *   bq_dct_views         forward_models.py:86-91,139-150,166-183 DCT stand-in view batch
 *   bq_born_views        (absent in reference; north star (1)) first-Born view batch
 *   bq_ls_*              (absent in reference; north star (1)(2)) Lippmann-Schwinger views
 */
#ifndef BQ_H_
#define BQ_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define BQ_OK 0
#define BQ_EINVAL -1      /* invalid argument (maps to ValueError) */
#define BQ_ECUDA -2       /* CUDA runtime / cuFFT failure (RuntimeError) */
#define BQ_ENOTPD -3      /* metric not positive definite (ValueError) */
#define BQ_ETIMEOUT -4    /* device-side grid barrier timed out (RuntimeError) */
#define BQ_ENOMEM -5

#define BQ_F32 0
#define BQ_F64 1

#define BQ_TV_ISO 0
#define BQ_TV_ANISO 1

#define BQ_MAX_RANK 8

typedef struct bq_ctx bq_ctx;

/* Context: one per (device, host thread).  Holds the cuFFT plan cache and,
 * PER STREAM (created on a stream's first use, up to 16 streams), the
 * grid-barrier/control/partials workspace of the persistent kernels and of the
 * helper reductions: calls on different streams of one context may run
 * concurrently; calls on one stream are ordered and share that stream's set. */
int bq_ctx_create(int device, bq_ctx** out);
int bq_ctx_destroy(bq_ctx* ctx);
const char* bq_last_error(void);
/* Version / capability string ("bq 0.1 sm_100a"). */
const char* bq_version(void);

/* ---------------------------------------------------------------------------
 * Weighted constrained TV prox (FGP dual iteration + structured WPM Newton).
 *   x* = argmin_{lo<=x<=hi} 1/2 ||x - v||_W^2 + reg TV(x),
 *   W = diag(d) + sign U U^T  (d == NULL: d == tau, the reference's tau*I)
 * Layout: flat Fortran order over dims (dims[0] fastest) == C-order (K3,K2,K1).
 * U: rank contiguous N-vectors (column c at U + c*N).  P: ndim contiguous
 * N-vectors.  beta: rank doubles (device).  One persistent cooperative
 * kernel runs the whole solve; every decision is taken on the device.
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t ndim;          /* 1..3 (the reference Grid.ndim; drives the step) */
  int32_t dtype;         /* BQ_F32 / BQ_F64 for every field */
  int64_t dims[3];       /* K1, K2, K3 (unused dims = 1) */
  int32_t mode;          /* BQ_TV_ISO / BQ_TV_ANISO */
  int32_t rank;          /* r = columns of U, 0..BQ_MAX_RANK */
  int32_t sign;          /* +1 / -1 */
  int32_t accelerated;   /* FISTA momentum on/off */
  double tau;            /* scalar diagonal (used when d == NULL) */
  double reg;            /* TV weight (>= 0) */
  double step;           /* dual step 1/(4 ndim omega reg); ignored when reg == 0 */
  double eps;            /* FGP relative-change tolerance */
  int32_t max_iter;      /* FGP cap */
  int32_t newton_max_iter;
  double newton_eps;
  double lo, hi;         /* scalar box (may be +/-inf) */
  const void* lo_arr;    /* optional per-voxel bounds (NULL -> scalar) */
  const void* hi_arr;
  const void* d;         /* optional per-voxel diagonal (NULL -> tau) */
  const void* U;         /* rank x N */
  const void* v;         /* N   center */
  void* p;               /* ndim x N  in: warm start (zeros if none); out: P* */
  void* pb;              /* ndim x N  scratch (momentum field) */
  void* a;               /* N   scratch */
  void* x;               /* N   out: the prox */
  double* beta;          /* rank doubles in (warm) / out (beta*) ; may be NULL if rank==0 */
  void* report;          /* device bq_wtv_report (out) */
  /* optional scratch enabling the fused single-pass-per-iteration kernel
   * (K1 in {4..128} dividing 128, 16-byte aligned fields): p2 = ndim x N
   * (third slot of the P ring, with p and pb), a2 = N (ping-pong of a). */
  void* p2;
  void* a2;
  /* optional device scalars of a GPU-resident outer loop (NULL: use tau/step
   * above): [0] tau (overrides `tau`; the dual step is then computed on the
   * device as 1/(4 ndim (1/tau) reg), dual_tv_solver.py:155-158), [1] the
   * effective rank of U (trailing columns are zero), [2] the effective rank of
   * the previous solve -- the beta warm start is zeroed when [1] != [2]
   * (dual_tv_solver.py:185-186) and [2] is set to [1] at the end.  Fused
   * kernel only (K1 in {4..128 dividing 128, 256}, scalar bounds, d == NULL). */
  double* dev_metric;
} bq_wtv_desc;

typedef struct {
  int32_t iterations;
  int32_t converged;
  int32_t newton_iterations;
  int32_t status;        /* 0 ok, BQ_ENOTPD, BQ_ETIMEOUT */
  double rel_change;
  double newton_residual; /* residual of the last wpm_box call */
  int32_t last_newton_iterations;
  int32_t last_newton_converged;
  /* device-side phase timeline (globaltimer at every grid barrier, taken by the
   * last-arriving block): nanoseconds and visits per phase
   * [setup, div, newton, dual, final, unused] */
  double phase_ns[6];
  int32_t phase_count[6];
  /* part of phase_ns spent before the LAST block arrived at the barrier
   * (i.e. the slowest block's work); the rest is barrier latency */
  double phase_work_ns[6];
} bq_wtv_report;

int bq_wtv_prox(bq_ctx* ctx, const bq_wtv_desc* desc, void* stream);

/* Structured weighted box projection (wpm_box) alone: x_out = clamp(x - sign D^-1 U beta*).
 * Uses the same device Newton as the prox; report as above (iterations = 1). */
int bq_wpm_box(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t rank, int32_t sign, double tau,
               const void* d, const void* U, const void* x, double lo, double hi,
               const void* lo_arr, const void* hi_arr, double* beta_inout, double newton_eps,
               int32_t newton_max_iter, void* x_out, void* a_scratch, void* report, void* stream);

/* GPU-resident BQNPM step (k > K_s): the aggregated metric and v_k with every
 * scalar on the device (solvers.py:67-89).  count (<= 8) slots in kappa order:
 * host arrays of device pointers x_t, g_t, u_t (N; zeros for a rejected SR1
 * term) and est_t (bq_sr1's device est: [0] tau_t, [1] has_u).  Writes Uc_out
 * (count x N: the accepted u_t compacted in slot order, zero columns after),
 * meta (device, >= 128 doubles: [0] tau_w = sum tau_t, [1] effective rank --
 * the layout bq_wtv_desc::dev_metric reads; [2] is left to the prox) and
 * v_out = W^-1 sum_t (tau_t x_t + u_t (u_t^T x_t) - step g_t), W = tau_w I + Uc Uc^T. */
int bq_bqnpm_metric_vk(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t count, const void* const* xs,
                       const void* const* gs, const void* const* us, const double* const* ests, double step,
                       void* Uc_out, double* meta, void* acc_scratch, void* v_out, void* stream);

/* ---------------------------------------------------------------------------
 * z-slab-sharded prox: one rank's passes (dual_tv_solver.py:221-239 over a
 * slab of planes [z0, z1) of a 3-D grid split along dims[2]).  The host runs
 * the FGP / Newton control and the NCCL steps between the passes
 * (paper_2307_02043_b200/slab_prox.py).  All buffers are the rank's local
 * slab (N = K1*K2*L voxels); halos are single K1*K2 planes.
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t dtype;         /* BQ_F32 / BQ_F64 for every field */
  int32_t mode;          /* BQ_TV_ISO / BQ_TV_ANISO */
  int32_t rank;          /* columns of U, 0..BQ_MAX_RANK */
  int32_t sign;          /* +1 / -1 */
  int64_t K1, K2, L;     /* slab: L planes of K1 x K2 */
  int32_t first, last;   /* the slab holds global plane 0 / K3-1 */
  double tau;            /* scalar diagonal when d == NULL */
  double reg;            /* TV weight */
  double lo, hi;         /* scalar box */
  const void* d;         /* local per-voxel diagonal or NULL */
  const void* U;         /* rank x N local */
  const void* v;         /* N local */
  double* ctl;           /* optional device control block (>= 128 doubles, see
                          * bq_slab_ctl): when set, the passes read c and beta
                          * from it (the host arrays may be NULL) and
                          * bq_slab_newton is a no-op once the Newton is done */
} bq_slab_desc;

/* t = D^-1 div(F) over the slab (F: 3 x N; halo_below = F_z of plane z0-1,
 * NULL when first); s_out (device, rank doubles) = U^T t (local sum). */
int bq_slab_div(bq_ctx* ctx, const bq_slab_desc* desc, const void* field, const void* halo_below,
                void* t_out, double* s_out, void* stream);
/* Newton residual / Jacobian partials at beta (host arrays c, beta: rank doubles;
 * c = cap^-1 s_global): out (device) = [U^T (w - clamp z) (rank) ;
 * lower triangle of sum_inside U_c U_c' / d (or / 1 with scalar tau)]. */
int bq_slab_newton(bq_ctx* ctx, const bq_slab_desc* desc, const void* t, const double* c,
                   const double* beta, double* out, void* stream);
/* q = clamp(z(beta)) over the slab. */
int bq_slab_q(bq_ctx* ctx, const bq_slab_desc* desc, const void* t, const double* c, const double* beta,
              void* q_out, void* stream);
/* P_next = project(Pbar + step grad q) (halo_above = q of plane z1, NULL when
 * last), Pbar_next = P_next + momentum (P_next - P), norms_out (device, 2
 * doubles) = local ||P_next - P||^2, ||P||^2. */
int bq_slab_dual(bq_ctx* ctx, const bq_slab_desc* desc, const void* pbar, const void* p, const void* q,
                 const void* halo_above, double step, double momentum, void* p_next, void* pbar_next,
                 double* norms_out, void* stream);

/* Device control of the sharded solve (one thread; every rank runs it on the
 * same all-reduced input, so every rank takes the same branch):
 *   op 0 INIT    ctl <- cap Cholesky factor (`in`, rank x rank, row-major L) and
 *                beta (`in` + 64), counters cleared
 *   op 1 COEF    in = s (rank): c = cap^-1 s; Newton state reset (best = inf,
 *                it = 0, done = rank == 0); beta saved for op 4
 *   op 2 NEWTON  in = [U^T (w - clamp z) (rank); lower triangle of H]: one step of
 *                wpm.py:207-224 (residual, best iterate, stop, Levenberg
 *                fallback); when it stops, beta <- best beta, totals updated
 *   op 3 NORMS   in = [||P_next - P||^2, ||P||^2]: rel-change (dual_tv_solver.py:
 *                229-231), fgp_done when rel < eps
 *   op 4 UNDO    drop a speculative iteration: beta and the Newton total as at op 1
 * Layout (doubles): [0] done [1] it [2] best_res [3] newton_total [4] rel
 * [5] fgp_done [6] last_it [8..15] beta [16..23] best beta [24..31] c
 * [32..39] saved beta [40..103] Cholesky factor. */
int bq_slab_ctl(bq_ctx* ctx, const bq_slab_desc* desc, int32_t op, const double* in, double newton_eps,
                int32_t newton_max_iter, double eps, void* stream);

/* ---------------------------------------------------------------------------
 * Standalone TV stencils (tv_ops.py:107-180); the prox kernels fuse them.
 * ------------------------------------------------------------------------ */
/* out = D^axis x (adjoint = 0) or (D^axis)^T x (adjoint = 1); axis 1-based. */
int bq_tv_diff(bq_ctx* ctx, int32_t dtype, int32_t ndim, const int64_t* dims, int32_t axis,
               int32_t adjoint, const void* x, void* out, void* stream);
/* p_out (ndim x N) = [D^1 x; ...; D^ndim x]  (gradient_stack / dual_adjoint). */
int bq_tv_grad_stack(bq_ctx* ctx, int32_t dtype, int32_t ndim, const int64_t* dims, const void* x,
                     void* p_out, void* stream);
/* out (N) = sum_a (D^a)^T p_a  (dual_divergence). */
int bq_tv_divergence(bq_ctx* ctx, int32_t dtype, int32_t ndim, const int64_t* dims, const void* p,
                     void* out, void* stream);
/* out = project_dual(p): per-voxel unit-ball (iso) or [-1, 1] clip (aniso). */
int bq_tv_project_dual(bq_ctx* ctx, int32_t dtype, int32_t ndim, int64_t n, int32_t mode, const void* p,
                       void* out, void* stream);
/* Structured-WPM residual phi(beta) = U^T (x - clamp(x - sign D^-1 U beta)) + beta and
 * the generalized Jacobian I + sign U_A^T D_A^-1 U_A (wpm.py:150-167):
 * beta (device, rank doubles) -> phi_out (device, rank), jac_out (device, rank*rank
 * row-major, may be NULL). */
int bq_wpm_phi(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t rank, int32_t sign, double tau,
               const void* d, const void* U, const void* x, double lo, double hi, const void* lo_arr,
               const void* hi_arr, const double* beta, double* phi_out, double* jac_out, void* stream);

/* ---------------------------------------------------------------------------
 * Metric algebra (W = diag(d) + sign U U^T), deterministic fixed-order reductions.
 * ------------------------------------------------------------------------ */
/* gram_out (device, rank*rank doubles, row-major) = U^T D^-1 U  (D = tau I when d == NULL). */
int bq_metric_gram(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t rank, double tau, const void* d,
                   const void* U, double* gram_out, void* stream);
/* out = W x  (or W^-1 x via Woodbury when inverse != 0).  For the inverse,
 * gram (device, rank*rank doubles) is bq_metric_gram's U^T D^-1 U; the
 * capacitance I + sign gram(/tau) is factorised on the device. */
int bq_metric_apply(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t rank, int32_t sign, double tau,
                    const void* d, const void* U, const double* gram, int32_t inverse,
                    const void* x, void* out, void* stream);

/* Construction-time check of W = diag(d) + sign U U^T in one pass with a small
 * per-SM footprint (it can run beside a persistent prox): out (device, 1 +
 * rank*rank doubles) = [min(d) (+inf when d == NULL), U^T D^-1 U (D = I when
 * d == NULL; row-major)]. */
int bq_metric_check(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t rank, const void* d, const void* U,
                    double* out, void* stream);

/* dots_out[k] = <a_k, b_k> for k < count (device doubles). */
int bq_dot(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t count, const void* const* a_ptrs,
           const void* const* b_ptrs, double* dots_out, void* stream);

/* SR1 estimate B = tau I + u u^T from (s, m) (hessian_sr1.py:52-101).
 * Writes u (N; zeros when rejected) and est_out (device, 9 doubles):
 * {tau, has_u, <s,m>, curv, <m,m>, nnz(s), ||s||, ||m - tau s||, status}. */
int bq_sr1(bq_ctx* ctx, int32_t dtype, int64_t n, const void* s, const void* m, double gamma,
           double alpha_fallback, void* u_out, double* est_out, void* stream);

/* v = W^-1 sum_t (tau_t x_t + u_t (u_t^T x_t) - step g_t)   (solvers.py:80-89).
 * slots: count (<= 8) triples; u_t may be NULL (rank-0 slot); taus is a host
 * array.  W = tau_w I + sign U_w U_w^T with gram_w = U_w^T U_w (device). */
int bq_vk(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t count, const void* const* xs,
          const void* const* gs, const void* const* us, const double* taus, double step,
          int32_t rank, int32_t sign, double tau_w, const void* U_w, const double* gram_w,
          void* acc_scratch, void* v_out, void* stream);

/* TV value (tv_ops.py:162-167) -> out (device double). */
int bq_tv_value(bq_ctx* ctx, int32_t dtype, int32_t ndim, const int64_t* dims, int32_t mode,
                const void* x, double* out, void* stream);

/* ---------------------------------------------------------------------------
 * Masked-spectrum view operators (the reference forward model,
 * forward_models.py:86-183).  Layout as above (dims[0] fastest).
 * ------------------------------------------------------------------------ */
/* Orthonormal DCT-II (inverse=0) or DCT-III (inverse=1) along one axis
 * (dims[axis] <= 512); out of place. */
int bq_dct_axis(bq_ctx* ctx, int32_t dtype, const int64_t* dims, int32_t axis, int32_t inverse,
                const void* in, void* out, void* stream);
/* 3-point edge-clamped mean along one axis (forward_models.py:139-150). */
int bq_smooth_axis(bq_ctx* ctx, int32_t dtype, const int64_t* dims, int32_t axis, const void* in,
                   void* out, void* stream);
/* Fused subset combine over `count` (<= 64) views of one spectrum F:
 *   r = scale * sum_i M_{v_i} (F - y_i)          (r_out may be NULL)
 *   cost_out[i] = 1/2 || M_{v_i} F - y_i ||^2    (cost_out may be NULL; device)
 * masks: one 64-bit view set per frequency; views_dev: device int32 ids. */
int bq_views_combine(bq_ctx* ctx, int32_t dtype, int64_t n, const void* F, const void* const* ys,
                     const uint64_t* masks, const int32_t* views_dev, int32_t count, double scale,
                     void* r_out, double* cost_out, void* stream);
/* Pointwise chain-rule helpers: op 0 out = x + s a^2; 1 out = x + 2s a b;
 * 2 out = a b; 3 out = x + 2s b; 4 out = s x. */
int bq_pointwise(bq_ctx* ctx, int32_t dtype, int32_t op, int64_t n, const void* x, const void* a,
                 const void* b, double s, void* out, void* stream);

/* ---------------------------------------------------------------------------
 * First-Born / Lippmann-Schwinger view batches (north star (1)(2); no
 * reference code -- the discretisation is specified in oracle/physics.py).
 * Complex fields are interleaved (re, im) in the field precision; B views per
 * call; the (2n)^3 transforms are batched cuFFT plans cached in the context.
 * ------------------------------------------------------------------------ */
/* khat ((2n)^3 complex) = FFT of the Green kernel K(d) = h^3 e^{i kb|d|}/(4 pi |d|). */
int bq_green_init(bq_ctx* ctx, int32_t dtype, int32_t n, double h, double kb, void* khat, void* stream);
/* out (B x n^3 complex) = plane waves exp(i k_b . r), kvec_dev = 3B doubles (device). */
int bq_ls_incident(bq_ctx* ctx, int32_t dtype, int32_t n, double h, int32_t B, const double* kvec_dev,
                   void* out, void* stream);
/* Green operator through the padded transform (pad_buf: B x (2n)^3 complex scratch):
 *  op 0: out = alpha v + beta G_dom(f . v)        op 1: out = alpha v + beta conj(f) . G_dom^H v
 *  op 2: out = G_det(f . v) (n^2 per view)        op 3: out = G^H P_det^T v (v: n^2 per view)
 *  ops 0, 1, 3 add `addend` (B x N, may be NULL) to the result. */
int bq_ls_conv(bq_ctx* ctx, int32_t dtype, int32_t n, int32_t B, int32_t op, const void* khat,
               const void* f, const void* v, double alpha, double beta, const void* addend,
               void* pad_buf, void* out, void* stream);
/* out_b = f . in_b (f real, N; in/out complex B x N). */
int bq_cscale_real(bq_ctx* ctx, int32_t dtype, int64_t N, int32_t B, const void* f, const void* in,
                   void* out, void* stream);
/* Device-resident batched BiCGSTAB, x_b = A^-1 rhs_b from x0 = 0 to the relative residual tol
 * (oracle/physics.py bicgstab per view): adjoint 0 solves A = I - G_dom diag f, 1 solves A^H.
 * vec_work: 6 B N complex; conv_scratch: the bq_ls_conv pad_buf; small_work:
 * bq_ls_bicgstab_small_bytes() bytes; iters: device, B ints.  Converged views are skipped. */
int64_t bq_ls_bicgstab_small_bytes(bq_ctx* ctx, int32_t n, int32_t B);
int bq_ls_bicgstab(bq_ctx* ctx, int32_t dtype, int32_t n, int32_t B, int32_t adjoint, const void* khat,
                   const void* f, const void* rhs, void* x, double tol, int32_t max_iter, void* vec_work,
                   void* conv_scratch, void* small_work, int32_t* iters, void* stream);
/* grad (+)= scale * sum_b Re(conj(fp u_b) w_b), views summed in order. */
int bq_ls_grad_accum(bq_ctx* ctx, int32_t dtype, int64_t N, int32_t B, const void* fp, const void* u,
                     const void* w, double scale, void* grad, int32_t accumulate, void* stream);
/* scattering potential f(x) and f'(x) (born: 2 k0^2 nb x; ls: k0^2((nb+x)^2 - nb^2)). */
int bq_ls_potential(bq_ctx* ctx, int32_t dtype, int64_t N, const void* x, double k0, double nb,
                    int32_t born, void* f, void* fp, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* BQ_H_ */
