// wtv_prox.cu — weighted constrained TV prox as ONE persistent cooperative
// kernel for sm_100a.
//
// Replaces (paths under /root/reference/pkg/src/tvqn/):
//   dual_tv_solver.py:161-250  solve()            FGP dual loop, FISTA momentum, rel-change stop
//   dual_tv_solver.py:119-135  w_of_p/_prox_of    v - reg W^-1 div(P), then wpm_box
//   tv_ops.py:107-159          apply_diff(+adjoint), gradient_stack, dual_divergence
//   tv_ops.py:170-180          project_dual       iso ball / aniso clamp
//   wpm.py:92-106              apply_metric_inverse (Woodbury, r x r Cholesky)
//   wpm.py:145-231             _shift_point, phi, _newton_matrix, semismooth_newton
//   wpm.py:234-253             wpm_box
// extended to W = diag(d) + sign U U^T (Theorem-1 extension; d == NULL is
// the reference's tau*I exactly).
//
// Design (B200-first):
//  * The whole solve is one launch.  Blocks (all co-resident) walk a fixed
//    phase machine; between phases they meet at a device-wide barrier whose
//    LAST arriving block reduces the per-block partial sums in block order
//    (deterministic, no float atomics) and runs the scalar controller (r x r
//    Cholesky / LU, Newton accept/stop, FISTA t-sequence, rel-change test).
//    No host round trip, no per-iteration launches.
//  * Phases per FGP iteration:  DIV (z-marching stencil: a = v - reg D^-1
//    div(P_bar), partial U^T D^-1 div)  ->  NEWTON x (1 + steps) (pointwise
//    phi / generalized-Jacobian partials over a, d, U)  ->  DUAL (z-marching:
//    q = clamp(...) evaluated on the fly, forward differences, projection,
//    momentum, in-place P/P_bar update, ||P_next-P||^2, ||P||^2 partials).
//  * Stencil phases: a warp owns 32 consecutive x (coalesced), 8 warps own 8
//    rows y, and each thread marches a z-chunk carrying the z-1 (DIV) / z+1
//    (DUAL) neighbour in registers; x+1 comes by warp shuffle.
//  * Fields: T (f32 or f64); every reduction and scalar in f64.
#include <cooperative_groups.h>

#include "common.cuh"

namespace bq {
namespace {

constexpr int TX = 32, TY = 8, NT = TX * TY;

enum Phase : int { PH_SETUP = 0, PH_DIV = 1, PH_NEWTON = 2, PH_DUAL = 3, PH_FINAL = 4, PH_DONE = 5 };

struct ProxCtl {
  int phase, abort, div_src, final_mode;
  int it, newton_it, newton_total, converged;
  int status, last_newton_it, last_newton_conv, pad_;
  double t, mom, rel, best_res, last_res, pad2_;
  double beta[BQ_MAX_RANK], best_beta[BQ_MAX_RANK], gw[BQ_MAX_RANK];
  double chol[BQ_MAX_RANK * BQ_MAX_RANK];
  unsigned long long t_last;
  unsigned long long phase_ns[6];
  int phase_cnt[6];
};

template <typename T>
struct ProxArgs {
  int ndim, mode, rank, sign, accelerated, max_iter, newton_max_iter, wpm_only;
  int K1, K2, K3;
  long long N, plane;
  double tau, reg, step, eps, newton_eps, lo, hi;
  const T* lo_arr;
  const T* hi_arr;
  const T* d;
  const T* U;
  const T* v;
  T* p;
  T* pb;
  T* a;
  T* x;
  double* beta_io;
  bq_wtv_report* report;
  double* partials;
  unsigned* bar;
  ProxCtl* ctl;
  int zc, ntx, nty, items;
};

template <int R>
struct NV {
  static constexpr int gram = R * (R + 1) / 2;
  static constexpr int newton = R + R * (R + 1) / 2;
  static constexpr int acc = newton > 2 ? newton : 2;
};

// ---------------------------------------------------------------------------
// Controller helpers (single thread, f64).  r <= 8.
// ---------------------------------------------------------------------------
__device__ __noinline__ bool chol_factor(double* a, int r) {  // in place, lower, row-major
  for (int j = 0; j < r; ++j) {
    double s = a[j * r + j];
    for (int k = 0; k < j; ++k) s -= a[j * r + k] * a[j * r + k];
    if (!(s > 0.0)) return false;
    double l = sqrt(s);
    a[j * r + j] = l;
    for (int i = j + 1; i < r; ++i) {
      double t = a[i * r + j];
      for (int k = 0; k < j; ++k) t -= a[i * r + k] * a[j * r + k];
      a[i * r + j] = t / l;
    }
    for (int i = 0; i < j; ++i) a[i * r + j] = 0.0;
  }
  return true;
}
__device__ void chol_solve(const double* l, int r, double* b) {
  for (int i = 0; i < r; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= l[i * r + k] * b[k];
    b[i] = s / l[i * r + i];
  }
  for (int i = r - 1; i >= 0; --i) {
    double s = b[i];
    for (int k = i + 1; k < r; ++k) s -= l[k * r + i] * b[k];
    b[i] = s / l[i * r + i];
  }
}
// LU with partial pivoting (the numpy.linalg.solve / LAPACK gesv algorithm);
// returns false on an exactly-zero pivot (LinAlgError in the reference).
__device__ __noinline__ bool lu_solve(double* a, int r, double* b) {
  for (int k = 0; k < r; ++k) {
    int piv = k;
    double best = fabs(a[k * r + k]);
    for (int i = k + 1; i < r; ++i)
      if (fabs(a[i * r + k]) > best) best = fabs(a[i * r + k]), piv = i;
    if (best == 0.0) return false;
    if (piv != k) {
      for (int j = 0; j < r; ++j) {
        double t = a[k * r + j];
        a[k * r + j] = a[piv * r + j];
        a[piv * r + j] = t;
      }
      double t = b[k];
      b[k] = b[piv];
      b[piv] = t;
    }
    for (int i = k + 1; i < r; ++i) {
      double f = a[i * r + k] / a[k * r + k];
      for (int j = k; j < r; ++j) a[i * r + j] -= f * a[k * r + j];
      b[i] -= f * b[k];
    }
  }
  for (int i = r - 1; i >= 0; --i) {
    double s = b[i];
    for (int j = i + 1; j < r; ++j) s -= a[i * r + j] * b[j];
    b[i] = s / a[i * r + i];
  }
  return true;
}

template <typename T, int R>
__device__ __noinline__ void controller(const ProxArgs<T>& A, int phase, const double* red) {
  ProxCtl* c = A.ctl;
  {
    const unsigned long long now = global_ns();
    if (phase == PH_SETUP) {
      for (int i = 0; i < 6; ++i) c->phase_ns[i] = 0, c->phase_cnt[i] = 0;
    } else {
      c->phase_ns[phase] += now - c->t_last;
      c->phase_cnt[phase] += 1;
    }
    c->t_last = now;
  }
  const bool diag = A.d != nullptr;
  auto start_newton = [&]() {
    c->newton_it = 0;
    c->best_res = INFINITY;
    for (int i = 0; i < R; ++i) c->best_beta[i] = c->beta[i];
    c->phase = PH_NEWTON;
  };
  auto finish_newton = [&](int converged) {
    for (int i = 0; i < R; ++i) c->beta[i] = c->best_beta[i];
    c->newton_total += c->newton_it;
    c->last_newton_it = c->newton_it;
    c->last_newton_conv = converged;
    c->last_res = (R == 0) ? 0.0 : c->best_res;
    if (c->final_mode) {
      c->phase = PH_FINAL;
    } else {
      double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * c->t * c->t));
      c->mom = A.accelerated ? (c->t - 1.0) / tn : 0.0;
      c->phase = PH_DUAL;
    }
  };
  auto after_div = [&]() {
    if (R == 0) {
      c->newton_it = 0;
      finish_newton(1);
      return;
    }
    start_newton();
  };

  switch (phase) {
    case PH_SETUP: {
      // cap = I + sign U^T D^-1 U  (wpm.py:50-56), lower Cholesky
      double cap[BQ_MAX_RANK * BQ_MAX_RANK];
      int k = 0;
      for (int i = 0; i < R; ++i)
        for (int j = 0; j <= i; ++j, ++k) {
          double g = diag ? red[k] : red[k] / A.tau;
          double val = (i == j ? 1.0 : 0.0) + A.sign * g;
          cap[i * R + j] = val;
          cap[j * R + i] = val;
        }
      c->status = 0;
      c->abort = 0;
      if (R > 0 && !chol_factor(cap, R)) {
        c->status = BQ_ENOTPD;
        c->phase = PH_DONE;
        A.report->status = BQ_ENOTPD;
        return;
      }
      for (int i = 0; i < R * R; ++i) c->chol[i] = cap[i];
      for (int i = 0; i < R; ++i) {
        c->beta[i] = A.beta_io ? A.beta_io[i] : 0.0;
        c->gw[i] = 0.0;
      }
      c->t = 1.0;
      c->mom = 0.0;
      c->it = 1;
      c->newton_total = 0;
      c->converged = 0;
      c->rel = INFINITY;
      c->last_newton_it = 0;
      c->last_newton_conv = 1;
      c->last_res = 0.0;
      const bool single = A.wpm_only || A.reg == 0.0;
      c->div_src = single ? 1 : 0;  // 1: P (final), 0: P_bar
      c->final_mode = single ? 1 : 0;
      c->phase = PH_DIV;
      return;
    }
    case PH_DIV: {
      // Woodbury coefficient: coef = cap^-1 U^T D^-1 div ; gw = reg * coef
      double coef[BQ_MAX_RANK > 0 ? BQ_MAX_RANK : 1];
      for (int i = 0; i < R; ++i) coef[i] = diag ? red[i] : red[i] / A.tau;
      if (R > 0) chol_solve(c->chol, R, coef);
      for (int i = 0; i < R; ++i) c->gw[i] = (A.reg == 0.0 || A.wpm_only) ? 0.0 : A.reg * coef[i];
      after_div();
      return;
    }
    case PH_NEWTON: {
      // wpm.py:170-231: residual at beta, best-residual tracking, stop tests, step
      double phi[BQ_MAX_RANK > 0 ? BQ_MAX_RANK : 1];
      double ss = 0.0;
      for (int i = 0; i < R; ++i) {
        phi[i] = red[i] + c->beta[i];
        ss += phi[i] * phi[i];
      }
      double res = sqrt(ss);
      if (res < c->best_res) {
        c->best_res = res;
        for (int i = 0; i < R; ++i) c->best_beta[i] = c->beta[i];
      }
      if (res <= A.newton_eps) {
        finish_newton(1);
        return;
      }
      if (c->newton_it == A.newton_max_iter) {
        finish_newton(0);
        return;
      }
      double h[BQ_MAX_RANK * BQ_MAX_RANK];
      int k = R;
      for (int i = 0; i < R; ++i)
        for (int j = 0; j <= i; ++j, ++k) {
          double g = diag ? red[k] : red[k] / A.tau;
          double val = (i == j ? 1.0 : 0.0) + A.sign * g;
          h[i * R + j] = val;
          h[j * R + i] = val;
        }
      double hs[BQ_MAX_RANK * BQ_MAX_RANK];
      for (int i = 0; i < R * R; ++i) hs[i] = h[i];
      double st[BQ_MAX_RANK > 0 ? BQ_MAX_RANK : 1];
      for (int i = 0; i < R; ++i) st[i] = phi[i];
      if (!lu_solve(hs, R, st)) {
        // Levenberg fallback: mu = 1e-8 ||H||_inf (wpm.py:219-223)
        double ninf = 0.0;
        for (int i = 0; i < R; ++i) {
          double rs = 0.0;
          for (int j = 0; j < R; ++j) rs += fabs(h[i * R + j]);
          ninf = fmax(ninf, rs);
        }
        for (int i = 0; i < R * R; ++i) hs[i] = h[i];
        for (int i = 0; i < R; ++i) hs[i * R + i] += 1e-8 * ninf, st[i] = phi[i];
        lu_solve(hs, R, st);
      }
      for (int i = 0; i < R; ++i) c->beta[i] -= st[i];
      c->newton_it += 1;
      c->phase = PH_NEWTON;
      return;
    }
    case PH_DUAL: {
      // dual_tv_solver.py:226-239
      double num = sqrt(red[0]), den = sqrt(red[1]);
      double rel = (num == 0.0) ? 0.0 : (den > 0.0 ? num / den : INFINITY);
      c->rel = rel;
      bool stop = false;
      if (rel < A.eps) {
        c->converged = 1;
        stop = true;
      } else {
        c->t = 0.5 * (1.0 + sqrt(1.0 + 4.0 * c->t * c->t));
        if (c->it >= A.max_iter) stop = true;
        else c->it += 1;
      }
      if (stop) {
        c->div_src = 1;
        c->final_mode = 1;
      }
      c->phase = PH_DIV;
      return;
    }
    case PH_FINAL: {
      bq_wtv_report* rp = A.report;
      const bool single = A.wpm_only || A.reg == 0.0;
      rp->iterations = single ? 1 : c->it;
      rp->converged = single ? 1 : c->converged;
      rp->rel_change = single ? 0.0 : c->rel;
      rp->newton_iterations = c->newton_total;
      rp->status = 0;
      rp->newton_residual = c->last_res;
      rp->last_newton_iterations = c->last_newton_it;
      rp->last_newton_converged = c->last_newton_conv;
      if (A.beta_io)
        for (int i = 0; i < R; ++i) A.beta_io[i] = c->beta[i];
      for (int i = 0; i < 6; ++i) rp->phase_ns[i] = (double)c->phase_ns[i], rp->phase_count[i] = c->phase_cnt[i];
      c->phase = PH_DONE;
      return;
    }
    default:
      c->phase = PH_DONE;
  }
}

// ---------------------------------------------------------------------------
// Per-voxel pieces
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T clampv(T z, T lo, T hi) {
  return fmin(fmax(z, lo), hi);  // np.clip == minimum(maximum(z, lo), hi)
}

template <typename T, int R>
struct Voxel {
  // shift point and clamp at voxel j (wpm.py:145-158 with W^-1 folded in):
  //   wv = a + sign (U.gw)/e ;  z = wv - sign (U.beta)/e ;  q = clamp(z)
  const ProxArgs<T>& A;
  const T* gw;
  const T* beta;
  __device__ __forceinline__ void eval(long long j, T& wv, T& z, T& e, T (&u)[R > 0 ? R : 1]) const {
    const T av = A.a[j];
    e = A.d ? __ldg(A.d + j) : (T)A.tau;
    T uw = 0, ub = 0;
#pragma unroll
    for (int c = 0; c < R; ++c) {
      u[c] = __ldg(A.U + (long long)c * A.N + j);
      uw += u[c] * gw[c];
      ub += u[c] * beta[c];
    }
    if (R > 0) {
      const T sg = (T)A.sign;
      wv = av + sg * uw / e;
      z = wv - sg * ub / e;
    } else {
      wv = av;
      z = av;
    }
  }
  __device__ __forceinline__ T bound_lo(long long j) const { return A.lo_arr ? __ldg(A.lo_arr + j) : (T)A.lo; }
  __device__ __forceinline__ T bound_hi(long long j) const { return A.hi_arr ? __ldg(A.hi_arr + j) : (T)A.hi; }
  __device__ __forceinline__ T q(long long j) const {
    T wv, z, e, u[R > 0 ? R : 1];
    eval(j, wv, z, e, u);
    return clampv(z, bound_lo(j), bound_hi(j));
  }
};

// ---------------------------------------------------------------------------
// The persistent kernel
// ---------------------------------------------------------------------------
template <typename T, int R>
__global__ void __launch_bounds__(NT, 2) wtv_prox_kernel(ProxArgs<T> A) {
  constexpr int NACC = NV<R>::acc;
  __shared__ double s_red[kMaxVals];
  __shared__ double s_bv[kMaxVals];
  __shared__ double s_scr[(NT / 32) * kMaxVals];
  __shared__ T s_gw[BQ_MAX_RANK], s_beta[BQ_MAX_RANK];
  __shared__ T s_mom;
  __shared__ int s_phase, s_div_src, s_abort;

  GridSync gs{A.bar, A.bar + 1, gridDim.x, 0};
  if (threadIdx.x == 0) gs.my_gen = ld_acquire_u32(A.bar + 1);

  const long long N = A.N;
  const long long stride = (long long)gridDim.x * NT;
  const long long gtid = (long long)blockIdx.x * NT + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool diag = A.d != nullptr;

  int phase = PH_SETUP;
  while (true) {
    double acc[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
    int nv = 0;
    Voxel<T, R> vox{A, s_gw, s_beta};

    if (phase == PH_SETUP) {
      // P_bar = P (dual_tv_solver.py:215) and Gram partials U^T D^-1 U
      nv = NV<R>::gram;
      const bool copy = !(A.wpm_only || A.reg == 0.0);
      for (long long j = gtid; j < N; j += stride) {
        if (copy)
          for (int n = 0; n < A.ndim; ++n) A.pb[n * N + j] = A.p[n * N + j];
        if (R > 0) {
          T u[R > 0 ? R : 1];
#pragma unroll
          for (int c = 0; c < R; ++c) u[c] = __ldg(A.U + (long long)c * N + j);
          const T e = diag ? __ldg(A.d + j) : (T)1;
          int k = 0;
#pragma unroll
          for (int c = 0; c < R; ++c)
#pragma unroll
            for (int c2 = 0; c2 <= c; ++c2, ++k) acc[k] += diag ? (double)(u[c] * u[c2] / e) : (double)u[c] * (double)u[c2];
        }
      }
    } else if (phase == PH_DIV) {
      nv = R;
      if (A.wpm_only || A.reg == 0.0) {
        for (long long j = gtid; j < N; j += stride) A.a[j] = A.v[j];
      } else {
        const T* __restrict__ F = s_div_src ? A.p : A.pb;
        const T reg = (T)A.reg;
        for (int item = blockIdx.x; item < A.items; item += gridDim.x) {
          const int tx = item % A.ntx, rest = item / A.ntx;
          const int ty = rest % A.nty, tz = rest / A.nty;
          const int x = tx * TX + lane, y = ty * TY + warp;
          const int z0 = tz * A.zc, z1 = min(z0 + A.zc, A.K3);
          if (x >= A.K1 || y >= A.K2) continue;
          long long j = (long long)z0 * A.plane + (long long)y * A.K1 + x;
          T prev3 = 0;
          if (A.ndim >= 3 && z0 > 0) prev3 = F[2 * N + j - A.plane];
          for (int z = z0; z < z1; ++z, j += A.plane) {
            // tv_ops.py:122-133 per dimension, dual_divergence :151-159 summed in order
            const T c1 = F[j];
            T div = (x < A.K1 - 1 ? -c1 : (T)0) + (x > 0 ? F[j - 1] : (T)0);
            if (A.ndim >= 2) {
              const T c2 = F[N + j];
              div += (y < A.K2 - 1 ? -c2 : (T)0) + (y > 0 ? F[N + j - A.K1] : (T)0);
            }
            if (A.ndim >= 3) {
              const T c3 = F[2 * N + j];
              div += (z < A.K3 - 1 ? -c3 : (T)0) + (z > 0 ? prev3 : (T)0);
              prev3 = c3;
            }
            const T e = diag ? __ldg(A.d + j) : (T)A.tau;
            const T de = div / e;
            A.a[j] = __ldg(A.v + j) - reg * de;
#pragma unroll
            for (int c = 0; c < R; ++c) acc[c] += (double)__ldg(A.U + (long long)c * N + j) * (double)(diag ? de : div);
          }
        }
      }
    } else if (phase == PH_NEWTON) {
      // phi(beta) partials U^T (wv - clamp(z)) and U_A^T D_A^-1 U_A (wpm.py:150-167)
      nv = NV<R>::newton;
      constexpr int UN = 2;
      for (long long j0 = gtid; j0 < N; j0 += stride * UN) {
#pragma unroll
        for (int uu = 0; uu < UN; ++uu) {
          const long long j = j0 + uu * stride;
          if (j < N) {
            T wv, z, e, u[R > 0 ? R : 1];
            vox.eval(j, wv, z, e, u);
            const T lo = vox.bound_lo(j), hi = vox.bound_hi(j);
            const T dl = wv - clampv(z, lo, hi);
#pragma unroll
            for (int c = 0; c < R; ++c) acc[c] += (double)(u[c] * dl);
            if (z > lo && z < hi) {
              int k = R;
#pragma unroll
              for (int c = 0; c < R; ++c)
#pragma unroll
                for (int c2 = 0; c2 <= c; ++c2, ++k)
                  acc[k] += diag ? (double)(u[c] * u[c2] / e) : (double)u[c] * (double)u[c2];
            }
          }
        }
      }
    } else if (phase == PH_DUAL) {
      // dual_tv_solver.py:225-239: P_next = Proj(P_bar + step D q), momentum
      nv = 2;
      const T step = (T)A.step, mom = s_mom;
      T* __restrict__ P = A.p;
      T* __restrict__ PB = A.pb;
      for (int item = blockIdx.x; item < A.items; item += gridDim.x) {
        const int tx = item % A.ntx, rest = item / A.ntx;
        const int ty = rest % A.nty, tz = rest / A.nty;
        const int x = tx * TX + lane, y = ty * TY + warp;
        const int z0 = tz * A.zc, z1 = min(z0 + A.zc, A.K3);
        if (y >= A.K2) continue;  // whole warp leaves together
        const bool act = x < A.K1;
        long long j = (long long)z0 * A.plane + (long long)y * A.K1 + x;
        T qc = act ? vox.q(j) : (T)0;
        for (int z = z0; z < z1; ++z, j += A.plane) {
          T qu = 0;
          const bool has_up = A.ndim >= 3 && z < A.K3 - 1;
          if (act && has_up) qu = vox.q(j + A.plane);
          T qr = __shfl_down_sync(0xffffffffu, qc, 1);
          if (!act) continue;
          const bool has_r = x < A.K1 - 1;
          if (has_r && lane == 31) qr = vox.q(j + 1);
          T g[3];
          g[0] = has_r ? qr - qc : (T)0;
          g[1] = (A.ndim >= 2 && y < A.K2 - 1) ? vox.q(j + A.K1) - qc : (T)0;
          g[2] = has_up ? qu - qc : (T)0;
          T w[3], po[3];
#pragma unroll
          for (int n = 0; n < 3; ++n) {
            if (n < A.ndim) {
              po[n] = P[n * N + j];
              w[n] = PB[n * N + j] + step * g[n];
            } else {
              po[n] = 0;
              w[n] = 0;
            }
          }
          if (A.mode == BQ_TV_ISO) {
            // tv_ops.py:177-179: p / max(||p_col||, 1)
            T ss = w[0] * w[0];
            if (A.ndim >= 2) ss += w[1] * w[1];
            if (A.ndim >= 3) ss += w[2] * w[2];
            const T den = fmax(sqrt(ss), (T)1);
#pragma unroll
            for (int n = 0; n < 3; ++n) w[n] = w[n] / den;
          } else {
#pragma unroll
            for (int n = 0; n < 3; ++n) w[n] = clampv(w[n], (T)-1, (T)1);
          }
#pragma unroll
          for (int n = 0; n < 3; ++n) {
            if (n < A.ndim) {
              const T df = w[n] - po[n];
              acc[0] += (double)df * (double)df;
              acc[1] += (double)po[n] * (double)po[n];
              P[n * N + j] = w[n];
              PB[n * N + j] = w[n] + mom * df;
            }
          }
          qc = qu;
        }
      }
    } else if (phase == PH_FINAL) {
      nv = 0;
      for (long long j = gtid; j < N; j += stride) A.x[j] = vox.q(j);
    }

    // ---- barrier + fused reduction + controller --------------------------
    if (nv > 0) block_sum_to<NT, NACC>(acc, nv, s_bv, s_scr);
    const int cur = phase;
    bool ok = grid_reduce_sync<NT>(gs, s_bv, nv, A.partials, s_red, s_scr, [&](const double* red) {
      if (threadIdx.x == 0) controller<T, R>(A, cur, red);
    });
    if (threadIdx.x == 0) {
      volatile ProxCtl* c = A.ctl;
      if (!ok) {
        c->abort = 1;
        A.report->status = BQ_ETIMEOUT;
      }
      s_phase = c->phase;
      s_abort = c->abort;
      s_div_src = c->div_src;
      s_mom = (T)c->mom;
      for (int i = 0; i < R; ++i) {
        s_gw[i] = (T)c->gw[i];
        s_beta[i] = (T)c->beta[i];
      }
    }
    __syncthreads();
    phase = s_phase;
    if (s_abort || phase == PH_DONE) break;
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
template <typename T, int R>
int launch(bq_ctx* ctx, const bq_wtv_desc& D, int wpm_only, cudaStream_t st) {
  ProxArgs<T> A{};
  A.ndim = D.ndim;
  A.mode = D.mode;
  A.rank = D.rank;
  A.sign = D.sign;
  A.accelerated = D.accelerated;
  A.max_iter = D.max_iter;
  A.newton_max_iter = D.newton_max_iter;
  A.wpm_only = wpm_only;
  A.K1 = (int)D.dims[0];
  A.K2 = (int)D.dims[1];
  A.K3 = (int)D.dims[2];
  A.N = D.dims[0] * D.dims[1] * D.dims[2];
  A.plane = D.dims[0] * D.dims[1];
  A.tau = D.tau;
  A.reg = D.reg;
  A.step = D.step;
  A.eps = D.eps;
  A.newton_eps = D.newton_eps;
  A.lo = D.lo;
  A.hi = D.hi;
  A.lo_arr = (const T*)D.lo_arr;
  A.hi_arr = (const T*)D.hi_arr;
  A.d = (const T*)D.d;
  A.U = (const T*)D.U;
  A.v = (const T*)D.v;
  A.p = (T*)D.p;
  A.pb = (T*)D.pb;
  A.a = (T*)D.a;
  A.x = (T*)D.x;
  A.beta_io = D.beta;
  A.report = (bq_wtv_report*)D.report;
  A.partials = ctx->ws.partials;
  A.bar = ctx->ws.barrier;
  A.ctl = (ProxCtl*)ctx->ws.ctl;

  auto kern = wtv_prox_kernel<T, R>;
  int per_sm = 0;
  BQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, 0));
  BQ_CHECK(per_sm > 0, BQ_ECUDA, "wtv_prox: kernel does not fit on an SM");
  long long max_blocks = std::min<long long>((long long)per_sm * ctx->num_sms, kMaxBlocks);
  // small problems: fewer blocks -> cheaper barriers
  long long want = std::max<long long>(1, (A.N + 4 * NT - 1) / (4 * NT));
  int G = (int)std::min<long long>(max_blocks, want);
  A.ntx = (A.K1 + TX - 1) / TX;
  A.nty = (A.K2 + TY - 1) / TY;
  // z-chunk: minimise the per-block critical path ceil(items/G) * (zc + 1)
  long long nxy = (long long)A.ntx * A.nty;
  int best_zc = A.K3;
  long long best_cost = -1;
  for (int zc = 1; zc <= A.K3; ++zc) {
    long long items = nxy * ((A.K3 + zc - 1) / zc);
    long long waves = (items + G - 1) / G;
    long long cost = waves * (zc + 1);
    if (best_cost < 0 || cost < best_cost) best_cost = cost, best_zc = zc;
  }
  A.zc = best_zc;
  A.items = (int)(nxy * ((A.K3 + best_zc - 1) / best_zc));

  BQ_CUDA(cudaMemsetAsync(ctx->ws.barrier, 0, 2 * sizeof(unsigned), st));
  void* args[] = {&A};
  BQ_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(G), dim3(NT), args, 0, st));
  return BQ_OK;
}

template <typename T>
int dispatch_rank(bq_ctx* ctx, const bq_wtv_desc& D, int wpm_only, cudaStream_t st) {
  switch (D.rank) {
    case 0: return launch<T, 0>(ctx, D, wpm_only, st);
    case 1: return launch<T, 1>(ctx, D, wpm_only, st);
    case 2: return launch<T, 2>(ctx, D, wpm_only, st);
    case 3: return launch<T, 3>(ctx, D, wpm_only, st);
    case 4: return launch<T, 4>(ctx, D, wpm_only, st);
    case 5: return launch<T, 5>(ctx, D, wpm_only, st);
    case 6: return launch<T, 6>(ctx, D, wpm_only, st);
    case 7: return launch<T, 7>(ctx, D, wpm_only, st);
    case 8: return launch<T, 8>(ctx, D, wpm_only, st);
  }
  set_error("wtv_prox: rank %d outside [0, %d]", D.rank, BQ_MAX_RANK);
  return BQ_EINVAL;
}

int validate(const bq_wtv_desc& D, bool wpm_only) {
  BQ_CHECK(D.ndim >= 1 && D.ndim <= 3, BQ_EINVAL, "ndim must be 1..3, got %d", D.ndim);
  for (int i = 0; i < 3; ++i) BQ_CHECK(D.dims[i] >= 1, BQ_EINVAL, "dims must be positive");
  for (int i = D.ndim; i < 3; ++i) BQ_CHECK(D.dims[i] == 1, BQ_EINVAL, "dims beyond ndim must be 1");
  BQ_CHECK(D.dims[0] * D.dims[1] * D.dims[2] < (1ll << 40), BQ_EINVAL, "grid too large");
  BQ_CHECK(D.dtype == BQ_F32 || D.dtype == BQ_F64, BQ_EINVAL, "dtype must be BQ_F32 or BQ_F64");
  BQ_CHECK(D.sign == 1 || D.sign == -1, BQ_EINVAL, "sign must be +1 or -1, got %d", D.sign);
  BQ_CHECK(D.d != nullptr || D.tau > 0, BQ_EINVAL, "tau must be positive, got %g", D.tau);
  BQ_CHECK(D.reg >= 0, BQ_EINVAL, "reg must be nonnegative");
  BQ_CHECK(D.rank == 0 || D.U != nullptr, BQ_EINVAL, "U is required for rank > 0");
  BQ_CHECK(D.v && D.x && D.a && D.report, BQ_EINVAL, "v, x, a and report are required");
  BQ_CHECK(D.newton_max_iter >= 0, BQ_EINVAL, "newton_max_iter must be >= 0");
  if (!wpm_only) {
    BQ_CHECK(D.eps > 0, BQ_EINVAL, "eps must be positive");
    BQ_CHECK(D.max_iter >= 1, BQ_EINVAL, "max_iter must be >= 1");
    BQ_CHECK(D.p && D.pb, BQ_EINVAL, "p and pb are required");
    BQ_CHECK(D.mode == BQ_TV_ISO || D.mode == BQ_TV_ANISO, BQ_EINVAL, "bad TV mode");
    BQ_CHECK(D.reg == 0 || D.step > 0, BQ_EINVAL, "step must be positive");
  }
  return BQ_OK;
}

}  // namespace
}  // namespace bq

extern "C" int bq_wtv_prox(bq_ctx* ctx, const bq_wtv_desc* desc, void* stream) {
  using namespace bq;
  BQ_CHECK(ctx && desc, BQ_EINVAL, "bq_wtv_prox: null argument");
  int rc = validate(*desc, false);
  if (rc) return rc;
  BQ_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = (cudaStream_t)stream;
  return desc->dtype == BQ_F32 ? dispatch_rank<float>(ctx, *desc, 0, st)
                               : dispatch_rank<double>(ctx, *desc, 0, st);
}

extern "C" int bq_wpm_box(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t rank, int32_t sign,
                          double tau, const void* d, const void* U, const void* x, double lo,
                          double hi, const void* lo_arr, const void* hi_arr, double* beta_inout,
                          double newton_eps, int32_t newton_max_iter, void* x_out, void* a_scratch,
                          void* report, void* stream) {
  using namespace bq;
  BQ_CHECK(ctx, BQ_EINVAL, "bq_wpm_box: null ctx");
  bq_wtv_desc D{};
  D.ndim = 1;
  D.dtype = dtype;
  D.dims[0] = n;
  D.dims[1] = 1;
  D.dims[2] = 1;
  D.mode = BQ_TV_ISO;
  D.rank = rank;
  D.sign = sign;
  D.accelerated = 0;
  D.tau = tau;
  D.reg = 0.0;
  D.step = 0.0;
  D.eps = 1.0;
  D.max_iter = 1;
  D.newton_max_iter = newton_max_iter;
  D.newton_eps = newton_eps;
  D.lo = lo;
  D.hi = hi;
  D.lo_arr = lo_arr;
  D.hi_arr = hi_arr;
  D.d = d;
  D.U = U;
  D.v = x;
  D.a = a_scratch;
  D.x = x_out;
  D.beta = beta_inout;
  D.report = report;
  int rc = validate(D, true);
  if (rc) return rc;
  BQ_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = (cudaStream_t)stream;
  return dtype == BQ_F32 ? dispatch_rank<float>(ctx, D, 1, st) : dispatch_rank<double>(ctx, D, 1, st);
}
