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
//  * The whole solve is one launch.  Blocks (all co-resident, one or two per
//    SM) walk a fixed phase machine.  Between phases they meet at a
//    device-wide barrier whose LAST arriving block reduces the per-block
//    partial sums in block order (deterministic, no float atomics) and
//    publishes the totals; every block then runs the scalar controller
//    (r x r Cholesky / LU, Newton accept/stop, FISTA t-sequence, rel-change
//    test) redundantly on its own shared-memory copy of the control state, so
//    no block ever waits on serialized global control traffic.
//  * Phases per FGP iteration:  DIV (z-marching stencil: a = v - reg D^-1
//    div(P_bar), partial U^T D^-1 div)  ->  NEWTON x (1 + steps) (pointwise
//    phi / generalized-Jacobian partials over a, d, U; 16-byte vector loads)
//    ->  DUAL (z-marching: q = clamp(...) evaluated on the fly, forward
//    differences, projection, momentum, in-place P/P_bar update,
//    ||P_next-P||^2 and ||P||^2 partials).
//  * Stencil phases: a warp owns 32 consecutive x (coalesced), the block's
//    warps own consecutive rows y, and each block marches one contiguous,
//    equal-length run of (tile, z) planes carrying the z-1 (DIV) / z+1 (DUAL)
//    neighbour in registers; x+1 comes by warp shuffle, y+1 through L1.
//  * Fields: T (f32 or f64); every reduction and scalar in f64.
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"

namespace bq {
namespace {

constexpr int TX = 32;

enum Phase : int { PH_SETUP = 0, PH_DIV = 1, PH_NEWTON = 2, PH_DUAL = 3, PH_FINAL = 4, PH_DONE = 5 };

// Control state; one copy per block in shared memory.
struct Ctl {
  int phase, div_src, final_mode, it;
  int newton_it, newton_total, converged, status;
  int last_newton_it, last_newton_conv, abort, pad_;
  double t, mom, rel, best_res, last_res;
  double beta[BQ_MAX_RANK], best_beta[BQ_MAX_RANK], gw[BQ_MAX_RANK];
  double chol[BQ_MAX_RANK * BQ_MAX_RANK];
  unsigned long long t_last;
  unsigned long long phase_ns[6];
  unsigned long long phase_work_ns[6];
  int phase_cnt[6];
};

template <typename T>
struct ProxArgs {
  int ndim, mode, rank, sign, accelerated, max_iter, newton_max_iter, wpm_only;
  int K1, K2, K3, vec, vx;
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
  double* red;  // published totals of the last barrier (kMaxVals)
  unsigned* bar;
  int ntx, nty;
  long long tile_planes;  // ntx * nty * K3
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

// Runs in thread 0 of EVERY block on its shared copy `c` (identical inputs ->
// identical decisions).  `writer` (block 0) also publishes report and beta*.
template <typename T, int R>
__device__ __noinline__ void controller(const ProxArgs<T>& A, Ctl& c, int phase, const double* red, bool writer) {
  const bool diag = A.d != nullptr;
  {
    const unsigned long long now = global_ns();
    if (phase == PH_SETUP) {
      for (int i = 0; i < 6; ++i) c.phase_ns[i] = 0, c.phase_work_ns[i] = 0, c.phase_cnt[i] = 0;
    } else {
      const unsigned long long arrive = __double_as_longlong(red[kMaxVals - 1]);
      c.phase_ns[phase] += now - c.t_last;
      if (arrive > c.t_last && arrive <= now) c.phase_work_ns[phase] += arrive - c.t_last;
      c.phase_cnt[phase] += 1;
    }
    c.t_last = now;
  }
  auto finish_newton = [&](int converged) {
    for (int i = 0; i < R; ++i) c.beta[i] = c.best_beta[i];
    c.newton_total += c.newton_it;
    c.last_newton_it = c.newton_it;
    c.last_newton_conv = converged;
    c.last_res = (R == 0) ? 0.0 : c.best_res;
    if (c.final_mode) {
      c.phase = PH_FINAL;
    } else {
      const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * c.t * c.t));
      c.mom = A.accelerated ? (c.t - 1.0) / tn : 0.0;
      c.phase = PH_DUAL;
    }
  };

  switch (phase) {
    case PH_SETUP: {
      // cap = I + sign U^T D^-1 U  (wpm.py:50-56), lower Cholesky
      double cap[BQ_MAX_RANK * BQ_MAX_RANK];
      int k = 0;
      for (int i = 0; i < R; ++i)
        for (int j = 0; j <= i; ++j, ++k) {
          const double g = diag ? red[k] : red[k] / A.tau;
          const double val = (i == j ? 1.0 : 0.0) + A.sign * g;
          cap[i * R + j] = val;
          cap[j * R + i] = val;
        }
      c.status = 0;
      c.abort = 0;
      if (R > 0 && !chol_factor(cap, R)) {
        c.status = BQ_ENOTPD;
        c.phase = PH_DONE;
        if (writer) A.report->status = BQ_ENOTPD;
        return;
      }
      for (int i = 0; i < R * R; ++i) c.chol[i] = cap[i];
      for (int i = 0; i < R; ++i) {
        c.beta[i] = A.beta_io ? A.beta_io[i] : 0.0;
        c.gw[i] = 0.0;
      }
      c.t = 1.0;
      c.mom = 0.0;
      c.it = 1;
      c.newton_total = 0;
      c.converged = 0;
      c.rel = INFINITY;
      c.last_newton_it = 0;
      c.last_newton_conv = 1;
      c.last_res = 0.0;
      const bool single = A.wpm_only || A.reg == 0.0;
      c.div_src = single ? 1 : 0;  // 1: P (final prox), 0: P_bar
      c.final_mode = single ? 1 : 0;
      c.phase = PH_DIV;
      return;
    }
    case PH_DIV: {
      // Woodbury coefficient: coef = cap^-1 U^T D^-1 div ; gw = reg * coef
      double coef[BQ_MAX_RANK > 0 ? BQ_MAX_RANK : 1];
      for (int i = 0; i < R; ++i) coef[i] = diag ? red[i] : red[i] / A.tau;
      if (R > 0) chol_solve(c.chol, R, coef);
      for (int i = 0; i < R; ++i) c.gw[i] = (A.reg == 0.0 || A.wpm_only) ? 0.0 : A.reg * coef[i];
      if (R == 0) {
        c.newton_it = 0;
        finish_newton(1);
        return;
      }
      c.newton_it = 0;
      c.best_res = INFINITY;
      for (int i = 0; i < R; ++i) c.best_beta[i] = c.beta[i];
      c.phase = PH_NEWTON;
      return;
    }
    case PH_NEWTON: {
      // wpm.py:170-231: residual at beta, best-residual tracking, stop tests, step
      double phi[BQ_MAX_RANK > 0 ? BQ_MAX_RANK : 1];
      double ss = 0.0;
      for (int i = 0; i < R; ++i) {
        phi[i] = red[i] + c.beta[i];
        ss += phi[i] * phi[i];
      }
      const double res = sqrt(ss);
      if (res < c.best_res) {
        c.best_res = res;
        for (int i = 0; i < R; ++i) c.best_beta[i] = c.beta[i];
      }
      if (res <= A.newton_eps) {
        finish_newton(1);
        return;
      }
      if (c.newton_it == A.newton_max_iter) {
        finish_newton(0);
        return;
      }
      double h[BQ_MAX_RANK * BQ_MAX_RANK];
      int k = R;
      for (int i = 0; i < R; ++i)
        for (int j = 0; j <= i; ++j, ++k) {
          const double g = diag ? red[k] : red[k] / A.tau;
          const double val = (i == j ? 1.0 : 0.0) + A.sign * g;
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
      for (int i = 0; i < R; ++i) c.beta[i] -= st[i];
      c.newton_it += 1;
      c.phase = PH_NEWTON;
      return;
    }
    case PH_DUAL: {
      // dual_tv_solver.py:226-239
      const double num = sqrt(red[0]), den = sqrt(red[1]);
      const double rel = (num == 0.0) ? 0.0 : (den > 0.0 ? num / den : INFINITY);
      c.rel = rel;
      bool stop = false;
      if (rel < A.eps) {
        c.converged = 1;
        stop = true;
      } else {
        c.t = 0.5 * (1.0 + sqrt(1.0 + 4.0 * c.t * c.t));
        if (c.it >= A.max_iter) stop = true;
        else c.it += 1;
      }
      if (stop) {
        c.div_src = 1;
        c.final_mode = 1;
      }
      c.phase = PH_DIV;
      return;
    }
    case PH_FINAL: {
      if (writer) {
        bq_wtv_report* rp = A.report;
        const bool single = A.wpm_only || A.reg == 0.0;
        rp->iterations = single ? 1 : c.it;
        rp->converged = single ? 1 : c.converged;
        rp->rel_change = single ? 0.0 : c.rel;
        rp->newton_iterations = c.newton_total;
        rp->status = 0;
        rp->newton_residual = c.last_res;
        rp->last_newton_iterations = c.last_newton_it;
        rp->last_newton_converged = c.last_newton_conv;
        if (A.beta_io)
          for (int i = 0; i < R; ++i) A.beta_io[i] = c.beta[i];
        for (int i = 0; i < 6; ++i) {
          rp->phase_ns[i] = (double)c.phase_ns[i];
          rp->phase_work_ns[i] = (double)c.phase_work_ns[i];
          rp->phase_count[i] = c.phase_cnt[i];
        }
      }
      c.phase = PH_DONE;
      return;
    }
    default:
      c.phase = PH_DONE;
  }
}

// ---------------------------------------------------------------------------
// Per-voxel pieces
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T clampv(T z, T lo, T hi) {
  return fmin(fmax(z, lo), hi);  // np.clip == minimum(maximum(z, lo), hi)
}

// Reciprocal: correctly rounded single-instruction-sequence in f32 (no IEEE
// division subroutine on the hot path); exact division in f64.
__device__ __forceinline__ float rcp(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double rcp(double x) { return 1.0 / x; }

// Isotropic dual-ball projection p / max(||p||, 1) (tv_ops.py:177-179).
__device__ __forceinline__ void ball(float (&w)[3], float ss) {
  if (ss > 1.0f) {
    const float s = rsqrtf(ss);
    w[0] *= s, w[1] *= s, w[2] *= s;
  }
}
__device__ __forceinline__ void ball(double (&w)[3], double ss) {
  const double den = fmax(sqrt(ss), 1.0);
  w[0] /= den, w[1] /= den, w[2] /= den;
}

// 4 consecutive elements; 16-byte vector loads (fp32) / 2 x 16 (fp64).
template <typename T>
struct Vec4;
template <>
struct Vec4<float> {
  static __device__ __forceinline__ void ro(const float* p, float (&o)[4]) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = v.x, o[1] = v.y, o[2] = v.z, o[3] = v.w;
  }
  static __device__ __forceinline__ void rw(const float* p, float (&o)[4]) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    o[0] = v.x, o[1] = v.y, o[2] = v.z, o[3] = v.w;
  }
  static __device__ __forceinline__ void st(float* p, const float (&o)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
  }
};
template <>
struct Vec4<double> {
  static __device__ __forceinline__ void ro(const double* p, double (&o)[4]) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    o[0] = a.x, o[1] = a.y, o[2] = b.x, o[3] = b.y;
  }
  static __device__ __forceinline__ void rw(const double* p, double (&o)[4]) {
    const double2 a = *reinterpret_cast<const double2*>(p);
    const double2 b = *(reinterpret_cast<const double2*>(p) + 1);
    o[0] = a.x, o[1] = a.y, o[2] = b.x, o[3] = b.y;
  }
  static __device__ __forceinline__ void st(double* p, const double (&o)[4]) {
    reinterpret_cast<double2*>(p)[0] = make_double2(o[0], o[1]);
    reinterpret_cast<double2*>(p)[1] = make_double2(o[2], o[3]);
  }
};

// Per-voxel shift point (wpm.py:145-158 with W^-1 folded in):
//   wv = a + sign (U.gw)/e ;  z = wv - sign (U.beta)/e
template <typename T, int R>
__device__ __forceinline__ void shift(T av, T e, const T (&u)[R > 0 ? R : 1], const T* gw, const T* beta, T sg,
                                      T& wv, T& z) {
  if (R > 0) {
    T uw = 0, ub = 0;
#pragma unroll
    for (int c = 0; c < R; ++c) {
      uw += u[c] * gw[c];
      ub += u[c] * beta[c];
    }
    const T ie = rcp(e);
    wv = av + sg * uw * ie;
    z = wv - sg * ub * ie;
  } else {
    wv = av;
    z = av;
  }
}

template <typename T, int R>
struct QEval {
  const T* __restrict__ a;
  const T* __restrict__ d;
  const T* __restrict__ U;
  const T* __restrict__ lo_arr;
  const T* __restrict__ hi_arr;
  long long N;
  T tau, lo, hi, sg;
  const T* gz;  // gw - beta: z = a + sign (U.gz)/e
  __device__ __forceinline__ T operator()(long long j) const {
    T z = a[j];
    if (R > 0) {
      const T e = d ? __ldg(d + j) : tau;
      T uz = 0;
#pragma unroll
      for (int c = 0; c < R; ++c) uz += __ldg(U + (long long)c * N + j) * gz[c];
      z += sg * uz * rcp(e);
    }
    return clampv(z, lo_arr ? __ldg(lo_arr + j) : lo, hi_arr ? __ldg(hi_arr + j) : hi);
  }
  // four consecutive voxels j..j+3 (j % 4 == 0, 16-byte aligned fields)
  __device__ __forceinline__ void q4(long long j, T (&q)[4]) const {
    Vec4<T>::rw(a + j, q);
    if (R > 0) {
      T e[4], uz[4] = {0, 0, 0, 0};
      if (d) Vec4<T>::ro(d + j, e);
      else e[0] = e[1] = e[2] = e[3] = tau;
#pragma unroll
      for (int c = 0; c < R; ++c) {
        T u[4];
        Vec4<T>::ro(U + (long long)c * N + j, u);
#pragma unroll
        for (int k = 0; k < 4; ++k) uz[k] += u[k] * gz[c];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) q[k] += sg * uz[k] * rcp(e[k]);
    }
    T l[4], h[4];
    if (lo_arr) Vec4<T>::ro(lo_arr + j, l);
    else l[0] = l[1] = l[2] = l[3] = lo;
    if (hi_arr) Vec4<T>::ro(hi_arr + j, h);
    else h[0] = h[1] = h[2] = h[3] = hi;
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = clampv(q[k], l[k], h[k]);
  }
};

// ---------------------------------------------------------------------------
// Stencil phases, x-vectorised: each lane owns 4 consecutive x (16-byte
// loads), a warp 128 x, the block TY rows; used when K1 % 4 == 0.
// ---------------------------------------------------------------------------
constexpr unsigned FULL = 0xffffffffu;
constexpr int TXV = 128;

// DIV: a = v - reg D^-1 div(F) ; acc[c] += U_c . D^-1 div(F)
template <typename T, int R, int TY, int NACC>
__device__ __forceinline__ void div_vec(const ProxArgs<T>& A, const T* __restrict__ F0, long long seg_begin,
                                        long long seg_end, int lane, int warp, double (&acc)[NACC]) {
  const long long N = A.N, plane = A.plane;
  const T* __restrict__ F1 = F0 + N;
  const T* __restrict__ F2 = F0 + 2 * N;
  T* __restrict__ Aout = A.a;
  const bool diag = A.d != nullptr;
  const T reg = (T)A.reg, tauT = (T)A.tau;
  const int K1 = A.K1, K2 = A.K2, K3 = A.K3, nd = A.ndim;
  long long pos = seg_begin;
  while (pos < seg_end) {
    const long long tile = pos / K3;
    const int z0 = (int)(pos - tile * K3);
    const int z1 = (int)min((long long)K3, z0 + (seg_end - pos));
    pos += z1 - z0;
    const int x0 = (int)(tile % A.ntx) * TXV;
    const int xb = x0 + 4 * lane;
    const int y = (int)(tile / A.ntx) * TY + warp;
    if (y >= K2) continue;  // warp-uniform
    const bool act = xb < K1;
    long long j = (long long)z0 * plane + (long long)y * K1 + xb;
    T prev3[4] = {0, 0, 0, 0};
    if (act && nd >= 3 && z0 > 0) Vec4<T>::rw(F2 + j - plane, prev3);
#pragma unroll 2
    for (int z = z0; z < z1; ++z, j += plane) {
      T c1[4] = {0, 0, 0, 0};
      if (act) Vec4<T>::rw(F0 + j, c1);
      T left = __shfl_up_sync(FULL, c1[3], 1);
      if (lane == 0) left = (act && xb > 0) ? F0[j - 1] : (T)0;
      if (!act) continue;
      // tv_ops.py:122-133 per dimension, summed in dimension order (:151-159)
      T dv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const T lk = (k == 0) ? left : c1[k - 1];
        dv[k] = (xb + k < K1 - 1 ? -c1[k] : (T)0) + (xb + k > 0 ? lk : (T)0);
      }
      if (nd >= 2) {
        T c2[4], l2[4] = {0, 0, 0, 0};
        Vec4<T>::rw(F1 + j, c2);
        if (y > 0) Vec4<T>::rw(F1 + j - K1, l2);
#pragma unroll
        for (int k = 0; k < 4; ++k) dv[k] += (y < K2 - 1 ? -c2[k] : (T)0) + l2[k];
      }
      if (nd >= 3) {
        T c3[4];
        Vec4<T>::rw(F2 + j, c3);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          dv[k] += (z < K3 - 1 ? -c3[k] : (T)0) + (z > 0 ? prev3[k] : (T)0);
          prev3[k] = c3[k];
        }
      }
      T e[4], vv[4], out[4];
      if (diag) Vec4<T>::ro(A.d + j, e);
      else e[0] = e[1] = e[2] = e[3] = tauT;
      Vec4<T>::ro(A.v + j, vv);
      T de[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        de[k] = dv[k] * rcp(e[k]);
        out[k] = vv[k] - reg * de[k];
      }
      Vec4<T>::st(Aout + j, out);
#pragma unroll
      for (int c = 0; c < R; ++c) {
        T u[4];
        Vec4<T>::ro(A.U + (long long)c * N + j, u);
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[c] += (double)u[k] * (double)(diag ? de[k] : dv[k]);
      }
    }
  }
}

// DUAL: P_next = Proj(P_bar + step D q), P_bar' = P_next + mom (P_next - P);
// acc[0] += ||P_next - P||^2, acc[1] += ||P||^2   (dual_tv_solver.py:225-239)
template <typename T, int R, int TY, int NACC>
__device__ __forceinline__ void dual_vec(const ProxArgs<T>& A, const QEval<T, R>& Q, T step, T mom,
                                         long long seg_begin, long long seg_end, int lane, int warp,
                                         double (&acc)[NACC]) {
  const long long N = A.N, plane = A.plane;
  T* __restrict__ P0 = A.p;
  T* __restrict__ PB0 = A.pb;
  const int K1 = A.K1, K2 = A.K2, K3 = A.K3, nd = A.ndim;
  const bool iso = A.mode == BQ_TV_ISO;
  long long pos = seg_begin;
  while (pos < seg_end) {
    const long long tile = pos / K3;
    const int z0 = (int)(pos - tile * K3);
    const int z1 = (int)min((long long)K3, z0 + (seg_end - pos));
    pos += z1 - z0;
    const int x0 = (int)(tile % A.ntx) * TXV;
    const int xb = x0 + 4 * lane;
    const int y = (int)(tile / A.ntx) * TY + warp;
    if (y >= K2) continue;  // warp-uniform
    const bool act = xb < K1;
    const bool has_y = nd >= 2 && y < K2 - 1;
    long long j = (long long)z0 * plane + (long long)y * K1 + xb;
    T qc[4] = {0, 0, 0, 0};
    if (act) Q.q4(j, qc);
#pragma unroll 1
    for (int z = z0; z < z1; ++z, j += plane) {
      const bool has_up = nd >= 3 && z < K3 - 1;
      T qu[4] = {0, 0, 0, 0}, qy[4] = {0, 0, 0, 0};
      if (act && has_up) Q.q4(j + plane, qu);
      if (act && has_y) Q.q4(j + K1, qy);
      T qn = __shfl_down_sync(FULL, qc[0], 1);
      if (lane == 31) qn = (act && xb + 4 < K1) ? Q(j + 4) : (T)0;
      if (act) {
        T w[3][4], po[3][4];
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          if (n < nd) {
            Vec4<T>::rw(P0 + n * N + j, po[n]);
            Vec4<T>::rw(PB0 + n * N + j, w[n]);
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const T right = (k < 3) ? qc[k + 1] : qn;
          T g[3];
          g[0] = (xb + k < K1 - 1) ? right - qc[k] : (T)0;
          g[1] = has_y ? qy[k] - qc[k] : (T)0;
          g[2] = has_up ? qu[k] - qc[k] : (T)0;
          T wk[3];
#pragma unroll
          for (int n = 0; n < 3; ++n) wk[n] = (n < nd) ? w[n][k] + step * g[n] : (T)0;
          if (iso) {
            T ss = wk[0] * wk[0];
            if (nd >= 2) ss += wk[1] * wk[1];
            if (nd >= 3) ss += wk[2] * wk[2];
            ball(wk, ss);
          } else {
#pragma unroll
            for (int n = 0; n < 3; ++n) wk[n] = clampv(wk[n], (T)-1, (T)1);
          }
#pragma unroll
          for (int n = 0; n < 3; ++n) {
            if (n < nd) {
              const T pk = (n < nd) ? po[n][k] : (T)0;
              const T df = wk[n] - pk;
              acc[0] += (double)df * (double)df;
              acc[1] += (double)pk * (double)pk;
              po[n][k] = wk[n];
              w[n][k] = wk[n] + mom * df;
            }
          }
        }
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          if (n < nd) {
            Vec4<T>::st(P0 + n * N + j, po[n]);
            Vec4<T>::st(PB0 + n * N + j, w[n]);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) qc[k] = qu[k];
    }
  }
}

// ---------------------------------------------------------------------------
// The persistent kernel
// ---------------------------------------------------------------------------
template <typename T, int R>
struct Cfg {
  // light variants: 512 threads x 2 blocks/SM (64 regs); heavier ones trade
  // block size for registers so the Newton accumulators never spill
  static constexpr bool kLight = sizeof(T) == 4 && R <= 2;
  static constexpr int NT = kLight ? 512 : 256;
  static constexpr int MINB = kLight ? 1 : (R <= 2 ? 2 : 1);
  static constexpr int TY = NT / TX;
};

template <typename T, int R>
__global__ void __launch_bounds__(Cfg<T, R>::NT, Cfg<T, R>::MINB) wtv_prox_kernel(ProxArgs<T> A) {
  constexpr int NT = Cfg<T, R>::NT;
  constexpr int TY = Cfg<T, R>::TY;
  constexpr int NACC = NV<R>::acc;
  __shared__ double s_red[kMaxVals];
  __shared__ double s_bv[kMaxVals];
  __shared__ double s_scr[(NT / 32) * kMaxVals];
  __shared__ Ctl s_c;
  __shared__ T s_gw[BQ_MAX_RANK], s_beta[BQ_MAX_RANK], s_gz[BQ_MAX_RANK];
  __shared__ T s_mom;
  __shared__ int s_phase, s_div_src, s_flag;

  unsigned my_gen = 0;
  if (threadIdx.x == 0) my_gen = ld_acquire_u32(A.bar + 1);

  const long long N = A.N;
  const long long stride = (long long)gridDim.x * NT;
  const long long gtid = (long long)blockIdx.x * NT + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool diag = A.d != nullptr;
  const T sg = (T)A.sign;
  const T tauT = (T)A.tau;
  // balanced contiguous run of (tile, z) planes for the stencil phases
  const long long seg_begin = (long long)blockIdx.x * A.tile_planes / gridDim.x;
  const long long seg_end = (long long)(blockIdx.x + 1) * A.tile_planes / gridDim.x;

  int phase = PH_SETUP;
  while (true) {
    double acc[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
    int nv = 0;

    if (phase == PH_SETUP) {
      // P_bar = P (dual_tv_solver.py:215) and Gram partials U^T D^-1 U
      nv = NV<R>::gram;
      const bool copy = !(A.wpm_only || A.reg == 0.0);
      const T* __restrict__ Pin = A.p;
      T* __restrict__ PBo = A.pb;
      for (long long j = gtid; j < N; j += stride) {
        if (copy)
          for (int n = 0; n < A.ndim; ++n) PBo[n * N + j] = Pin[n * N + j];
        if (R > 0) {
          T u[R > 0 ? R : 1];
#pragma unroll
          for (int c = 0; c < R; ++c) u[c] = __ldg(A.U + (long long)c * N + j);
          const T e = diag ? __ldg(A.d + j) : (T)1;
          int k = 0;
#pragma unroll
          for (int c = 0; c < R; ++c)
#pragma unroll
            for (int c2 = 0; c2 <= c; ++c2, ++k)
              acc[k] += diag ? (double)(u[c] * u[c2] / e) : (double)u[c] * (double)u[c2];
        }
      }
    } else if (phase == PH_DIV) {
      nv = R;
      T* __restrict__ Aout = A.a;
      const T* __restrict__ V = A.v;
      if (A.wpm_only || A.reg == 0.0) {
        for (long long j = gtid; j < N; j += stride) Aout[j] = V[j];
      } else if (A.vx) {
        div_vec<T, R, TY, NACC>(A, s_div_src ? A.p : A.pb, seg_begin, seg_end, lane, warp, acc);
      } else {
        const T* __restrict__ F0 = s_div_src ? A.p : A.pb;
        const T* __restrict__ F1 = F0 + N;
        const T* __restrict__ F2 = F0 + 2 * N;
        const T* __restrict__ Dd = A.d;
        const T* __restrict__ Uu = A.U;
        const T reg = (T)A.reg;
        const int K1 = A.K1, K2 = A.K2, K3 = A.K3, nd = A.ndim;
        long long pos = seg_begin;
        while (pos < seg_end) {
          const long long tile = pos / K3;
          const int z0 = (int)(pos - tile * K3);
          const int z1 = (int)min((long long)K3, z0 + (seg_end - pos));
          pos += z1 - z0;
          const int x = (int)(tile % A.ntx) * TX + lane;
          const int y = (int)(tile / A.ntx) * TY + warp;
          if (x >= K1 || y >= K2) continue;
          long long j = (long long)z0 * A.plane + (long long)y * K1 + x;
          T prev3 = (nd >= 3 && z0 > 0) ? F2[j - A.plane] : (T)0;
#pragma unroll 2
          for (int z = z0; z < z1; ++z, j += A.plane) {
            // tv_ops.py:122-133 per dimension, dual_divergence :151-159 summed in order
            const T c1 = F0[j];
            const T l1 = x > 0 ? F0[j - 1] : (T)0;
            T dv = (x < K1 - 1 ? -c1 : (T)0) + l1;
            if (nd >= 2) {
              const T c2 = F1[j];
              const T l2 = y > 0 ? F1[j - K1] : (T)0;
              dv += (y < K2 - 1 ? -c2 : (T)0) + l2;
            }
            if (nd >= 3) {
              const T c3 = F2[j];
              dv += (z < K3 - 1 ? -c3 : (T)0) + (z > 0 ? prev3 : (T)0);
              prev3 = c3;
            }
            const T e = diag ? __ldg(Dd + j) : tauT;
            const T de = dv * rcp(e);
            Aout[j] = __ldg(V + j) - reg * de;
#pragma unroll
            for (int c = 0; c < R; ++c) acc[c] += (double)__ldg(Uu + (long long)c * N + j) * (double)(diag ? de : dv);
          }
        }
      }
    } else if (phase == PH_NEWTON) {
      // phi(beta) partials U^T (wv - clamp(z)) and U_A^T D_A^-1 U_A (wpm.py:150-167)
      nv = NV<R>::newton;
      const T* __restrict__ Aa = A.a;
      auto body = [&](T av, T e, const T (&u)[R > 0 ? R : 1], T lo, T hi) {
        T wv, z;
        shift<T, R>(av, e, u, s_gw, s_beta, sg, wv, z);
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
      };
      if (A.vec) {
        const long long N4 = N >> 2;
#pragma unroll 2
        for (long long q4 = gtid; q4 < N4; q4 += stride) {
          const long long j = q4 << 2;
          T av[4], e[4], u[R > 0 ? R : 1][4], lo[4], hi[4];
          Vec4<T>::rw(Aa + j, av);
          if (diag) Vec4<T>::ro(A.d + j, e);
          else e[0] = e[1] = e[2] = e[3] = tauT;
#pragma unroll
          for (int c = 0; c < R; ++c) Vec4<T>::ro(A.U + (long long)c * N + j, u[c]);
          if (A.lo_arr) Vec4<T>::ro(A.lo_arr + j, lo);
          else lo[0] = lo[1] = lo[2] = lo[3] = (T)A.lo;
          if (A.hi_arr) Vec4<T>::ro(A.hi_arr + j, hi);
          else hi[0] = hi[1] = hi[2] = hi[3] = (T)A.hi;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            T uk[R > 0 ? R : 1];
#pragma unroll
            for (int c = 0; c < R; ++c) uk[c] = u[c][k];
            body(av[k], e[k], uk, lo[k], hi[k]);
          }
        }
      } else {
        for (long long j = gtid; j < N; j += stride) {
          T u[R > 0 ? R : 1];
#pragma unroll
          for (int c = 0; c < R; ++c) u[c] = __ldg(A.U + (long long)c * N + j);
          body(Aa[j], diag ? __ldg(A.d + j) : tauT, u, A.lo_arr ? __ldg(A.lo_arr + j) : (T)A.lo,
               A.hi_arr ? __ldg(A.hi_arr + j) : (T)A.hi);
        }
      }
    } else if (phase == PH_DUAL) {
      // dual_tv_solver.py:225-239: P_next = Proj(P_bar + step D q), momentum
      nv = 2;
      const T step = (T)A.step, mom = s_mom;
      T* __restrict__ P0 = A.p;
      T* __restrict__ PB0 = A.pb;
      const QEval<T, R> qv{A.a, A.d, A.U, A.lo_arr, A.hi_arr, N, tauT, (T)A.lo, (T)A.hi, sg, s_gz};
      const int K1 = A.K1, K2 = A.K2, K3 = A.K3, nd = A.ndim;
      const bool iso = A.mode == BQ_TV_ISO;
      long long pos = A.vx ? seg_end : seg_begin;
      if (A.vx) dual_vec<T, R, TY, NACC>(A, qv, step, mom, seg_begin, seg_end, lane, warp, acc);
      while (pos < seg_end) {
        const long long tile = pos / K3;
        const int z0 = (int)(pos - tile * K3);
        const int z1 = (int)min((long long)K3, z0 + (seg_end - pos));
        pos += z1 - z0;
        const int x = (int)(tile % A.ntx) * TX + lane;
        const int y = (int)(tile / A.ntx) * TY + warp;
        if (y >= K2) continue;  // whole warp leaves together
        const bool act = x < K1;
        const bool has_r = x < K1 - 1;
        const bool has_y = nd >= 2 && y < K2 - 1;
        long long j = (long long)z0 * A.plane + (long long)y * K1 + x;
        T qc = act ? qv(j) : (T)0;
#pragma unroll 2
        for (int z = z0; z < z1; ++z, j += A.plane) {
          const bool has_up = nd >= 3 && z < K3 - 1;
          const T qu = (act && has_up) ? qv(j + A.plane) : (T)0;
          const T qy = (act && has_y) ? qv(j + K1) : (T)0;
          T qr = __shfl_down_sync(0xffffffffu, qc, 1);
          if (act) {
            if (has_r && lane == 31) qr = qv(j + 1);
            T g[3];
            g[0] = has_r ? qr - qc : (T)0;
            g[1] = has_y ? qy - qc : (T)0;
            g[2] = has_up ? qu - qc : (T)0;
            T w[3], po[3];
#pragma unroll
            for (int n = 0; n < 3; ++n) {
              if (n < nd) {
                po[n] = P0[n * N + j];
                w[n] = PB0[n * N + j] + step * g[n];
              } else {
                po[n] = 0;
                w[n] = 0;
              }
            }
            if (iso) {
              T ss = w[0] * w[0];
              if (nd >= 2) ss += w[1] * w[1];
              if (nd >= 3) ss += w[2] * w[2];
              ball(w, ss);
            } else {
#pragma unroll
              for (int n = 0; n < 3; ++n) w[n] = clampv(w[n], (T)-1, (T)1);
            }
#pragma unroll
            for (int n = 0; n < 3; ++n) {
              if (n < nd) {
                const T df = w[n] - po[n];
                acc[0] += (double)df * (double)df;
                acc[1] += (double)po[n] * (double)po[n];
                P0[n * N + j] = w[n];
                PB0[n * N + j] = w[n] + mom * df;
              }
            }
          }
          qc = qu;
        }
      }
    } else if (phase == PH_FINAL) {
      nv = 0;
      const QEval<T, R> qv{A.a, A.d, A.U, A.lo_arr, A.hi_arr, N, tauT, (T)A.lo, (T)A.hi, sg, s_gz};
      T* __restrict__ X = A.x;
      for (long long j = gtid; j < N; j += stride) X[j] = qv(j);
    }

    // ---- barrier + fused deterministic reduction -------------------------
    const int cur = phase;
    if (cur != PH_FINAL) {
      if (nv > 0) block_sum_to<NT, NACC>(acc, nv, s_bv, s_scr);
      if (threadIdx.x < nv) A.partials[(size_t)blockIdx.x * kMaxVals + threadIdx.x] = s_bv[threadIdx.x];
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        const unsigned old = atomicAdd(A.bar, 1u);
        s_flag = (old == gridDim.x - 1) ? 1 : 0;
        if (s_flag) {
          __threadfence();
          const double t_arr = __longlong_as_double((long long)global_ns());
          s_red[kMaxVals - 1] = t_arr;
          __stcg(&A.red[kMaxVals - 1], t_arr);
        }
      }
      __syncthreads();
      if (s_flag == 1) {
        // last block: fixed-order reduction over blocks, publish, release
        for (int k = warp; k < nv; k += NT / 32) {
          double s = 0.0;
          for (unsigned b = lane; b < gridDim.x; b += 32) s += __ldcg(&A.partials[(size_t)b * kMaxVals + k]);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
          if (lane == 0) {
            s_red[k] = s;
            __stcg(&A.red[k], s);
          }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          A.bar[0] = 0;
          __threadfence();
          atomicAdd(A.bar + 1, 1u);
        }
      } else {
        if (threadIdx.x == 0) {
          const uint64_t t0 = global_ns();
          unsigned spins = 0;
          while (ld_acquire_u32(A.bar + 1) == my_gen) {
            __nanosleep(32);
            if (((++spins) & 1023u) == 0 && global_ns() - t0 > 20ull * 1000000000ull) {
              s_flag = -1;  // timeout
              break;
            }
          }
          __threadfence();
        }
        __syncthreads();
        if (s_flag == -1) {
          if (blockIdx.x == 0 && threadIdx.x == 0) A.report->status = BQ_ETIMEOUT;
          break;
        }
        if (threadIdx.x < nv) s_red[threadIdx.x] = __ldcg(&A.red[threadIdx.x]);
        if (threadIdx.x == NT - 1) s_red[kMaxVals - 1] = __ldcg(&A.red[kMaxVals - 1]);
      }
      my_gen += 1;
      __syncthreads();
    }
    // ---- redundant controller on the block's shared state ----------------
    if (threadIdx.x == 0) {
      controller<T, R>(A, s_c, cur, s_red, blockIdx.x == 0);
      s_phase = s_c.phase;
      s_div_src = s_c.div_src;
      s_mom = (T)s_c.mom;
      for (int i = 0; i < R; ++i) {
        s_gw[i] = (T)s_c.gw[i];
        s_beta[i] = (T)s_c.beta[i];
        s_gz[i] = (T)(s_c.gw[i] - s_c.beta[i]);
      }
    }
    __syncthreads();
    phase = s_phase;
    if (phase == PH_DONE) break;
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
bool aligned16(const void* p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; }

template <typename T, int R>
int launch(bq_ctx* ctx, const bq_wtv_desc& D, int wpm_only, cudaStream_t st) {
  constexpr int NT = Cfg<T, R>::NT;
  constexpr int TY = Cfg<T, R>::TY;
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
  BQ_STREAM_WS(sw, ctx, st);
  A.partials = sw->ws.partials;
  A.red = (double*)sw->ws.ctl;
  A.bar = sw->ws.barrier;
  A.vec = (A.N % 4 == 0) && aligned16(D.a) && aligned16(D.d) && aligned16(D.U) && aligned16(D.lo_arr) &&
          aligned16(D.hi_arr);

  auto kern = wtv_prox_kernel<T, R>;
  int per_sm = 0;
  BQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, 0));
  BQ_CHECK(per_sm > 0, BQ_ECUDA, "wtv_prox: kernel does not fit on an SM");
  per_sm = std::min(per_sm, Cfg<T, R>::MINB);
  const long long max_blocks = std::min<long long>((long long)per_sm * ctx->num_sms, kMaxBlocks);
  // small problems: fewer blocks -> cheaper barriers
  const long long want = std::max<long long>(1, (A.N + 4LL * NT - 1) / (4LL * NT));
  const int G = (int)std::min<long long>(max_blocks, want);
  A.vx = A.vec && (A.K1 % 4 == 0) && aligned16(D.p) && aligned16(D.pb) && aligned16(D.v);
  const int tx = A.vx ? TXV : TX;
  A.ntx = (A.K1 + tx - 1) / tx;
  A.nty = (A.K2 + TY - 1) / TY;
  A.tile_planes = (long long)A.ntx * A.nty * A.K3;

  BQ_CUDA(cudaMemsetAsync(sw->ws.barrier, 0, 2 * sizeof(unsigned), st));
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
  BQ_CHECK(D.dims[0] < (1 << 30) && D.dims[1] < (1 << 30) && D.dims[2] < (1 << 30), BQ_EINVAL, "side too large");
  BQ_CHECK(D.dtype == BQ_F32 || D.dtype == BQ_F64, BQ_EINVAL, "dtype must be BQ_F32 or BQ_F64");
  BQ_CHECK(D.sign == 1 || D.sign == -1, BQ_EINVAL, "sign must be +1 or -1, got %d", D.sign);
  BQ_CHECK(D.d != nullptr || D.tau > 0 || D.dev_metric, BQ_EINVAL, "tau must be positive, got %g", D.tau);
  BQ_CHECK(!D.dev_metric || (D.d == nullptr && !wpm_only), BQ_EINVAL, "dev_metric needs a scalar-tau prox");
  BQ_CHECK(D.reg >= 0, BQ_EINVAL, "reg must be nonnegative");
  BQ_CHECK(D.rank == 0 || D.U != nullptr, BQ_EINVAL, "U is required for rank > 0");
  BQ_CHECK(D.v && D.x && D.a && D.report, BQ_EINVAL, "v, x, a and report are required");
  BQ_CHECK(D.newton_max_iter >= 0, BQ_EINVAL, "newton_max_iter must be >= 0");
  if (!wpm_only) {
    BQ_CHECK(D.eps > 0, BQ_EINVAL, "eps must be positive");
    BQ_CHECK(D.max_iter >= 1, BQ_EINVAL, "max_iter must be >= 1");
    BQ_CHECK(D.p && D.pb, BQ_EINVAL, "p and pb are required");
    BQ_CHECK(D.mode == BQ_TV_ISO || D.mode == BQ_TV_ANISO, BQ_EINVAL, "bad TV mode");
    BQ_CHECK(D.reg == 0 || D.step > 0 || D.dev_metric, BQ_EINVAL, "step must be positive");
  }
  return BQ_OK;
}

}  // namespace
bool fused_eligible(const bq_wtv_desc& D);
int fused_dispatch(bq_ctx* ctx, const bq_wtv_desc& D, int wpm_only, cudaStream_t st);
}  // namespace bq

extern "C" int bq_wtv_prox(bq_ctx* ctx, const bq_wtv_desc* desc, void* stream) {
  using namespace bq;
  BQ_CHECK(ctx && desc, BQ_EINVAL, "bq_wtv_prox: null argument");
  int rc = validate(*desc, false);
  if (rc) return rc;
  BQ_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (fused_eligible(*desc) && !getenv("BQ_PROX_GENERAL")) return fused_dispatch(ctx, *desc, 0, st);
  BQ_CHECK(!desc->dev_metric, BQ_EINVAL, "bq_wtv_prox: dev_metric needs the fused kernel (K1 in {4..128 dividing "
           "128, 256}, 16-byte aligned fields, scalar bounds)");
  return desc->dtype == BQ_F32 ? dispatch_rank<float>(ctx, *desc, 0, st)
                               : dispatch_rank<double>(ctx, *desc, 0, st);
}

extern "C" int bq_wpm_box(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t rank, int32_t sign, double tau,
                          const void* d, const void* U, const void* x, double lo, double hi, const void* lo_arr,
                          const void* hi_arr, double* beta_inout, double newton_eps, int32_t newton_max_iter,
                          void* x_out, void* a_scratch, void* report, void* stream) {
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
  D.tau = tau;
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
