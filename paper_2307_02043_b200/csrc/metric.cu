// metric.cu — metric algebra, SR1 estimate, v_k, dots and TV value.
//
// Replaces (paths under /root/reference/pkg/src/tvqn/):
//   wpm.py:50-56     DiagPlusLowRank capacitance I +/- U^T U / tau   -> bq_metric_gram
//   wpm.py:81-89     apply_metric                                      -> bq_metric_apply(inverse=0)
//   wpm.py:92-106    apply_metric_inverse (Woodbury)                   -> bq_metric_apply(inverse=1)
//   hessian_sr1.py:52-101 estimate_sr1                                 -> bq_sr1
//   solvers.py:80-89 compute_v_k                                       -> bq_vk
//   tv_ops.py:162-167 tv_value                                         -> bq_tv_value
//
// All reductions are "last block done": every block writes its partial
// vector, the last block to arrive sums them in block order (deterministic,
// no float atomics, no co-residency requirement) and runs a tiny scalar
// epilogue.  Scalars stay on the device, so a GPU-resident outer loop never
// syncs with the host.
#include <algorithm>

#include "common.cuh"
#include "reduce.cuh"

namespace bq {
namespace {

constexpr int NT = 256;
constexpr int MAXB = 1184;  // 148 SMs x 8

int grid_for(bq_ctx* ctx, long long n) {
  long long want = (n + 4LL * NT - 1) / (4LL * NT);
  return (int)std::max<long long>(1, std::min<long long>(want, std::min(MAXB, ctx->num_sms * 4)));
}


// cap = I + sign gram_scaled ; chol in place (lower).  Single thread.
__device__ bool cap_chol(const double* gram, int r, int sign, double tau, bool diag, double* L) {
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) L[i * r + j] = (i == j ? 1.0 : 0.0) + sign * (diag ? gram[i * r + j] : gram[i * r + j] / tau);
  for (int j = 0; j < r; ++j) {
    double s = L[j * r + j];
    for (int k = 0; k < j; ++k) s -= L[j * r + k] * L[j * r + k];
    if (!(s > 0.0)) return false;
    double l = sqrt(s);
    L[j * r + j] = l;
    for (int i = j + 1; i < r; ++i) {
      double t = L[i * r + j];
      for (int k = 0; k < j; ++k) t -= L[i * r + k] * L[j * r + k];
      L[i * r + j] = t / l;
    }
  }
  return true;
}
__device__ void chol_solve_l(const double* L, int r, double* b) {
  for (int i = 0; i < r; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= L[i * r + k] * b[k];
    b[i] = s / L[i * r + i];
  }
  for (int i = r - 1; i >= 0; --i) {
    double s = b[i];
    for (int k = i + 1; k < r; ++k) s -= L[k * r + i] * b[k];
    b[i] = s / L[i * r + i];
  }
}

// ------------------------------- gram -------------------------------------
template <typename T, int R>
__global__ void __launch_bounds__(NT) gram_kernel(long long n, const T* __restrict__ d, const T* __restrict__ U,
                                                  double* out, RedWs ws) {
  constexpr int NA = R * (R + 1) / 2 > 0 ? R * (R + 1) / 2 : 1;
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  double acc[NA];
#pragma unroll
  for (int k = 0; k < NA; ++k) acc[k] = 0.0;
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT) {
    T u[R];
#pragma unroll
    for (int c = 0; c < R; ++c) u[c] = U[c * n + j];
    const T e = d ? d[j] : (T)1;
    int k = 0;
#pragma unroll
    for (int c = 0; c < R; ++c)
#pragma unroll
      for (int c2 = 0; c2 <= c; ++c2, ++k) acc[k] += d ? (double)(u[c] * u[c2] / e) : (double)u[c] * (double)u[c2];
  }
  if (last_block_reduce<NT, NA>(acc, R * (R + 1) / 2, ws, red, scr) && threadIdx.x == 0) {
    int k = 0;
    for (int c = 0; c < R; ++c)
      for (int c2 = 0; c2 <= c; ++c2, ++k) out[c * R + c2] = out[c2 * R + c] = red[k];
  }
}

// --------------------------- apply / inverse -------------------------------
// pass 1: rhs = U^T (D^-1 x)  (inverse)  or  U^T x  (apply)
template <typename T, int R>
__global__ void __launch_bounds__(NT) utx_kernel(long long n, const T* __restrict__ d, const T* __restrict__ U,
                                                 const T* __restrict__ x, int scale_by_d, double* out, RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  double acc[R];
#pragma unroll
  for (int k = 0; k < R; ++k) acc[k] = 0.0;
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT) {
    T xv = x[j];
    if (scale_by_d && d) xv = xv / d[j];
#pragma unroll
    for (int c = 0; c < R; ++c) acc[c] += (double)U[c * n + j] * (double)xv;
  }
  if (last_block_reduce<NT, R>(acc, R, ws, red, scr) && threadIdx.x < R) out[threadIdx.x] = red[threadIdx.x];
}

// pass 2: out = W x = D x + sign U (U^T x)      (apply)
//         out = W^-1 x = D^-1 x - sign D^-1 U cap^-1 rhs   (inverse; scalar: rhs/tau^2 form)
template <typename T, int R>
__global__ void __launch_bounds__(NT) metric_out_kernel(long long n, int sign, double tau, const T* __restrict__ d,
                                                        const T* __restrict__ U, const double* gram,
                                                        const double* rhs, int inverse, const T* __restrict__ x,
                                                        T* __restrict__ out, int* status) {
  __shared__ T coef[R > 0 ? R : 1];
  if (threadIdx.x == 0) {
    double b[R > 0 ? R : 1];
    for (int i = 0; i < R; ++i) b[i] = rhs[i];
    if (inverse) {
      double L[R * R > 0 ? R * R : 1];
      if (!cap_chol(gram, R, sign, tau, d != nullptr, L)) {
        if (blockIdx.x == 0 && status) *status = BQ_ENOTPD;
      } else {
        chol_solve_l(L, R, b);
      }
    }
    for (int i = 0; i < R; ++i) coef[i] = (T)b[i];
  }
  __syncthreads();
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT) {
    const T xv = x[j];
    T uc = 0;
#pragma unroll
    for (int c = 0; c < R; ++c) uc += U[c * n + j] * coef[c];
    if (!inverse) {
      // wpm.py:84-88: tau*x + sign*U(U^T x)
      const T e = d ? d[j] : (T)tau;
      out[j] = (R > 0) ? e * xv + (T)sign * uc : e * xv;
    } else if (d) {
      const T e = d[j];
      out[j] = (R > 0) ? xv / e - (T)sign * uc / e : xv / e;
    } else {
      // wpm.py:99-105: x/tau - sign*(U coef)/tau^2
      const T t = (T)tau;
      out[j] = (R > 0) ? xv / t - (T)sign * uc / (t * t) : xv / t;
    }
  }
}

// ------------------------------- dots -------------------------------------
struct DotPtrs {
  const void* a[8];
  const void* b[8];
};
template <typename T, int C>
__global__ void __launch_bounds__(NT) dots_kernel(long long n, DotPtrs P, double* out, RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  double acc[C];
#pragma unroll
  for (int k = 0; k < C; ++k) acc[k] = 0.0;
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT) {
#pragma unroll
    for (int k = 0; k < C; ++k) acc[k] += (double)((const T*)P.a[k])[j] * (double)((const T*)P.b[k])[j];
  }
  if (last_block_reduce<NT, C>(acc, C, ws, red, scr) && threadIdx.x < C) out[threadIdx.x] = red[threadIdx.x];
}

// ------------------------------- SR1 --------------------------------------
// est layout (device doubles): [0] tau [1] has_u [2] sm [3] curv [4] mm [5] nnz(s)
//                              [6] ||s|| [7] ||resid|| [8] status
template <typename T>
__global__ void __launch_bounds__(NT) sr1_pass1(long long n, const T* __restrict__ s, const T* __restrict__ m,
                                                double gamma, double alpha, double* est, RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  double acc[3] = {0.0, 0.0, 0.0};
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT) {
    const double sv = s[j], mv = m[j];
    acc[0] += sv * mv;
    acc[1] += mv * mv;
    acc[2] += (sv != 0.0) ? 1.0 : 0.0;
  }
  if (last_block_reduce<NT, 3>(acc, 3, ws, red, scr) && threadIdx.x == 0) {
    // hessian_sr1.py:90-95
    const double sm = red[0], mm = red[1];
    est[2] = sm;
    est[4] = mm;
    est[5] = red[2];
    est[8] = (red[2] == 0.0) ? BQ_EINVAL : 0.0;
    double tau;
    int stage;  // 0: fallback alpha, 1: tau only (decided in pass 2), 2: needs pass 2
    if (sm == 0.0) {
      tau = alpha, stage = 0;
    } else {
      tau = gamma * mm / sm;
      if (tau < 0.0) tau = alpha, stage = 0;
      else stage = 2;
    }
    est[0] = tau;
    est[1] = (stage == 2) ? -1.0 : 0.0;  // -1: undecided
  }
}
template <typename T>
__global__ void __launch_bounds__(NT) sr1_pass2(long long n, const T* __restrict__ s, const T* __restrict__ m,
                                                double* est, RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  const double und = est[1];
  double acc[3] = {0.0, 0.0, 0.0};
  if (und < 0.0) {
    const T tau = (T)est[0];
    for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT) {
      const T sv = s[j];
      const T r = m[j] - tau * sv;
      acc[0] += (double)r * (double)sv;
      acc[1] += (double)sv * (double)sv;
      acc[2] += (double)r * (double)r;
    }
  }
  if (last_block_reduce<NT, 3>(acc, 3, ws, red, scr) && threadIdx.x == 0 && und < 0.0) {
    // hessian_sr1.py:96-100 skip rule
    const double curv = red[0], ns = sqrt(red[1]), nr = sqrt(red[2]);
    est[3] = curv;
    est[6] = ns;
    est[7] = nr;
    const bool skip = (curv <= 1e-8 * ns * nr) || (curv <= 0.0);
    est[1] = skip ? 0.0 : 1.0;
  }
}
template <typename T>
__global__ void __launch_bounds__(NT) sr1_pass3(long long n, const T* __restrict__ s, const T* __restrict__ m,
                                                const double* est, T* __restrict__ u) {
  const bool has = est[1] > 0.0;
  const T tau = (T)est[0];
  const T inv = has ? (T)sqrt(est[3]) : (T)1;
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT)
    u[j] = has ? (m[j] - tau * s[j]) / inv : (T)0;
}

// ------------------------------- v_k --------------------------------------
struct VkPtrs {
  const void* x[8];
  const void* g[8];
  const void* u[8];
  double tau[8];
};
// pass 1: u_t^T x_t
template <typename T>
__global__ void __launch_bounds__(NT) vk_pass1(long long n, int count, VkPtrs P, double* out, RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  double acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.0;
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < count && P.u[k]) acc[k] += (double)((const T*)P.u[k])[j] * (double)((const T*)P.x[k])[j];
  }
  if (last_block_reduce<NT, 8>(acc, count, ws, red, scr) && threadIdx.x < count) out[threadIdx.x] = red[threadIdx.x];
}
// pass 2: acc = sum_t (tau_t x_t + u_t (u_t^T x_t) - step g_t) (solvers.py:86-88), plus
//         Woodbury rhs = U_w^T acc (U_w = aggregated columns)
template <typename T, int R>
__global__ void __launch_bounds__(NT) vk_pass2(long long n, int count, VkPtrs P, const double* utx, double step,
                                               const T* __restrict__ Uw, T* __restrict__ accbuf, double* rhs,
                                               RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  __shared__ T s_utx[8], s_tau[8];
  if (threadIdx.x < 8) {
    s_utx[threadIdx.x] = (threadIdx.x < count) ? (T)utx[threadIdx.x] : (T)0;
    s_tau[threadIdx.x] = (T)P.tau[threadIdx.x];
  }
  __syncthreads();
  double acc[R > 0 ? R : 1];
#pragma unroll
  for (int k = 0; k < (R > 0 ? R : 1); ++k) acc[k] = 0.0;
  const T stp = (T)step;
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT) {
    T a = 0;
    for (int k = 0; k < count; ++k) {
      const T xv = ((const T*)P.x[k])[j];
      T bx = s_tau[k] * xv;  // Sr1Estimate.apply: tau*x (+ u*(u.x))
      if (P.u[k]) bx = bx + ((const T*)P.u[k])[j] * s_utx[k];
      a += bx - stp * ((const T*)P.g[k])[j];
    }
    accbuf[j] = a;
#pragma unroll
    for (int c = 0; c < R; ++c) acc[c] += (double)Uw[c * n + j] * (double)a;
  }
  if (last_block_reduce<NT, (R > 0 ? R : 1)>(acc, R, ws, red, scr) && threadIdx.x < R) rhs[threadIdx.x] = red[threadIdx.x];
}

// ------------------------------- TV value ---------------------------------
template <typename T>
__global__ void __launch_bounds__(NT) tv_kernel(int ndim, int K1, int K2, int K3, int mode, const T* __restrict__ x,
                                                double* out, RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  double acc[1] = {0.0};
  const long long n = (long long)K1 * K2 * K3, plane = (long long)K1 * K2;
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT) {
    const int xi = (int)(j % K1);
    const int yi = (int)((j / K1) % K2);
    const int zi = (int)(j / plane);
    const T c = x[j];
    const T g1 = (xi < K1 - 1) ? x[j + 1] - c : (T)0;
    const T g2 = (ndim >= 2 && yi < K2 - 1) ? x[j + K1] - c : (T)0;
    const T g3 = (ndim >= 3 && zi < K3 - 1) ? x[j + plane] - c : (T)0;
    if (mode == BQ_TV_ISO) {
      double ss = (double)g1 * g1;
      if (ndim >= 2) ss += (double)g2 * g2;
      if (ndim >= 3) ss += (double)g3 * g3;
      acc[0] += sqrt(ss);
    } else {
      acc[0] += fabs((double)g1) + fabs((double)g2) + fabs((double)g3);
    }
  }
  if (last_block_reduce<NT, 1>(acc, 1, ws, red, scr) && threadIdx.x == 0) out[0] = red[0];
}

}  // namespace
}  // namespace bq

using namespace bq;


// ---------------------------- wpm phi ---------------------------------------
// phi(beta) = U^T (x - clamp(x - sign D^-1 U beta)) + beta and the generalized
// Jacobian I + sign U_A^T D_A^-1 U_A over the strictly-inside set (wpm.py:150-167).
template <typename T, int R>
__global__ void __launch_bounds__(NT) phi_kernel(long long n, int sign, double tau, const T* __restrict__ d,
                                                 const T* __restrict__ U, const T* __restrict__ x, double lo,
                                                 double hi, const T* __restrict__ lo_a, const T* __restrict__ hi_a,
                                                 const double* beta, double* phi_out, double* jac_out, RedWs ws) {
  constexpr int NV = R + R * (R + 1) / 2;
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  __shared__ T b[R];
  if (threadIdx.x < R) b[threadIdx.x] = (T)beta[threadIdx.x];
  __syncthreads();
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT) {
    T u[R];
    T ub = (T)0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      u[k] = U[k * n + j];
      ub += u[k] * b[k];
    }
    const T xv = x[j];
    const T z = d ? xv - (T)sign * ub / d[j] : xv - (T)sign * ub / (T)tau;  // wpm.py:145-147
    const T l = lo_a ? lo_a[j] : (T)lo;
    const T h = hi_a ? hi_a[j] : (T)hi;
    const T r = xv - min(max(z, l), h);
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] += (double)(u[k] * r);
    if (z > l && z < h) {
      int m = R;
#pragma unroll
      for (int k = 0; k < R; ++k)
#pragma unroll
        for (int k2 = 0; k2 <= k; ++k2, ++m) acc[m] += d ? (double)(u[k] * u[k2] / d[j]) : (double)(u[k] * u[k2]);
    }
  }
  if (last_block_reduce<NT, NV>(acc, NV, ws, red, scr) && threadIdx.x == 0) {
    for (int k = 0; k < R; ++k) phi_out[k] = red[k] + beta[k];
    if (jac_out) {
      int m = R;
      for (int k = 0; k < R; ++k)
        for (int k2 = 0; k2 <= k; ++k2, ++m) {
          const double g = d ? red[m] : red[m] / tau;
          jac_out[k * R + k2] = jac_out[k2 * R + k] = (k == k2 ? 1.0 : 0.0) + sign * g;
        }
    }
  }
}


// --------------------- metric check (gram + min(d)) ---------------------------
// DiagPlusLowRank's construction-time validation in ONE small-footprint pass:
// min(d) (the positivity test and omega, D-6) and the gram U^T D^-1 U.  128
// threads and ~4 KB of shared memory per block, at most one block per SM: it
// fits beside a running persistent prox block (1 block / SM, ~200 KB smem), so
// the next problem's build can overlap the current solve (bench e2e).
constexpr int NTC = 128;
template <typename T, int R>
__global__ void __launch_bounds__(NTC, 16) check_kernel(long long n, const T* __restrict__ d, const T* __restrict__ U,
                                                       double* out, double* partials, unsigned* count) {
  constexpr int NA = R * (R + 1) / 2 > 0 ? R * (R + 1) / 2 : 1;
  __shared__ double s_w[NTC / 32][NA + 1];
  __shared__ int s_last;
  double acc[NA];
#pragma unroll
  for (int k = 0; k < NA; ++k) acc[k] = 0.0;
  double mn = INFINITY;
#pragma unroll 4
  for (long long j = (long long)blockIdx.x * NTC + threadIdx.x; j < n; j += (long long)gridDim.x * NTC) {
    const T e = d ? d[j] : (T)1;
    if (d) mn = (e == e) ? fmin(mn, (double)e) : -INFINITY;  // a NaN fails the d > 0 test
    if (R > 0) {
      T u[R > 0 ? R : 1];
#pragma unroll
      for (int c = 0; c < R; ++c) u[c] = U[c * n + j];
      int k = 0;
#pragma unroll
      for (int c = 0; c < R; ++c)
#pragma unroll
        for (int c2 = 0; c2 <= c; ++c2, ++k) acc[k] += d ? (double)(u[c] * u[c2] / e) : (double)u[c] * (double)u[c2];
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_down_sync(0xffffffffu, mn, o));
#pragma unroll
  for (int k = 0; k < NA; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_down_sync(0xffffffffu, acc[k], o);
  if (lane == 0) {
    s_w[warp][0] = mn;
    for (int k = 0; k < NA; ++k) s_w[warp][k + 1] = acc[k];
  }
  __syncthreads();
  if (threadIdx.x <= NA) {  // block partial, fixed warp order
    double v = s_w[0][threadIdx.x];
    for (int w = 1; w < NTC / 32; ++w) v = threadIdx.x == 0 ? fmin(v, s_w[w][0]) : v + s_w[w][threadIdx.x];
    partials[(size_t)blockIdx.x * kMaxVals + threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(count, 1u) == gridDim.x - 1;
    if (s_last) __threadfence();
  }
  __syncthreads();
  if (!s_last) return;
  if (threadIdx.x <= NA) {  // totals in block order (deterministic)
    double v = __ldcg(&partials[threadIdx.x]);
    for (unsigned b = 1; b < gridDim.x; ++b) {
      const double p = __ldcg(&partials[(size_t)b * kMaxVals + threadIdx.x]);
      v = threadIdx.x == 0 ? fmin(v, p) : v + p;
    }
    s_w[0][threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out[0] = s_w[0][0];
    int k = 0;
    for (int c = 0; c < R; ++c)
      for (int c2 = 0; c2 <= c; ++c2, ++k) out[1 + c * R + c2] = out[1 + c2 * R + c] = s_w[0][k + 1];
    *count = 0;
  }
}

#define RANK_SWITCH(r, BODY)                       \
  switch (r) {                                     \
    case 1: { constexpr int R = 1; BODY; } break;  \
    case 2: { constexpr int R = 2; BODY; } break;  \
    case 3: { constexpr int R = 3; BODY; } break;  \
    case 4: { constexpr int R = 4; BODY; } break;  \
    case 5: { constexpr int R = 5; BODY; } break;  \
    case 6: { constexpr int R = 6; BODY; } break;  \
    case 7: { constexpr int R = 7; BODY; } break;  \
    case 8: { constexpr int R = 8; BODY; } break;  \
    default: set_error("rank %d outside [1, 8]", r); return BQ_EINVAL; \
  }

extern "C" int bq_metric_gram(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t rank, double tau, const void* d,
                              const void* U, double* gram_out, void* stream) {
  BQ_CHECK(ctx && U && gram_out && n > 0, BQ_EINVAL, "bq_metric_gram: bad arguments");
  BQ_CHECK(d || tau > 0, BQ_EINVAL, "tau must be positive");
  cudaStream_t st = (cudaStream_t)stream;
  const int G = grid_for(ctx, n);
  BQ_STREAM_WS(sw, ctx, st);
  RedWs ws = red_ws(sw);
  if (dtype == BQ_F32) {
    RANK_SWITCH(rank, (gram_kernel<float, R><<<G, NT, 0, st>>>(n, (const float*)d, (const float*)U, gram_out, ws)));
  } else {
    RANK_SWITCH(rank, (gram_kernel<double, R><<<G, NT, 0, st>>>(n, (const double*)d, (const double*)U, gram_out, ws)));
  }
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_metric_apply(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t rank, int32_t sign, double tau,
                               const void* d, const void* U, const double* gram, int32_t inverse, const void* x,
                               void* out, void* stream) {
  BQ_CHECK(ctx && x && out && n > 0, BQ_EINVAL, "bq_metric_apply: bad arguments");
  BQ_CHECK(d || tau > 0, BQ_EINVAL, "tau must be positive");
  BQ_CHECK(sign == 1 || sign == -1, BQ_EINVAL, "sign must be +/-1");
  BQ_CHECK(rank == 0 || (U && (gram || !inverse)), BQ_EINVAL, "U (and gram for the inverse) required");
  cudaStream_t st = (cudaStream_t)stream;
  const int G = grid_for(ctx, n);
  BQ_STREAM_WS(sw, ctx, st);
  RedWs ws = red_ws(sw);
  double* rhs = sw->ws.scratch;
  int* status = (int*)(sw->ws.scratch + 64);
  if (rank == 0) {
    if (dtype == BQ_F32)
      metric_out_kernel<float, 0><<<G, NT, 0, st>>>(n, sign, tau, (const float*)d, nullptr, nullptr, nullptr, inverse,
                                                     (const float*)x, (float*)out, nullptr);
    else
      metric_out_kernel<double, 0><<<G, NT, 0, st>>>(n, sign, tau, (const double*)d, nullptr, nullptr, nullptr,
                                                      inverse, (const double*)x, (double*)out, nullptr);
  } else if (dtype == BQ_F32) {
    RANK_SWITCH(rank, (utx_kernel<float, R><<<G, NT, 0, st>>>(n, (const float*)d, (const float*)U, (const float*)x,
                                                               inverse, rhs, ws),
                       metric_out_kernel<float, R><<<G, NT, 0, st>>>(n, sign, tau, (const float*)d,
                                                                      (const float*)U, gram, rhs, inverse,
                                                                      (const float*)x, (float*)out, status)));
  } else {
    RANK_SWITCH(rank, (utx_kernel<double, R><<<G, NT, 0, st>>>(n, (const double*)d, (const double*)U,
                                                                (const double*)x, inverse, rhs, ws),
                       metric_out_kernel<double, R><<<G, NT, 0, st>>>(n, sign, tau, (const double*)d,
                                                                       (const double*)U, gram, rhs, inverse,
                                                                       (const double*)x, (double*)out, status)));
  }
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_dot(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t count, const void* const* a_ptrs,
                      const void* const* b_ptrs, double* dots_out, void* stream) {
  BQ_CHECK(ctx && a_ptrs && b_ptrs && dots_out && n > 0, BQ_EINVAL, "bq_dot: bad arguments");
  BQ_CHECK(count >= 1 && count <= 8, BQ_EINVAL, "bq_dot: count must be 1..8");
  DotPtrs P{};
  for (int k = 0; k < count; ++k) P.a[k] = a_ptrs[k], P.b[k] = b_ptrs[k];
  cudaStream_t st = (cudaStream_t)stream;
  const int G = grid_for(ctx, n);
  BQ_STREAM_WS(sw, ctx, st);
  RedWs ws = red_ws(sw);
#define DOTS(T)                                                                   \
  switch (count) {                                                                \
    case 1: dots_kernel<T, 1><<<G, NT, 0, st>>>(n, P, dots_out, ws); break;       \
    case 2: dots_kernel<T, 2><<<G, NT, 0, st>>>(n, P, dots_out, ws); break;       \
    case 3: dots_kernel<T, 3><<<G, NT, 0, st>>>(n, P, dots_out, ws); break;       \
    case 4: dots_kernel<T, 4><<<G, NT, 0, st>>>(n, P, dots_out, ws); break;       \
    default: dots_kernel<T, 8><<<G, NT, 0, st>>>(n, P, dots_out, ws); break;      \
  }
  // counts 5..7 run the 8-wide kernel; the padding slots re-read a[0]*b[0]
  // and are never written out (only `count` totals are reduced).
  for (int k = count; k < 8; ++k) P.a[k] = a_ptrs[0], P.b[k] = b_ptrs[0];
  if (dtype == BQ_F32) {
    DOTS(float)
  } else {
    DOTS(double)
  }
#undef DOTS
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_sr1(bq_ctx* ctx, int32_t dtype, int64_t n, const void* s, const void* m, double gamma,
                      double alpha_fallback, void* u_out, double* est_out, void* stream) {
  BQ_CHECK(ctx && s && m && u_out && est_out && n > 0, BQ_EINVAL, "bq_sr1: bad arguments");
  BQ_CHECK(gamma > 0.0 && gamma < 1.0, BQ_EINVAL, "gamma must lie in (0, 1), got %g", gamma);
  BQ_CHECK(alpha_fallback > 0.0, BQ_EINVAL, "alpha_fallback must be positive, got %g", alpha_fallback);
  cudaStream_t st = (cudaStream_t)stream;
  const int G = grid_for(ctx, n);
  BQ_STREAM_WS(sw, ctx, st);
  RedWs ws = red_ws(sw);
  if (dtype == BQ_F32) {
    sr1_pass1<float><<<G, NT, 0, st>>>(n, (const float*)s, (const float*)m, gamma, alpha_fallback, est_out, ws);
    sr1_pass2<float><<<G, NT, 0, st>>>(n, (const float*)s, (const float*)m, est_out, ws);
    sr1_pass3<float><<<G, NT, 0, st>>>(n, (const float*)s, (const float*)m, est_out, (float*)u_out);
  } else {
    sr1_pass1<double><<<G, NT, 0, st>>>(n, (const double*)s, (const double*)m, gamma, alpha_fallback, est_out, ws);
    sr1_pass2<double><<<G, NT, 0, st>>>(n, (const double*)s, (const double*)m, est_out, ws);
    sr1_pass3<double><<<G, NT, 0, st>>>(n, (const double*)s, (const double*)m, est_out, (double*)u_out);
  }
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_vk(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t count, const void* const* xs,
                     const void* const* gs, const void* const* us, const double* taus, double step, int32_t rank,
                     int32_t sign, double tau_w, const void* U_w, const double* gram_w, void* acc_scratch,
                     void* v_out, void* stream) {
  BQ_CHECK(ctx && xs && gs && taus && acc_scratch && v_out && n > 0, BQ_EINVAL, "bq_vk: bad arguments");
  BQ_CHECK(count >= 1 && count <= 8, BQ_EINVAL, "bq_vk: 1..8 slots");
  BQ_CHECK(rank >= 0 && rank <= 8 && (rank == 0 || (U_w && gram_w)), BQ_EINVAL, "bq_vk: bad metric");
  BQ_CHECK(tau_w > 0, BQ_EINVAL, "bq_vk: the aggregated metric needs a positive scalar tau (no per-voxel d)");
  BQ_CHECK(sign == 1 || sign == -1, BQ_EINVAL, "bq_vk: sign must be +/-1");
  VkPtrs P{};
  for (int k = 0; k < count; ++k) {
    P.x[k] = xs[k];
    P.g[k] = gs[k];
    P.u[k] = us ? us[k] : nullptr;
    P.tau[k] = taus[k];
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int G = grid_for(ctx, n);
  BQ_STREAM_WS(sw, ctx, st);
  RedWs ws = red_ws(sw);
  double* utx = sw->ws.scratch + 128;
  double* rhs = sw->ws.scratch + 160;
  int* status = (int*)(sw->ws.scratch + 192);
  if (dtype == BQ_F32) {
    vk_pass1<float><<<G, NT, 0, st>>>(n, count, P, utx, ws);
    if (rank == 0) {
      vk_pass2<float, 0><<<G, NT, 0, st>>>(n, count, P, utx, step, nullptr, (float*)acc_scratch, rhs, ws);
      metric_out_kernel<float, 0><<<G, NT, 0, st>>>(n, sign, tau_w, nullptr, nullptr, nullptr, nullptr, 1,
                                                     (const float*)acc_scratch, (float*)v_out, nullptr);
    } else {
      RANK_SWITCH(rank, (vk_pass2<float, R><<<G, NT, 0, st>>>(n, count, P, utx, step, (const float*)U_w,
                                                               (float*)acc_scratch, rhs, ws),
                         metric_out_kernel<float, R><<<G, NT, 0, st>>>(n, sign, tau_w, nullptr, (const float*)U_w,
                                                                        gram_w, rhs, 1, (const float*)acc_scratch,
                                                                        (float*)v_out, status)));
    }
  } else {
    vk_pass1<double><<<G, NT, 0, st>>>(n, count, P, utx, ws);
    if (rank == 0) {
      vk_pass2<double, 0><<<G, NT, 0, st>>>(n, count, P, utx, step, nullptr, (double*)acc_scratch, rhs, ws);
      metric_out_kernel<double, 0><<<G, NT, 0, st>>>(n, sign, tau_w, nullptr, nullptr, nullptr, nullptr, 1,
                                                      (const double*)acc_scratch, (double*)v_out, nullptr);
    } else {
      RANK_SWITCH(rank, (vk_pass2<double, R><<<G, NT, 0, st>>>(n, count, P, utx, step, (const double*)U_w,
                                                                (double*)acc_scratch, rhs, ws),
                         metric_out_kernel<double, R><<<G, NT, 0, st>>>(n, sign, tau_w, nullptr,
                                                                         (const double*)U_w, gram_w, rhs, 1,
                                                                         (const double*)acc_scratch,
                                                                         (double*)v_out, status)));
    }
  }
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_tv_value(bq_ctx* ctx, int32_t dtype, int32_t ndim, const int64_t* dims, int32_t mode,
                           const void* x, double* out, void* stream) {
  BQ_CHECK(ctx && dims && x && out && ndim >= 1 && ndim <= 3, BQ_EINVAL, "bq_tv_value: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const long long n = dims[0] * dims[1] * dims[2];
  const int G = grid_for(ctx, n);
  BQ_STREAM_WS(sw, ctx, st);
  RedWs ws = red_ws(sw);
  if (dtype == BQ_F32)
    tv_kernel<float><<<G, NT, 0, st>>>(ndim, (int)dims[0], (int)dims[1], (int)dims[2], mode, (const float*)x, out, ws);
  else
    tv_kernel<double><<<G, NT, 0, st>>>(ndim, (int)dims[0], (int)dims[1], (int)dims[2], mode, (const double*)x, out,
                                        ws);
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_wpm_phi(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t rank, int32_t sign, double tau,
                          const void* d, const void* U, const void* x, double lo, double hi, const void* lo_arr,
                          const void* hi_arr, const double* beta, double* phi_out, double* jac_out, void* stream) {
  BQ_CHECK(ctx && U && x && beta && phi_out && n > 0, BQ_EINVAL, "bq_wpm_phi: bad arguments");
  BQ_CHECK(d || tau > 0, BQ_EINVAL, "tau must be positive");
  BQ_CHECK(sign == 1 || sign == -1, BQ_EINVAL, "sign must be +/-1");
  cudaStream_t st = (cudaStream_t)stream;
  const int G = grid_for(ctx, n);
  BQ_STREAM_WS(sw, ctx, st);
  RedWs ws = red_ws(sw);
  if (dtype == BQ_F32) {
    RANK_SWITCH(rank, (phi_kernel<float, R><<<G, NT, 0, st>>>(n, sign, tau, (const float*)d, (const float*)U,
                                                               (const float*)x, lo, hi, (const float*)lo_arr,
                                                               (const float*)hi_arr, beta, phi_out, jac_out, ws)));
  } else {
    RANK_SWITCH(rank, (phi_kernel<double, R><<<G, NT, 0, st>>>(n, sign, tau, (const double*)d, (const double*)U,
                                                                (const double*)x, lo, hi, (const double*)lo_arr,
                                                                (const double*)hi_arr, beta, phi_out, jac_out, ws)));
  }
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_metric_check(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t rank, const void* d, const void* U,
                               double* out, void* stream) {
  BQ_CHECK(ctx && out && n > 0 && rank >= 0 && rank <= BQ_MAX_RANK && (rank == 0 || U), BQ_EINVAL,
           "bq_metric_check: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  BQ_STREAM_WS(sw, ctx, st);
  const int G = (int)std::max<long long>(1, std::min<long long>((n + NTC * 8 - 1) / (NTC * 8), ctx->num_sms));
  double* part = sw->ws.partials;
  unsigned* cnt = sw->ws.barrier + 8;
  // the carveout of a running persistent prox (maximum shared memory): a block
  // with another preferred split could not share the SM with it
#define CHECK_CASE(RR)                                                                                              \
  case RR:                                                                                                          \
    if (dtype == BQ_F32) {                                                                                          \
      cudaFuncSetAttribute(check_kernel<float, RR>, cudaFuncAttributePreferredSharedMemoryCarveout,                 \
                           cudaSharedmemCarveoutMaxShared);                                                         \
      check_kernel<float, RR><<<G, NTC, 0, st>>>(n, (const float*)d, (const float*)U, out, part, cnt);             \
    } else {                                                                                                        \
      cudaFuncSetAttribute(check_kernel<double, RR>, cudaFuncAttributePreferredSharedMemoryCarveout,                \
                           cudaSharedmemCarveoutMaxShared);                                                         \
      check_kernel<double, RR><<<G, NTC, 0, st>>>(n, (const double*)d, (const double*)U, out, part, cnt);          \
    }                                                                                                               \
    break;
  switch (rank) {
    CHECK_CASE(0) CHECK_CASE(1) CHECK_CASE(2) CHECK_CASE(3) CHECK_CASE(4) CHECK_CASE(5) CHECK_CASE(6) CHECK_CASE(7)
    CHECK_CASE(8)
  }
#undef CHECK_CASE
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}
