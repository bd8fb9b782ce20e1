// bqnpm_step.cu — the aggregated metric and the centre v_k of one BQNPM outer
// iteration k > K_s with every scalar on the device (no host round trip), for
// the GPU-resident / CUDA-graph outer loop of solvers.py.
//
// Replaces (paths under /root/reference/pkg/src/tvqn/):
//   solvers.py:67-77  aggregate_metric: tau = sum_t tau_t, U = the nonzero u_t
//                     stacked in slot order (rank = number of accepted SR1 terms)
//   solvers.py:80-89  compute_v_k: v = W^-1 sum_t (tau_t x_t + u_t (u_t^T x_t) - a g_t)
//   wpm.py:92-106     the Woodbury inverse of W = tau I + U U^T
//
// The host does not know which SR1 terms were accepted (that is decided on
// the device by bq_sr1), so U is written compacted into a FIXED count x N
// buffer: the accepted columns first, in slot order, zero columns after.  A
// zero column leaves W, the Woodbury solve and the prox's Newton iteration
// unchanged (its beta entry stays 0), so the prox runs at the fixed rank
// `count` and reads tau / the effective rank from `meta` (bq_wtv_desc::
// dev_metric).  Three launches:
//   pass 1  u_t^T x_t and the slot gram u_t^T u_s (deterministic block
//           reduction); epilogue: tau_w, the compaction map, Cholesky of
//           cap = I + U^T U / tau_w
//   pass 2  acc = sum_t (tau_t x_t + u_t (u_t^T x_t) - a g_t), the compacted U
//           copy, rhs = U^T acc; epilogue: coef = cap^-1 rhs
//   pass 3  v = acc / tau - U coef / tau^2     (the reference's operation order)
#include <algorithm>

#include "common.cuh"
#include "reduce.cuh"

namespace bq {
namespace {

constexpr int NT = 256;
constexpr int M_TAU = 0, M_RANK = 1, M_MAP = 8, M_UTX = 16, M_CHOL = 24, M_COEF = 88, M_STATUS = 96;

struct SlotPtrs {
  const void* x[8];
  const void* g[8];
  const void* u[8];
  const double* est[8];
};

template <typename T>
__global__ void __launch_bounds__(NT) agg_pass1(long long n, int count, SlotPtrs P, double* meta, RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  constexpr int NV = 8 + 36;
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT) {
    T u[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) u[t] = t < count ? ((const T*)P.u[t])[j] : (T)0;
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (t < count) acc[t] += (double)u[t] * (double)((const T*)P.x[t])[j];
    int k = 8;
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b <= a; ++b, ++k)
        if (a < count) acc[k] += (double)u[a] * (double)u[b];
  }
  const int nv = 8 + count * (count + 1) / 2;
  if (last_block_reduce<NT, NV>(acc, nv, ws, red, scr) && threadIdx.x == 0) {
    double tau = 0.0;  // sum(s.hess.tau for s in slots), in slot order
    int map[8], r = 0;
    for (int t = 0; t < count; ++t) {
      tau += P.est[t][0];
      if (P.est[t][1] > 0.0) map[r++] = t;
      meta[M_UTX + t] = red[t];
    }
    meta[M_TAU] = tau;
    meta[M_RANK] = (double)r;
    for (int c = 0; c < 8; ++c) meta[M_MAP + c] = c < r ? (double)map[c] : -1.0;
    // cap = I + U^T U / tau over the accepted columns (identity beyond r), Cholesky in place
    double L[64];
    for (int a = 0; a < count; ++a)
      for (int b = 0; b < count; ++b) {
        double g = 0.0;
        if (a < r && b < r) {
          const int ta = map[a], tb = map[b];
          const int hi = ta > tb ? ta : tb, lo = ta > tb ? tb : ta;
          g = red[8 + hi * (hi + 1) / 2 + lo] / tau;
        }
        L[a * count + b] = (a == b ? 1.0 : 0.0) + g;
      }
    int ok = 1;
    for (int j = 0; j < count; ++j) {
      double s = L[j * count + j];
      for (int k = 0; k < j; ++k) s -= L[j * count + k] * L[j * count + k];
      if (!(s > 0.0)) { ok = 0; s = 1.0; }
      const double l = sqrt(s);
      L[j * count + j] = l;
      for (int i = j + 1; i < count; ++i) {
        double t = L[i * count + j];
        for (int k = 0; k < j; ++k) t -= L[i * count + k] * L[j * count + k];
        L[i * count + j] = t / l;
      }
    }
    for (int i = 0; i < count * count; ++i) meta[M_CHOL + i] = L[i];
    meta[M_STATUS] = ok ? 0.0 : (double)BQ_ENOTPD;
  }
}

template <typename T>
__global__ void __launch_bounds__(NT) agg_pass2(long long n, int count, SlotPtrs P, double step, double* meta,
                                                T* __restrict__ Uc, T* __restrict__ accbuf, RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  __shared__ T s_utx[8], s_tau[8];
  __shared__ int s_map[8], s_r;
  if (threadIdx.x < 8) {
    const int t = threadIdx.x;
    s_utx[t] = t < count ? (T)meta[M_UTX + t] : (T)0;
    s_tau[t] = t < count ? (T)P.est[t][0] : (T)0;
    s_map[t] = (int)meta[M_MAP + t];
  }
  if (threadIdx.x == 0) s_r = (int)meta[M_RANK];
  __syncthreads();
  const int r = s_r;
  double acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.0;
  const T stp = (T)step;
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT) {
    T a = 0;
    for (int t = 0; t < count; ++t) {  // solvers.py:86-88, Sr1Estimate.apply = tau x + u (u.x)
      T bx = s_tau[t] * ((const T*)P.x[t])[j];
      bx = bx + ((const T*)P.u[t])[j] * s_utx[t];  // u_t == 0 for a rejected term
      a += bx - stp * ((const T*)P.g[t])[j];
    }
    accbuf[j] = a;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c < count) {
        const T uc = c < r ? ((const T*)P.u[s_map[c]])[j] : (T)0;
        Uc[(long long)c * n + j] = uc;
        acc[c] += (double)uc * (double)a;
      }
    }
  }
  if (last_block_reduce<NT, 8>(acc, count, ws, red, scr) && threadIdx.x == 0) {
    const double* L = meta + M_CHOL;
    double b[8];
    for (int i = 0; i < count; ++i) b[i] = red[i];
    for (int i = 0; i < count; ++i) {  // forward / back substitution with the stored factor
      double s = b[i];
      for (int k = 0; k < i; ++k) s -= L[i * count + k] * b[k];
      b[i] = s / L[i * count + i];
    }
    for (int i = count - 1; i >= 0; --i) {
      double s = b[i];
      for (int k = i + 1; k < count; ++k) s -= L[k * count + i] * b[k];
      b[i] = s / L[i * count + i];
    }
    for (int i = 0; i < count; ++i) meta[M_COEF + i] = b[i];
  }
}

template <typename T>
__global__ void __launch_bounds__(NT) agg_out(long long n, int count, const double* meta, const T* __restrict__ Uc,
                                              const T* __restrict__ accbuf, T* __restrict__ v) {
  __shared__ T s_coef[8];
  __shared__ T s_tau;
  if (threadIdx.x < 8) s_coef[threadIdx.x] = threadIdx.x < count ? (T)meta[M_COEF + threadIdx.x] : (T)0;
  if (threadIdx.x == 0) s_tau = (T)meta[M_TAU];
  __syncthreads();
  const T t = s_tau;
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT) {
    T uc = 0;
    for (int c = 0; c < count; ++c) uc += Uc[(long long)c * n + j] * s_coef[c];
    v[j] = accbuf[j] / t - uc / (t * t);  // wpm.py:99-105 (sign +)
  }
}

int grid_for(bq_ctx* ctx, long long n) {
  long long want = (n + 4LL * NT - 1) / (4LL * NT);
  return (int)std::max<long long>(1, std::min<long long>(want, std::min(1184, ctx->num_sms * 4)));
}

}  // namespace
}  // namespace bq

using namespace bq;

extern "C" int bq_bqnpm_metric_vk(bq_ctx* ctx, int32_t dtype, int64_t n, int32_t count, const void* const* xs,
                                  const void* const* gs, const void* const* us, const double* const* ests,
                                  double step, void* Uc_out, double* meta, void* acc_scratch, void* v_out,
                                  void* stream) {
  BQ_CHECK(ctx && xs && gs && us && ests && Uc_out && meta && acc_scratch && v_out && n > 0, BQ_EINVAL,
           "bq_bqnpm_metric_vk: bad arguments");
  BQ_CHECK(count >= 1 && count <= 8, BQ_EINVAL, "bq_bqnpm_metric_vk: 1..8 slots");
  SlotPtrs P{};
  for (int t = 0; t < count; ++t) {
    BQ_CHECK(xs[t] && gs[t] && us[t] && ests[t], BQ_EINVAL, "bq_bqnpm_metric_vk: slot %d incomplete", t);
    P.x[t] = xs[t];
    P.g[t] = gs[t];
    P.u[t] = us[t];
    P.est[t] = ests[t];
  }
  cudaStream_t st = (cudaStream_t)stream;
  BQ_STREAM_WS(sw, ctx, st);
  RedWs ws = red_ws(sw);
  const int G = grid_for(ctx, n);
  if (dtype == BQ_F32) {
    agg_pass1<float><<<G, NT, 0, st>>>(n, count, P, meta, ws);
    agg_pass2<float><<<G, NT, 0, st>>>(n, count, P, step, meta, (float*)Uc_out, (float*)acc_scratch, ws);
    agg_out<float><<<G, NT, 0, st>>>(n, count, meta, (const float*)Uc_out, (const float*)acc_scratch, (float*)v_out);
  } else {
    agg_pass1<double><<<G, NT, 0, st>>>(n, count, P, meta, ws);
    agg_pass2<double><<<G, NT, 0, st>>>(n, count, P, step, meta, (double*)Uc_out, (double*)acc_scratch, ws);
    agg_out<double><<<G, NT, 0, st>>>(n, count, meta, (const double*)Uc_out, (const double*)acc_scratch,
                                      (double*)v_out);
  }
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}
