// views_ls.cu — first-Born and Lippmann-Schwinger view batches on the device.
//
// No reference implementation exists: the discretisation is the
// builder's specification in oracle/physics.py.
// Every operator here mirrors one function of that oracle:
//   bq_green_init        green_kernel_hat       K on the 2n-padded grid, FFT'd once
//   bq_ls_incident       incident               plane waves generated in-kernel
//   bq_ls_conv           Green.dom / dom_adj / det / det_adj (+ the LS operator A, A^H)
//   bq_cdot / bq_bicg_*  bicgstab               batched BiCGSTAB vector algebra
//
// B200 design: views are batched (B views per call); the 3-D transforms of the
// (2n)^3 padded grid are batched cuFFT C2C/Z2Z plans (plan cache in the
// context); padding + contrast multiply, the spectral Green multiply and the
// crop + axpy are each ONE fused pointwise kernel over the batch; per-view
// dot products are deterministic two-stage reductions (no float atomics).
#include <cufft.h>

#include <map>
#include <tuple>

#include "common.cuh"

namespace bq {

struct FftCache {
  std::map<std::tuple<int, int, int>, cufftHandle> plans;  // (m, batch, dtype)
};

void fft_cache_destroy(void* cache) {
  auto* c = (FftCache*)cache;
  if (!c) return;
  for (auto& kv : c->plans) cufftDestroy(kv.second);
  delete c;
}

namespace {

template <typename T>
struct Cx;
template <>
struct Cx<float> {
  using V = float2;
};
template <>
struct Cx<double> {
  using V = double2;
};

template <typename V>
__device__ __forceinline__ V cmul(V a, V b) {
  V r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}
template <typename V>
__device__ __forceinline__ V cconjmul(V a, V b) {  // conj(a) * b
  V r;
  r.x = a.x * b.x + a.y * b.y;
  r.y = a.x * b.y - a.y * b.x;
  return r;
}

int fft_plan(bq_ctx* ctx, int m, int batch, int dtype, cufftHandle* out) {
  if (!ctx->fft_cache) ctx->fft_cache = new FftCache();
  auto* c = (FftCache*)ctx->fft_cache;
  auto key = std::make_tuple(m, batch, dtype);
  auto it = c->plans.find(key);
  if (it != c->plans.end()) {
    *out = it->second;
    return BQ_OK;
  }
  cufftHandle h;
  int dims[3] = {m, m, m};
  cufftResult r = cufftPlanMany(&h, 3, dims, nullptr, 1, m * m * m, nullptr, 1, m * m * m,
                                dtype == BQ_F32 ? CUFFT_C2C : CUFFT_Z2Z, batch);
  if (r != CUFFT_SUCCESS) {
    set_error("cufftPlanMany(%d^3 x %d) failed: %d", m, batch, (int)r);
    return BQ_ECUDA;
  }
  c->plans[key] = h;
  *out = h;
  return BQ_OK;
}

int fft_exec(bq_ctx* ctx, int m, int batch, int dtype, void* buf, int direction, cudaStream_t st) {
  cufftHandle h;
  int rc = fft_plan(ctx, m, batch, dtype, &h);
  if (rc) return rc;
  if (cufftSetStream(h, st) != CUFFT_SUCCESS) {
    set_error("cufftSetStream failed");
    return BQ_ECUDA;
  }
  cufftResult r = dtype == BQ_F32 ? cufftExecC2C(h, (cufftComplex*)buf, (cufftComplex*)buf, direction)
                                  : cufftExecZ2Z(h, (cufftDoubleComplex*)buf, (cufftDoubleComplex*)buf, direction);
  if (r != CUFFT_SUCCESS) {
    set_error("cufftExec failed: %d", (int)r);
    return BQ_ECUDA;
  }
  return BQ_OK;
}

// K(d) = h^3 exp(i kb |d|) / (4 pi |d|), ball-averaged self term (oracle/physics.py)
template <typename T>
__global__ void green_fill_kernel(int n, double h, double kb, typename Cx<T>::V* K) {
  const int m = 2 * n;
  const long long M = (long long)m * m * m;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < M; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % m), y = (int)((i / m) % m), z = (int)(i / ((long long)m * m));
    const double ox = (x <= n ? x : x - m) * h, oy = (y <= n ? y : y - m) * h, oz = (z <= n ? z : z - m) * h;
    const double r = sqrt(ox * ox + oy * oy + oz * oz);
    double re, im;
    if (i == 0) {
      const double a = h * cbrt(3.0 / (4.0 * M_PI));
      double s, c;
      sincos(kb * a, &s, &c);
      // (exp(i kb a)(1 - i kb a) - 1) / kb^2
      re = (c + kb * a * s - 1.0) / (kb * kb);
      im = (s - kb * a * c) / (kb * kb);
    } else {
      double s, c;
      sincos(kb * r, &s, &c);
      const double g = h * h * h / (4.0 * M_PI * r);
      re = g * c;
      im = g * s;
    }
    K[i].x = (T)re;
    K[i].y = (T)im;
  }
}

// incident plane waves u_in[b](r) = exp(i k_b . r)
template <typename T>
__global__ void incident_kernel(int n, double h, int B, const double* kvec /* 3B */, typename Cx<T>::V* out) {
  const long long N = (long long)n * n * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N * B; t += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(t / N);
    const long long j = t - (long long)b * N;
    const int x = (int)(j % n), y = (int)((j / n) % n), z = (int)(j / ((long long)n * n));
    const double ph = kvec[3 * b] * (x + 0.5) * h + kvec[3 * b + 1] * (y + 0.5) * h + kvec[3 * b + 2] * (z + 0.5) * h;
    double s, c;
    sincos(ph, &s, &c);
    out[t].x = (T)c;
    out[t].y = (T)s;
  }
}

// pad: P[b] = embed(f . v[b]) (f may be NULL -> v) on the (2n)^3 grid; zero elsewhere.
// det mode: P[b] = r[b] placed on plane z = n (rows y < n, cols x < n).
template <typename T>
__global__ void pad_kernel(int n, int B, const T* __restrict__ f, const typename Cx<T>::V* __restrict__ v,
                           int det_mode, typename Cx<T>::V* __restrict__ P) {
  using V = typename Cx<T>::V;
  const int m = 2 * n;
  const long long M = (long long)m * m * m, N = (long long)n * n * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < M * B; t += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(t / M);
    const long long i = t - (long long)b * M;
    const int x = (int)(i % m), y = (int)((i / m) % m), z = (int)(i / ((long long)m * m));
    V val;
    val.x = 0;
    val.y = 0;
    if (!det_mode) {
      if (x < n && y < n && z < n) {
        const long long j = ((long long)z * n + y) * n + x;
        val = v[(long long)b * N + j];
        if (f) {
          const T fj = f[j];
          val.x *= fj;
          val.y *= fj;
        }
      }
    } else if (z == n && x < n && y < n) {
      val = v[(long long)b * n * n + (long long)y * n + x];
    }
    P[t] = val;
  }
}

// P[b] *= Khat (or conj(Khat))
template <typename T>
__global__ void spec_mul_kernel(long long M, int B, const typename Cx<T>::V* __restrict__ Kh, int conj,
                                typename Cx<T>::V* __restrict__ P) {
  using V = typename Cx<T>::V;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < M * B; t += (long long)gridDim.x * blockDim.x) {
    const long long i = t % M;
    V k = Kh[i];
    if (conj) k.y = -k.y;
    P[t] = cmul(P[t], k);
  }
}

// crop the domain: out[b] = alpha v[b] + beta * s * g(P[b]|dom), g = id or conj(f) .
template <typename T>
__global__ void crop_kernel(int n, int B, const typename Cx<T>::V* __restrict__ P, double scale,
                            const typename Cx<T>::V* __restrict__ v, double alpha, double beta,
                            const T* __restrict__ fconj, const typename Cx<T>::V* __restrict__ addend,
                            typename Cx<T>::V* __restrict__ out) {
  using V = typename Cx<T>::V;
  const int m = 2 * n;
  const long long M = (long long)m * m * m, N = (long long)n * n * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N * B; t += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(t / N);
    const long long j = t - (long long)b * N;
    const int x = (int)(j % n), y = (int)((j / n) % n), z = (int)(j / ((long long)n * n));
    V p = P[(long long)b * M + ((long long)z * m + y) * m + x];
    p.x *= (T)scale;
    p.y *= (T)scale;
    if (fconj) {  // multiply by conj(f): f is real
      const T fj = fconj[j];
      p.x *= fj;
      p.y *= fj;
    }
    V r;
    r.x = (T)beta * p.x;
    r.y = (T)beta * p.y;
    if (v && alpha != 0.0) {
      const V vv = v[t];
      r.x += (T)alpha * vv.x;
      r.y += (T)alpha * vv.y;
    }
    if (addend) {
      r.x += addend[t].x;
      r.y += addend[t].y;
    }
    out[t] = r;
  }
}

// out[b] = f . in[b]  (f real, e.g. conj(f) . w for the adjoint right-hand side)
template <typename T>
__global__ void cscale_kernel(long long N, int B, const T* __restrict__ f, const typename Cx<T>::V* __restrict__ in,
                              typename Cx<T>::V* __restrict__ out) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N * B; t += (long long)gridDim.x * blockDim.x) {
    const T fj = f[t % N];
    auto v = in[t];
    v.x *= fj;
    v.y *= fj;
    out[t] = v;
  }
}

// detector plane z = n of P[b] -> out[b] (n^2), scaled
template <typename T>
__global__ void det_kernel(int n, int B, const typename Cx<T>::V* __restrict__ P, double scale,
                           typename Cx<T>::V* __restrict__ out) {
  const int m = 2 * n;
  const long long M = (long long)m * m * m, n2 = (long long)n * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n2 * B; t += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(t / n2);
    const long long j = t - (long long)b * n2;
    const int x = (int)(j % n), y = (int)(j / n);
    typename Cx<T>::V p = P[(long long)b * M + ((long long)n * m + y) * m + x];
    p.x *= (T)scale;
    p.y *= (T)scale;
    out[t] = p;
  }
}

// per-view dots <a_b, c_b> = sum conj(a) c   (stage 1: per-block partials)
template <typename T>
__global__ void cdot_kernel(long long N, int B, const typename Cx<T>::V* __restrict__ a,
                            const typename Cx<T>::V* __restrict__ c, double* __restrict__ partials) {
  const int b = blockIdx.y;
  double re = 0.0, im = 0.0;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    const auto av = a[(long long)b * N + j];
    const auto cv = c[(long long)b * N + j];
    re += (double)av.x * cv.x + (double)av.y * cv.y;
    im += (double)av.x * cv.y - (double)av.y * cv.x;
  }
  __shared__ double sr[32], si[32];
  for (int o = 16; o > 0; o >>= 1) {
    re += __shfl_down_sync(0xffffffffu, re, o);
    im += __shfl_down_sync(0xffffffffu, im, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sr[warp] = re, si[warp] = im;
  __syncthreads();
  if (threadIdx.x == 0) {
    double R = 0, I = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) R += sr[w], I += si[w];
    partials[((long long)b * gridDim.x + blockIdx.x) * 2] = R;
    partials[((long long)b * gridDim.x + blockIdx.x) * 2 + 1] = I;
  }
}
__global__ void cdot_finish(int nblk, int B, const double* partials, double* out /* 2B */) {
  const int b = threadIdx.x;
  if (b < B) {
    double R = 0, I = 0;
    for (int k = 0; k < nblk; ++k) R += partials[((long long)b * nblk + k) * 2], I += partials[((long long)b * nblk + k) * 2 + 1];
    out[2 * b] = R;
    out[2 * b + 1] = I;
  }
}

// out[b] = a[b] + coef[b] * c[b]   (coef complex per view, optionally conjugated/negated)
template <typename T>
__global__ void caxpy_kernel(long long N, int B, const typename Cx<T>::V* __restrict__ a, const double* __restrict__ coef,
                             int cstride, double sgn, const typename Cx<T>::V* __restrict__ c,
                             typename Cx<T>::V* __restrict__ out, const int* __restrict__ active) {
  using V = typename Cx<T>::V;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N * B; t += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(t / N);
    if (active && !active[b]) continue;
    V k;
    k.x = (T)(sgn * coef[cstride * b]);
    k.y = (T)(sgn * coef[cstride * b + 1]);
    const V r = cmul(k, c[t]);
    V o;
    o.x = a[t].x + r.x;
    o.y = a[t].y + r.y;
    out[t] = o;
  }
}

// BiCGSTAB scalar recurrences per view (oracle/physics.py bicgstab)
//  stage 0: rho_new = d0; beta = (rho_new/rho)(alpha/omega); -> coef[beta, -omega]
//  stage 1: alpha = rho_new / d0 (d0 = <rh, v>)
//  stage 2: omega = d0 / d1 (d0 = <t, s>, d1 = <t, t>); rho = rho_new
// state per view (doubles): [rho(2), alpha(2), omega(2), rho_new(2)]
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double den = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
}
__device__ __forceinline__ double2 cmuld(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__global__ void bicg_scalar_kernel(int B, int stage, const double* d0, const double* d1, double* state, double* coef) {
  const int b = threadIdx.x;
  if (b >= B) return;
  double* s = state + 8 * b;
  double2 rho = make_double2(s[0], s[1]), alpha = make_double2(s[2], s[3]), omega = make_double2(s[4], s[5]);
  if (stage == 0) {
    const double2 rn = make_double2(d0[2 * b], d0[2 * b + 1]);
    const double2 beta = cmuld(cdiv(rn, rho), cdiv(alpha, omega));
    s[6] = rn.x, s[7] = rn.y;
    coef[4 * b] = beta.x, coef[4 * b + 1] = beta.y;
    coef[4 * b + 2] = omega.x, coef[4 * b + 3] = omega.y;
  } else if (stage == 1) {
    const double2 rn = make_double2(s[6], s[7]);
    alpha = cdiv(rn, make_double2(d0[2 * b], d0[2 * b + 1]));
    s[2] = alpha.x, s[3] = alpha.y;
  } else {
    omega = cdiv(make_double2(d0[2 * b], d0[2 * b + 1]), make_double2(d1[2 * b], d1[2 * b + 1]));
    s[4] = omega.x, s[5] = omega.y;
    s[0] = s[6], s[1] = s[7];
  }
}

// p = r + beta (p - omega v)      (per view, active only)
template <typename T>
__global__ void bicg_p_kernel(long long N, int B, const typename Cx<T>::V* __restrict__ r,
                              const typename Cx<T>::V* __restrict__ v, const double* __restrict__ coef,
                              typename Cx<T>::V* __restrict__ p, const int* __restrict__ active) {
  using V = typename Cx<T>::V;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N * B; t += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(t / N);
    if (!active[b]) continue;
    V beta, omega;
    beta.x = (T)coef[4 * b], beta.y = (T)coef[4 * b + 1];
    omega.x = (T)coef[4 * b + 2], omega.y = (T)coef[4 * b + 3];
    const V ov = cmul(omega, v[t]);
    V q;
    q.x = p[t].x - ov.x;
    q.y = p[t].y - ov.y;
    const V bq = cmul(beta, q);
    V o;
    o.x = r[t].x + bq.x;
    o.y = r[t].y + bq.y;
    p[t] = o;
  }
}

// x += alpha p + omega s ; r = s - omega t   (stage "full"); or x += alpha p (early exit)
template <typename T>
__global__ void bicg_x_kernel(long long N, int B, const double* __restrict__ state, const typename Cx<T>::V* __restrict__ p,
                              const typename Cx<T>::V* __restrict__ s, const typename Cx<T>::V* __restrict__ tt,
                              typename Cx<T>::V* __restrict__ x, typename Cx<T>::V* __restrict__ r,
                              const int* __restrict__ mode /* per view: 0 skip, 1 early, 2 full */) {
  using V = typename Cx<T>::V;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N * B; t += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(t / N);
    const int md = mode[b];
    if (md == 0) continue;
    V alpha, omega;
    alpha.x = (T)state[8 * b + 2], alpha.y = (T)state[8 * b + 3];
    omega.x = (T)state[8 * b + 4], omega.y = (T)state[8 * b + 5];
    const V ap = cmul(alpha, p[t]);
    V xo = x[t];
    xo.x += ap.x;
    xo.y += ap.y;
    if (md == 2) {
      const V os = cmul(omega, s[t]);
      xo.x += os.x;
      xo.y += os.y;
      const V ot = cmul(omega, tt[t]);
      V rr;
      rr.x = s[t].x - ot.x;
      rr.y = s[t].y - ot.y;
      r[t] = rr;
    }
    x[t] = xo;
  }
}

// grad[j] += Re(conj(fp_j u_b[j]) * w_b[j]) summed over the batch in view order
template <typename T>
__global__ void grad_accum_kernel(long long N, int B, const T* __restrict__ fp, const typename Cx<T>::V* __restrict__ u,
                                  const typename Cx<T>::V* __restrict__ w, double scale, T* __restrict__ grad,
                                  int accumulate) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    T acc = accumulate ? grad[j] : (T)0;
    const T f = fp[j];
    for (int b = 0; b < B; ++b) {
      const auto uu = u[(long long)b * N + j];
      const auto ww = w[(long long)b * N + j];
      acc += (T)scale * f * (uu.x * ww.x + uu.y * ww.y);  // Re(conj(f u) w), f real
    }
    grad[j] = acc;
  }
}

// potential f and f' from x (oracle ScatterModel.pot): born 2k0^2 nb x ; ls k0^2((nb+x)^2 - nb^2)
template <typename T>
__global__ void potential_kernel(long long N, const T* __restrict__ x, double k0, double nb, int born, T* __restrict__ f,
                                 T* __restrict__ fp) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    const double xv = x[j];
    if (born) {
      f[j] = (T)(2.0 * k0 * k0 * nb * xv);
      fp[j] = (T)(2.0 * k0 * k0 * nb);
    } else {
      f[j] = (T)(k0 * k0 * ((nb + xv) * (nb + xv) - nb * nb));
      fp[j] = (T)(2.0 * k0 * k0 * (nb + xv));
    }
  }
}

int grid_for(bq_ctx* ctx, long long n) {
  return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, (long long)ctx->num_sms * 8));
}

}  // namespace
}  // namespace bq

using namespace bq;

#define DT_SWITCH(dtype, BODY)         \
  if ((dtype) == BQ_F32) {             \
    using T = float;                   \
    BODY;                              \
  } else {                             \
    using T = double;                  \
    BODY;                              \
  }

extern "C" int bq_green_init(bq_ctx* ctx, int32_t dtype, int32_t n, double h, double kb, void* khat, void* stream) {
  BQ_CHECK(ctx && khat && n >= 2 && n <= 512, BQ_EINVAL, "bq_green_init: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const long long M = 8LL * n * n * n;
  DT_SWITCH(dtype, (green_fill_kernel<T><<<grid_for(ctx, M), 256, 0, st>>>(n, h, kb, (typename Cx<T>::V*)khat)));
  BQ_CUDA(cudaGetLastError());
  return fft_exec(ctx, 2 * n, 1, dtype, khat, CUFFT_FORWARD, st);
}

extern "C" int bq_ls_incident(bq_ctx* ctx, int32_t dtype, int32_t n, double h, int32_t B, const double* kvec_dev,
                              void* out, void* stream) {
  BQ_CHECK(ctx && kvec_dev && out && B >= 1, BQ_EINVAL, "bq_ls_incident: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const long long N = (long long)n * n * n;
  DT_SWITCH(dtype, (incident_kernel<T><<<grid_for(ctx, N * B), 256, 0, st>>>(n, h, B, kvec_dev, (typename Cx<T>::V*)out)));
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

namespace bq {
namespace {
template <typename T>
int ls_conv_impl(bq_ctx* ctx, int dtype, int n, int B, int op, const void* khat, const void* f, const void* v,
                 double alpha, double beta, const void* addend, void* pad_buf, void* out, cudaStream_t st) {
  using V = typename Cx<T>::V;
  const int m = 2 * n;
  const long long M = (long long)m * m * m, N = (long long)n * n * n;
  const double scale = 1.0 / (double)M;
  const bool adj = (op == 1 || op == 3);
  int rc = ls_conv_pruned(ctx, dtype, n, B, op, khat, f, v, alpha, beta, addend, pad_buf, out, st);
  if (rc != 1) return rc;  // handled by the pruned line passes (ls_fft.cu)
  pad_kernel<T><<<grid_for(ctx, M * B), 256, 0, st>>>(n, B, (op == 0 || op == 2) ? (const T*)f : nullptr,
                                                      (const V*)v, op == 3, (V*)pad_buf);
  BQ_CUDA(cudaGetLastError());
  if ((rc = fft_exec(ctx, m, B, dtype, pad_buf, CUFFT_FORWARD, st))) return rc;
  spec_mul_kernel<T><<<grid_for(ctx, M * B), 256, 0, st>>>(M, B, (const V*)khat, adj ? 1 : 0, (V*)pad_buf);
  if ((rc = fft_exec(ctx, m, B, dtype, pad_buf, CUFFT_INVERSE, st))) return rc;
  if (op == 2) {
    det_kernel<T><<<grid_for(ctx, (long long)n * n * B), 256, 0, st>>>(n, B, (const V*)pad_buf, scale, (V*)out);
  } else {
    crop_kernel<T><<<grid_for(ctx, N * B), 256, 0, st>>>(n, B, (const V*)pad_buf, scale,
                                                         op == 3 ? nullptr : (const V*)v, op == 3 ? 0.0 : alpha,
                                                         op == 3 ? 1.0 : beta, op == 1 ? (const T*)f : nullptr,
                                                         (const V*)addend, (V*)out);
  }
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}
}  // namespace
}  // namespace bq

// Green operator on a batch, all through the padded (2n)^3 transform:
//   op 0: out = alpha v + beta G_dom(f . v)            (f may be NULL; A v: alpha 1 beta -1)
//   op 1: out = alpha v + beta conj(f) . G_dom^H v      (A^H v: alpha 1 beta -1, fconj = f)
//   op 2: out = G_det(f . v)           (n^2 per view)
//   op 3: out = G^H P_det^T r          (r: n^2 per view -> N per view)
extern "C" int bq_ls_conv(bq_ctx* ctx, int32_t dtype, int32_t n, int32_t B, int32_t op, const void* khat,
                          const void* f, const void* v, double alpha, double beta, const void* addend,
                          void* pad_buf, void* out, void* stream) {
  BQ_CHECK(ctx && khat && v && pad_buf && out && B >= 1 && op >= 0 && op <= 3, BQ_EINVAL, "bq_ls_conv: bad arguments");
  BQ_CHECK(op != 2 || addend == nullptr, BQ_EINVAL, "bq_ls_conv: no addend for the detector op");
  cudaStream_t st = (cudaStream_t)stream;
  return dtype == BQ_F32 ? ls_conv_impl<float>(ctx, dtype, n, B, op, khat, f, v, alpha, beta, addend, pad_buf, out, st)
                         : ls_conv_impl<double>(ctx, dtype, n, B, op, khat, f, v, alpha, beta, addend, pad_buf, out,
                                                st);
}

extern "C" int bq_cscale_real(bq_ctx* ctx, int32_t dtype, int64_t N, int32_t B, const void* f, const void* in,
                              void* out, void* stream) {
  BQ_CHECK(ctx && f && in && out && B >= 1, BQ_EINVAL, "bq_cscale_real: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  DT_SWITCH(dtype, (cscale_kernel<T><<<grid_for(ctx, N * B), 256, 0, st>>>(N, B, (const T*)f,
                                                                            (const typename Cx<T>::V*)in,
                                                                            (typename Cx<T>::V*)out)));
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_cdot(bq_ctx* ctx, int32_t dtype, int64_t N, int32_t B, const void* a, const void* c, double* out,
                       void* stream) {
  BQ_CHECK(ctx && a && c && out && B >= 1 && B <= 256, BQ_EINVAL, "bq_cdot: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const int nblk = (int)std::min<long long>(64, std::max<long long>(1, (N + 255) / 256));
  double* partials = ctx->ws.partials;
  BQ_CHECK((long long)nblk * B * 2 <= (long long)kMaxBlocks * kMaxVals, BQ_EINVAL, "bq_cdot: batch too large");
  DT_SWITCH(dtype, (cdot_kernel<T><<<dim3(nblk, B), 256, 0, st>>>(N, B, (const typename Cx<T>::V*)a,
                                                                   (const typename Cx<T>::V*)c, partials)));
  cdot_finish<<<1, 256, 0, st>>>(nblk, B, partials, out);
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_caxpy(bq_ctx* ctx, int32_t dtype, int64_t N, int32_t B, const void* a, const double* coef,
                        int32_t coef_stride, double sgn, const void* c, void* out, const int32_t* active,
                        void* stream) {
  BQ_CHECK(ctx && a && coef && c && out, BQ_EINVAL, "bq_caxpy: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  DT_SWITCH(dtype, (caxpy_kernel<T><<<grid_for(ctx, N * B), 256, 0, st>>>(N, B, (const typename Cx<T>::V*)a, coef,
                                                                           coef_stride, sgn,
                                                                           (const typename Cx<T>::V*)c,
                                                                           (typename Cx<T>::V*)out, active)));
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_bicg_scalars(bq_ctx* ctx, int32_t B, int32_t stage, const double* d0, const double* d1,
                               double* state, double* coef, void* stream) {
  BQ_CHECK(ctx && state && B >= 1 && B <= 256 && stage >= 0 && stage <= 2, BQ_EINVAL, "bq_bicg_scalars: bad arguments");
  bicg_scalar_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(B, stage, d0, d1, state, coef);
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_bicg_p(bq_ctx* ctx, int32_t dtype, int64_t N, int32_t B, const void* r, const void* v,
                         const double* coef, void* p, const int32_t* active, void* stream) {
  BQ_CHECK(ctx && r && v && coef && p && active, BQ_EINVAL, "bq_bicg_p: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  DT_SWITCH(dtype, (bicg_p_kernel<T><<<grid_for(ctx, N * B), 256, 0, st>>>(N, B, (const typename Cx<T>::V*)r,
                                                                            (const typename Cx<T>::V*)v, coef,
                                                                            (typename Cx<T>::V*)p, active)));
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_bicg_x(bq_ctx* ctx, int32_t dtype, int64_t N, int32_t B, const double* state, const void* p,
                         const void* s, const void* t, void* x, void* r, const int32_t* mode, void* stream) {
  BQ_CHECK(ctx && state && p && x && mode, BQ_EINVAL, "bq_bicg_x: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  DT_SWITCH(dtype, (bicg_x_kernel<T><<<grid_for(ctx, N * B), 256, 0, st>>>(
                        N, B, state, (const typename Cx<T>::V*)p, (const typename Cx<T>::V*)s,
                        (const typename Cx<T>::V*)t, (typename Cx<T>::V*)x, (typename Cx<T>::V*)r, mode)));
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_ls_grad_accum(bq_ctx* ctx, int32_t dtype, int64_t N, int32_t B, const void* fp, const void* u,
                                const void* w, double scale, void* grad, int32_t accumulate, void* stream) {
  BQ_CHECK(ctx && fp && u && w && grad, BQ_EINVAL, "bq_ls_grad_accum: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  DT_SWITCH(dtype, (grad_accum_kernel<T><<<grid_for(ctx, N), 256, 0, st>>>(N, B, (const T*)fp,
                                                                            (const typename Cx<T>::V*)u,
                                                                            (const typename Cx<T>::V*)w, scale, (T*)grad,
                                                                            accumulate)));
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_ls_potential(bq_ctx* ctx, int32_t dtype, int64_t N, const void* x, double k0, double nb,
                               int32_t born, void* f, void* fp, void* stream) {
  BQ_CHECK(ctx && x && f && fp, BQ_EINVAL, "bq_ls_potential: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  DT_SWITCH(dtype, (potential_kernel<T><<<grid_for(ctx, N), 256, 0, st>>>(N, (const T*)x, k0, nb, born, (T*)f, (T*)fp)));
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}
