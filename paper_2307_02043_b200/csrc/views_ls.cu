// views_ls.cu — first-Born and Lippmann-Schwinger view batches on the device.
//
// No reference implementation exists: the discretisation is the
// builder's specification in oracle/physics.py.
// Every operator here mirrors one function of that oracle:
//   bq_green_init        green_kernel_hat       K on the 2n-padded grid, FFT'd once
//   bq_ls_incident       incident               plane waves generated in-kernel
//   bq_ls_conv           Green.dom / dom_adj / det / det_adj (+ the LS operator A, A^H)
//   bq_ls_bicgstab       bicgstab               device-resident batched BiCGSTAB
//
// B200 design: views are batched (B views per call).  For padded sizes 16..512
// the convolution is ls_fft.cu's five pruned line passes (the padded grid is
// never formed); other sizes use batched cuFFT C2C/Z2Z plans (plan cache in the
// context) between fused pad / spectral-multiply / crop kernels.  The
// BiCGSTAB below keeps every scalar and decision on the device; its per-view
// dot products are fixed-order block partials (no float atomics).
#include <cufft.h>

#include <map>
#include <tuple>
#include <type_traits>

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

// complex double helpers of the BiCGSTAB recurrences
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double den = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
}
__device__ __forceinline__ double2 cmuld(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
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

// ===========================================================================
// Device-resident batched BiCGSTAB (oracle/physics.py bicgstab, per view):
// all scalar recurrences and stopping decisions are made on the device; the
// dots ride in the producing kernels (the Green convolution's epilogue, the
// s and x/r updates) as fixed-order per-block partials; converged views are
// skipped by every kernel (the convolution passes included).  The host only
// learns "how many views are still active" one iteration late through a
// pinned flag, so the GPU never idles on a host round trip.
// ===========================================================================
namespace bq {
namespace {

// state per view (doubles): rho(2) alpha(2) omega(2) rho_new(2) nb beta(2) -> 16
constexpr int kBS = 16;
enum { BG_INIT = 0, BG_ALPHA = 1, BG_S = 2, BG_OMEGA = 3, BG_END = 4 };

__device__ __forceinline__ void block_part3(double a, double b, double c, double* out) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
    c += __shfl_down_sync(0xffffffffu, c, o);
  }
  __shared__ double red[3][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[0][w] = a, red[1][w] = b, red[2][w] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s0 += red[0][q], s1 += red[1][q], s2 += red[2][q];
    out[0] = s0, out[1] = s1, out[2] = s2;
  }
}

template <typename T>
__global__ void bg_init_kernel(long long N, const typename Cx<T>::V* __restrict__ rhs, typename Cx<T>::V* x,
                               typename Cx<T>::V* r, typename Cx<T>::V* rh, typename Cx<T>::V* p,
                               typename Cx<T>::V* v, double* part) {
  using V = typename Cx<T>::V;
  const int b = blockIdx.y;
  const long long o = (long long)b * N;
  V z;
  z.x = 0, z.y = 0;
  double nn = 0.0;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    const V bb = rhs[o + j];
    x[o + j] = z, r[o + j] = bb, rh[o + j] = bb, p[o + j] = z, v[o + j] = z;
    nn += (double)bb.x * bb.x + (double)bb.y * bb.y;
  }
  block_part3(nn, 0.0, nn, part + ((long long)b * gridDim.x + blockIdx.x) * 3);
}

// p = r + beta (p - omega v)
template <typename T>
__global__ void bg_p_kernel(long long N, const typename Cx<T>::V* __restrict__ r, const typename Cx<T>::V* __restrict__ v,
                            const double* __restrict__ state, typename Cx<T>::V* p, const int* __restrict__ active) {
  using V = typename Cx<T>::V;
  const int b = blockIdx.y;
  if (!active[b]) return;
  const double* s = state + kBS * b;
  V beta, omega;
  beta.x = (T)s[9], beta.y = (T)s[10];
  omega.x = (T)s[4], omega.y = (T)s[5];
  const long long o = (long long)b * N;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    const V ov = cmul(omega, v[o + j]);
    V q;
    q.x = p[o + j].x - ov.x;
    q.y = p[o + j].y - ov.y;
    const V bq = cmul(beta, q);
    V out;
    out.x = r[o + j].x + bq.x;
    out.y = r[o + j].y + bq.y;
    p[o + j] = out;
  }
}

// s = r - alpha v, partial ||s||^2
template <typename T>
__global__ void bg_s_kernel(long long N, const typename Cx<T>::V* __restrict__ r, const typename Cx<T>::V* __restrict__ v,
                            const double* __restrict__ state, typename Cx<T>::V* __restrict__ s,
                            const int* __restrict__ active, double* part) {
  using V = typename Cx<T>::V;
  const int b = blockIdx.y;
  if (!active[b]) return;
  V alpha;
  alpha.x = (T)state[kBS * b + 2], alpha.y = (T)state[kBS * b + 3];
  const long long o = (long long)b * N;
  double nn = 0.0;
  auto upd = [&](V rv, V vv) {
    const V av = cmul(alpha, vv);
    V q;
    q.x = rv.x - av.x;
    q.y = rv.y - av.y;
    nn += (double)q.x * q.x + (double)q.y * q.y;
    return q;
  };
  const long long gs = (long long)gridDim.x * blockDim.x, j0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (std::is_same<T, float>::value && (N & 1) == 0) {
    // complex64 pairs: 16-byte loads and stores (o = b N is even)
    const float4* r4 = reinterpret_cast<const float4*>(r + o);
    const float4* v4 = reinterpret_cast<const float4*>(v + o);
    float4* s4 = reinterpret_cast<float4*>(s + o);
    for (long long j = j0; j < (N >> 1); j += gs) {
      const float4 rv = __ldg(&r4[j]), vv = __ldg(&v4[j]);
      const V q0 = upd(V{(T)rv.x, (T)rv.y}, V{(T)vv.x, (T)vv.y});
      const V q1 = upd(V{(T)rv.z, (T)rv.w}, V{(T)vv.z, (T)vv.w});
      s4[j] = make_float4((float)q0.x, (float)q0.y, (float)q1.x, (float)q1.y);
    }
  } else {
    for (long long j = j0; j < N; j += gs) s[o + j] = upd(r[o + j], v[o + j]);
  }
  block_part3(nn, 0.0, nn, part + ((long long)b * gridDim.x + blockIdx.x) * 3);
}

// mode 1: x += alpha p ; mode 2: x += alpha p + omega s, r = s - omega t, partials (<rh, r>, ||r||^2)
template <typename T>
__global__ void bg_x_kernel(long long N, const double* __restrict__ state, const typename Cx<T>::V* __restrict__ p,
                            const typename Cx<T>::V* __restrict__ s, const typename Cx<T>::V* __restrict__ t,
                            const typename Cx<T>::V* __restrict__ rh, typename Cx<T>::V* x, typename Cx<T>::V* r,
                            const int* __restrict__ mode, double* part) {
  using V = typename Cx<T>::V;
  const int b = blockIdx.y;
  const int md = mode[b];
  if (md == 0) return;
  const double* st = state + kBS * b;
  V alpha, omega;
  alpha.x = (T)st[2], alpha.y = (T)st[3];
  omega.x = (T)st[4], omega.y = (T)st[5];
  const long long o = (long long)b * N;
  double dre = 0.0, dim = 0.0, dnn = 0.0;
  // x += alpha p (+ omega s); r = s - omega t and <rh, r>, |r|^2 (md == 2)
  auto upd = [&](V pv, V xo, V sv, V tv, V a, V& rr) {
    const V ap = cmul(alpha, pv);
    xo.x += ap.x;
    xo.y += ap.y;
    if (md == 2) {
      const V os = cmul(omega, sv);
      xo.x += os.x;
      xo.y += os.y;
      const V ot = cmul(omega, tv);
      rr.x = sv.x - ot.x;
      rr.y = sv.y - ot.y;
      dre += (double)a.x * rr.x + (double)a.y * rr.y;
      dim += (double)a.x * rr.y - (double)a.y * rr.x;
      dnn += (double)rr.x * rr.x + (double)rr.y * rr.y;
    }
    return xo;
  };
  const long long gs = (long long)gridDim.x * blockDim.x, j0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (std::is_same<T, float>::value && (N & 1) == 0) {
    // complex64 pairs: 16-byte loads and stores (o = b N is even)
    const long long N2 = N >> 1;
    auto ld = [&](const V* a, long long j) { return __ldg(reinterpret_cast<const float4*>(a + o) + j); };
    for (long long j = j0; j < N2; j += gs) {
      const float4 pv = ld(p, j);
      const float4 xv = reinterpret_cast<const float4*>(x + o)[j];
      float4 sv = make_float4(0.f, 0.f, 0.f, 0.f), tv = sv, av = sv;
      if (md == 2) sv = ld(s, j), tv = ld(t, j), av = ld(rh, j);
      V r0, r1;
      const V x0 = upd(V{(T)pv.x, (T)pv.y}, V{(T)xv.x, (T)xv.y}, V{(T)sv.x, (T)sv.y}, V{(T)tv.x, (T)tv.y},
                       V{(T)av.x, (T)av.y}, r0);
      const V x1 = upd(V{(T)pv.z, (T)pv.w}, V{(T)xv.z, (T)xv.w}, V{(T)sv.z, (T)sv.w}, V{(T)tv.z, (T)tv.w},
                       V{(T)av.z, (T)av.w}, r1);
      if (md == 2) reinterpret_cast<float4*>(r + o)[j] = make_float4((float)r0.x, (float)r0.y, (float)r1.x, (float)r1.y);
      reinterpret_cast<float4*>(x + o)[j] = make_float4((float)x0.x, (float)x0.y, (float)x1.x, (float)x1.y);
    }
  } else {
    for (long long j = j0; j < N; j += gs) {
      V rr;
      const V xo = upd(p[o + j], x[o + j], md == 2 ? s[o + j] : V{}, md == 2 ? t[o + j] : V{},
                       md == 2 ? rh[o + j] : V{}, rr);
      if (md == 2) r[o + j] = rr;
      x[o + j] = xo;
    }
  }
  block_part3(dre, dim, dnn, part + ((long long)b * gridDim.x + blockIdx.x) * 3);
}

// scalar recurrences and decisions, one 256-thread block per view (fixed-order sums)
__global__ void bg_ctl_kernel(int stage, int nblk, const double* __restrict__ part, double* state, int* mode,
                              int* active, int* act2, int* iters, int it, double tol, int* count) {
  const int b = blockIdx.x;
  const bool need = stage == BG_INIT || (stage == BG_OMEGA ? mode[b] == 2 : active[b] != 0);
  if (!need) return;  // block-uniform
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int k = threadIdx.x; k < nblk; k += blockDim.x) {
    const double* q = part + ((long long)b * nblk + k) * 3;
    s0 += q[0], s1 += q[1], s2 += q[2];
  }
  __shared__ double tot[3];
  block_part3(s0, s1, s2, tot);
  __syncthreads();
  if (threadIdx.x != 0) return;
  s0 = tot[0], s1 = tot[1], s2 = tot[2];
  double* s = state + kBS * b;
  if (stage == BG_INIT) {
    const double nb = sqrt(s2);
    s[0] = 1.0, s[1] = 0.0, s[2] = 1.0, s[3] = 0.0, s[4] = 1.0, s[5] = 0.0;
    s[6] = s0, s[7] = 0.0;  // rho_new = <rh, r> = ||b||^2
    s[8] = nb;
    s[9] = s0, s[10] = 0.0;  // beta = (rho_new / 1) (1 / 1)
    iters[b] = 0;
    mode[b] = 0;
    act2[b] = 0;
    active[b] = (nb > 0.0 && 1.0 > tol) ? 1 : 0;  // res = ||r0|| / ||b|| = 1
    return;
  }
  if (!need) return;
  if (stage == BG_ALPHA) {
    const double2 a = cdiv(make_double2(s[6], s[7]), make_double2(s0, s1));
    s[2] = a.x, s[3] = a.y;
  } else if (stage == BG_S) {
    const bool early = sqrt(s2) <= tol * s[8];
    mode[b] = early ? 1 : 2;
    act2[b] = early ? 0 : 1;
  } else if (stage == BG_OMEGA) {
    // <t, s> = sum conj(t) s = conj(sum conj(s) t)
    const double2 om = cdiv(make_double2(s0, -s1), make_double2(s2, 0.0));
    s[4] = om.x, s[5] = om.y;
  } else {  // BG_END
    iters[b] = it;
    bool done = true;
    if (mode[b] == 2) {
      const double2 rho = make_double2(s[6], s[7]);  // rho = rho_new
      s[0] = rho.x, s[1] = rho.y;
      s[6] = s0, s[7] = s1;  // next rho_new = <rh, r>
      done = sqrt(s2) / s[8] <= tol;
      if (!done) {
        const double2 beta = cmuld(cdiv(make_double2(s0, s1), rho), cdiv(make_double2(s[2], s[3]), make_double2(s[4], s[5])));
        s[9] = beta.x, s[10] = beta.y;
      }
    }
    active[b] = done ? 0 : 1;
    mode[b] = 0;
    act2[b] = 0;
    if (!done) atomicAdd(count, 1);
  }
}

// per-view (sum conj(a) c, ||c||^2) block partials (cuFFT path of the convolution)
template <typename T>
__global__ void bg_dot_kernel(long long N, const typename Cx<T>::V* __restrict__ a, const typename Cx<T>::V* __restrict__ c,
                              double* part) {
  const int b = blockIdx.y;
  const long long o = (long long)b * N;
  double dre = 0.0, dim = 0.0, dnn = 0.0;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    const auto av = a[o + j];
    const auto cv = c[o + j];
    dre += (double)av.x * cv.x + (double)av.y * cv.y;
    dim += (double)av.x * cv.y - (double)av.y * cv.x;
    dnn += (double)cv.x * cv.x + (double)cv.y * cv.y;
  }
  block_part3(dre, dim, dnn, part + ((long long)b * gridDim.x + blockIdx.x) * 3);
}

int bg_vec_blocks(bq_ctx* ctx, long long N, int B) {
  const long long want = std::max<long long>(1, (long long)ctx->num_sms * 8 / B);
  return (int)std::max<long long>(1, std::min<long long>(want, (N + 255) / 256));
}

int bg_conv_blocks(int n) {
  // rows of the XI pass / lines per block (ls_fft.cu run<>: L = min(256 / C, m))
  const int m = 2 * n;
  int C = 0;
  switch (m) {
    case 16: case 32: C = 4; break;
    case 64: case 128: C = 8; break;
    case 256: case 512: C = 16; break;
    default: return 0;
  }
#ifndef LS_LR512
#define LS_LR512 8  // (ls_fft.cu: rows per block of the row passes at m = 512)
#endif
  const int L = m == 512 ? LS_LR512 : std::min(256 / C, m);
  return (n * n + L - 1) / L;
}

template <typename T>
int bg_conv(bq_ctx* ctx, int dtype, int n, int B, int op, const void* khat, const void* f, const void* v, void* scratch,
            void* out, const int* active, const void* da, double* part, int nbv, int* nblk, cudaStream_t st) {
  int rc = ls_conv_pruned(ctx, dtype, n, B, op, khat, f, v, 1.0, -1.0, nullptr, scratch, out, st, active, da, part,
                          nblk);
  if (rc != 1) return rc;
  if ((rc = ls_conv_impl<T>(ctx, dtype, n, B, op, khat, f, v, 1.0, -1.0, nullptr, scratch, out, st))) return rc;
  const long long N = (long long)n * n * n;
  bg_dot_kernel<T><<<dim3(nbv, B), 256, 0, st>>>(N, (const typename Cx<T>::V*)da, (const typename Cx<T>::V*)out, part);
  *nblk = nbv;
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

template <typename T>
int bicgstab_impl(bq_ctx* ctx, int dtype, int n, int B, int adjoint, const void* khat, const void* f, const void* rhs,
                  void* xout, double tol, int max_iter, void* vec_work, void* conv_scratch, void* small_work,
                  int* iters, cudaStream_t st) {
  using V = typename Cx<T>::V;
  const long long N = (long long)n * n * n;
  V* r = (V*)vec_work;
  V* rh = r + B * N;
  V* p = rh + B * N;
  V* v = p + B * N;
  V* s = v + B * N;
  V* t = s + B * N;
  V* x = (V*)xout;
  const int nbv = bg_vec_blocks(ctx, N, B);
  const int pmax = std::max(nbv, bg_conv_blocks(n));
  double* part = (double*)small_work;
  double* state = part + (size_t)B * pmax * 3;
  int* mode = (int*)(state + (size_t)B * kBS);
  int* active = mode + B;
  int* act2 = active + B;
  int* count = act2 + B;
  BQ_STREAM_WS(sw, ctx, st);
  if (!sw->host_flags) {
    BQ_CUDA(cudaHostAlloc((void**)&sw->host_flags, 4 * sizeof(int), cudaHostAllocDefault));
    BQ_CUDA(cudaEventCreateWithFlags(&sw->flag_ev[0], cudaEventDisableTiming));
    BQ_CUDA(cudaEventCreateWithFlags(&sw->flag_ev[1], cudaEventDisableTiming));
  }
  const int op = adjoint ? 1 : 0;
  const dim3 vg(nbv, B);
  bg_init_kernel<T><<<vg, 256, 0, st>>>(N, (const V*)rhs, x, r, rh, p, v, part);
  bg_ctl_kernel<<<B, 256, 0, st>>>(BG_INIT, nbv, part, state, mode, active, act2, iters, 0, tol, count);
  BQ_CUDA(cudaGetLastError());
  int rc;
  for (int it = 1; it <= max_iter; ++it) {
    int nb = 0;
    bg_p_kernel<T><<<vg, 256, 0, st>>>(N, r, v, state, p, active);
    if ((rc = bg_conv<T>(ctx, dtype, n, B, op, khat, f, p, conv_scratch, v, active, rh, part, nbv, &nb, st))) return rc;
    bg_ctl_kernel<<<B, 256, 0, st>>>(BG_ALPHA, nb, part, state, mode, active, act2, iters, it, tol, count);
    bg_s_kernel<T><<<vg, 256, 0, st>>>(N, r, v, state, s, active, part);
    bg_ctl_kernel<<<B, 256, 0, st>>>(BG_S, nbv, part, state, mode, active, act2, iters, it, tol, count);
    if ((rc = bg_conv<T>(ctx, dtype, n, B, op, khat, f, s, conv_scratch, t, act2, s, part, nbv, &nb, st))) return rc;
    bg_ctl_kernel<<<B, 256, 0, st>>>(BG_OMEGA, nb, part, state, mode, active, act2, iters, it, tol, count);
    BQ_CUDA(cudaMemsetAsync(count, 0, sizeof(int), st));
    bg_x_kernel<T><<<vg, 256, 0, st>>>(N, state, p, s, t, rh, x, r, mode, part);
    bg_ctl_kernel<<<B, 256, 0, st>>>(BG_END, nbv, part, state, mode, active, act2, iters, it, tol, count);
    BQ_CUDA(cudaGetLastError());
    BQ_CUDA(cudaMemcpyAsync(&sw->host_flags[it & 1], count, sizeof(int), cudaMemcpyDeviceToHost, st));
    BQ_CUDA(cudaEventRecord(sw->flag_ev[it & 1], st));
    if (it >= 2) {  // one iteration late: the GPU already has iteration `it` queued
      BQ_CUDA(cudaEventSynchronize(sw->flag_ev[(it - 1) & 1]));
      if (sw->host_flags[(it - 1) & 1] == 0) break;
    }
  }
  return BQ_OK;
}

}  // namespace
}  // namespace bq

extern "C" int64_t bq_ls_bicgstab_small_bytes(bq_ctx* ctx, int32_t n, int32_t B) {
  if (!ctx || n < 1 || B < 1) return -1;
  const long long N = (long long)n * n * n;
  const int pmax = std::max(bg_vec_blocks(ctx, N, B), bg_conv_blocks(n));
  return (int64_t)((size_t)B * pmax * 3 * sizeof(double) + (size_t)B * kBS * sizeof(double) + (3 * (size_t)B + 4) * sizeof(int));
}

// x_b = A^-1 b_b (adjoint = 0: A = I - G_dom diag f; 1: A^H = I - diag(f) G_dom^H) for the B views, BiCGSTAB from
// x0 = 0 to the relative residual tol; iters (device, B ints) = iterations per view (oracle/physics.py bicgstab).
extern "C" int bq_ls_bicgstab(bq_ctx* ctx, int32_t dtype, int32_t n, int32_t B, int32_t adjoint, const void* khat,
                              const void* f, const void* rhs, void* x, double tol, int32_t max_iter, void* vec_work,
                              void* conv_scratch, void* small_work, int32_t* iters, void* stream) {
  BQ_CHECK(ctx && khat && f && rhs && x && vec_work && conv_scratch && small_work && iters && B >= 1 && n >= 1 &&
               max_iter >= 0,
           BQ_EINVAL, "bq_ls_bicgstab: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  return dtype == BQ_F32 ? bicgstab_impl<float>(ctx, dtype, n, B, adjoint, khat, f, rhs, x, tol, max_iter, vec_work,
                                                 conv_scratch, small_work, (int*)iters, st)
                         : bicgstab_impl<double>(ctx, dtype, n, B, adjoint, khat, f, rhs, x, tol, max_iter, vec_work,
                                                  conv_scratch, small_work, (int*)iters, st);
}
