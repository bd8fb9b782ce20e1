// tv_stencil.cu — the standalone TV stencils of tvqn.tv_ops on the device.
//
// Replaces (paths under /root/reference/pkg/src/tvqn/):
//   tv_ops.py:107-119  apply_diff               -> bq_tv_diff(adjoint = 0)
//   tv_ops.py:122-133  apply_diff_adjoint       -> bq_tv_diff(adjoint = 1)
//   tv_ops.py:136-148  gradient_stack / dual_adjoint -> bq_tv_grad_stack
//   tv_ops.py:151-159  dual_divergence          -> bq_tv_divergence
//   tv_ops.py:170-180  project_dual             -> bq_tv_project_dual
//
// Inside the FGP solve these stencils are fused into the persistent prox
// kernels (wtv_fused_impl.cuh, wtv_prox.cu) and never launched alone; these
// entry points serve the reference's public helpers (w_of_p, dual_gradient,
// dual/primal objectives) and the z-slab sharded prox's halo-aware passes.
//
// Layout: flat Fortran order over dims (dims[0] fastest) == C-order (K3,K2,K1);
// the dual field is ndim contiguous N-vectors.  Every voxel is one thread of
// a grid-stride loop over x-rows: consecutive threads read consecutive x, so
// each stencil pass is one coalesced read of its inputs and one write; the
// rows' neighbours along y/z come from the same L2 lines the neighbouring
// rows read (HBM traffic = inputs + outputs).
#include <algorithm>

#include "common.cuh"

namespace bq {
namespace {

constexpr int NT = 256;

struct Geo {
  long long N;
  int K[3];
  long long S[3];  // strides 1, K1, K1*K2
  int ndim;
};

Geo make_geo(int ndim, const int64_t* dims) {
  Geo g{};
  g.ndim = ndim;
  g.K[0] = (int)dims[0];
  g.K[1] = ndim > 1 ? (int)dims[1] : 1;
  g.K[2] = ndim > 2 ? (int)dims[2] : 1;
  g.S[0] = 1;
  g.S[1] = g.K[0];
  g.S[2] = (long long)g.K[0] * g.K[1];
  g.N = (long long)g.K[0] * g.K[1] * g.K[2];
  return g;
}

__device__ __forceinline__ int coord(const Geo& g, long long j, int a) {
  return (int)((j / g.S[a]) % g.K[a]);
}

// forward difference along a: D x (j) = x(j + s_a) - x(j), zero on the far face
template <typename T>
__device__ __forceinline__ T fdiff(const Geo& g, const T* __restrict__ x, long long j, int a) {
  return coord(g, j, a) < g.K[a] - 1 ? x[j + g.S[a]] - x[j] : (T)0;
}

// adjoint: (D^T y)(j) = y(j - s_a) [i_a >= 1] - y(j) [i_a < K_a - 1]
// (same order of operations as tv_ops.py:129-131: the -= then the +=)
template <typename T>
__device__ __forceinline__ T adiff(const Geo& g, const T* __restrict__ y, long long j, int a) {
  const int i = coord(g, j, a);
  T o = (T)0;
  if (i < g.K[a] - 1) o -= y[j];
  if (i >= 1) o += y[j - g.S[a]];
  return o;
}

template <typename T>
__global__ void __launch_bounds__(NT) diff_kernel(Geo g, int a, int adjoint, const T* __restrict__ x,
                                                  T* __restrict__ out) {
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < g.N; j += (long long)gridDim.x * NT)
    out[j] = adjoint ? adiff(g, x, j, a) : fdiff(g, x, j, a);
}

template <typename T>
__global__ void __launch_bounds__(NT) grad_stack_kernel(Geo g, const T* __restrict__ x, T* __restrict__ p) {
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < g.N; j += (long long)gridDim.x * NT)
    for (int a = 0; a < g.ndim; ++a) p[a * g.N + j] = fdiff(g, x, j, a);
}

template <typename T>
__global__ void __launch_bounds__(NT) divergence_kernel(Geo g, const T* __restrict__ p, T* __restrict__ out) {
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < g.N; j += (long long)gridDim.x * NT) {
    T s = (T)0;  // tv_ops.py:157-158 accumulates dimension by dimension from zero
    for (int a = 0; a < g.ndim; ++a) s += adiff(g, p + a * g.N, j, a);
    out[j] = s;
  }
}

template <typename T>
__global__ void __launch_bounds__(NT) project_kernel(long long n, int nd, int iso, const T* __restrict__ p,
                                                     T* __restrict__ out) {
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < n; j += (long long)gridDim.x * NT) {
    if (iso) {
      T ss = (T)0;
      for (int a = 0; a < nd; ++a) ss += p[a * n + j] * p[a * n + j];
      const T den = max(sqrt(ss), (T)1);  // p / max(||p_j||, 1), tv_ops.py:177-179
      for (int a = 0; a < nd; ++a) out[a * n + j] = p[a * n + j] / den;
    } else {
      for (int a = 0; a < nd; ++a) out[a * n + j] = min(max(p[a * n + j], (T)-1), (T)1);
    }
  }
}

int grid_blocks(bq_ctx* ctx, long long n) {
  long long want = (n + NT - 1) / NT;
  return (int)std::max<long long>(1, std::min<long long>(want, (long long)ctx->num_sms * 8));
}

}  // namespace
}  // namespace bq

using namespace bq;

#define BQ_GEO_CHECK(ctx, ndim, dims)                                                                         \
  BQ_CHECK(ctx && dims && ndim >= 1 && ndim <= 3, BQ_EINVAL, "tv stencil: bad grid");                       \
  for (int a_ = 0; a_ < ndim; ++a_) BQ_CHECK(dims[a_] >= 1, BQ_EINVAL, "tv stencil: dims must be positive")

extern "C" int bq_tv_diff(bq_ctx* ctx, int32_t dtype, int32_t ndim, const int64_t* dims, int32_t axis,
                          int32_t adjoint, const void* x, void* out, void* stream) {
  BQ_GEO_CHECK(ctx, ndim, dims);
  BQ_CHECK(axis >= 1 && axis <= ndim, BQ_EINVAL, "dimension index %d out of range for %d-D grid", axis, ndim);
  BQ_CHECK(x && out && x != out, BQ_EINVAL, "bq_tv_diff: distinct input and output required");
  const Geo g = make_geo(ndim, dims);
  cudaStream_t st = (cudaStream_t)stream;
  const int G = grid_blocks(ctx, g.N);
  if (dtype == BQ_F32)
    diff_kernel<float><<<G, NT, 0, st>>>(g, axis - 1, adjoint, (const float*)x, (float*)out);
  else
    diff_kernel<double><<<G, NT, 0, st>>>(g, axis - 1, adjoint, (const double*)x, (double*)out);
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_tv_grad_stack(bq_ctx* ctx, int32_t dtype, int32_t ndim, const int64_t* dims, const void* x,
                                void* p_out, void* stream) {
  BQ_GEO_CHECK(ctx, ndim, dims);
  BQ_CHECK(x && p_out, BQ_EINVAL, "bq_tv_grad_stack: null buffer");
  const Geo g = make_geo(ndim, dims);
  cudaStream_t st = (cudaStream_t)stream;
  const int G = grid_blocks(ctx, g.N);
  if (dtype == BQ_F32)
    grad_stack_kernel<float><<<G, NT, 0, st>>>(g, (const float*)x, (float*)p_out);
  else
    grad_stack_kernel<double><<<G, NT, 0, st>>>(g, (const double*)x, (double*)p_out);
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_tv_divergence(bq_ctx* ctx, int32_t dtype, int32_t ndim, const int64_t* dims, const void* p,
                                void* out, void* stream) {
  BQ_GEO_CHECK(ctx, ndim, dims);
  BQ_CHECK(p && out, BQ_EINVAL, "bq_tv_divergence: null buffer");
  const Geo g = make_geo(ndim, dims);
  cudaStream_t st = (cudaStream_t)stream;
  const int G = grid_blocks(ctx, g.N);
  if (dtype == BQ_F32)
    divergence_kernel<float><<<G, NT, 0, st>>>(g, (const float*)p, (float*)out);
  else
    divergence_kernel<double><<<G, NT, 0, st>>>(g, (const double*)p, (double*)out);
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_tv_project_dual(bq_ctx* ctx, int32_t dtype, int32_t ndim, int64_t n, int32_t mode, const void* p,
                                  void* out, void* stream) {
  BQ_CHECK(ctx && p && out && n >= 1 && ndim >= 1 && ndim <= 3, BQ_EINVAL, "bq_tv_project_dual: bad arguments");
  BQ_CHECK(mode == BQ_TV_ISO || mode == BQ_TV_ANISO, BQ_EINVAL, "bq_tv_project_dual: bad mode %d", mode);
  cudaStream_t st = (cudaStream_t)stream;
  const int G = grid_blocks(ctx, n);
  if (dtype == BQ_F32)
    project_kernel<float><<<G, NT, 0, st>>>(n, ndim, mode == BQ_TV_ISO, (const float*)p, (float*)out);
  else
    project_kernel<double><<<G, NT, 0, st>>>(n, ndim, mode == BQ_TV_ISO, (const double*)p, (double*)out);
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}
