// views_dct.cu — the reference's masked-spectrum view operators on the device.
//
// Reference: /root/reference/pkg/src/tvqn/forward_models.py
//   _dct_flat/_idct_flat :86-91   orthonormal DCT-II / DCT-III (scipy.fft.dctn/idctn, norm="ortho")
//   _smooth_flat         :139-150 separable 3-point edge-clamped mean
//   nonlinear_map/jac_vec/adj_vec :166-183  H(x) = M DCT(x + s (Ax)^2) and its JVP/VJP
//   subset_gradient      :304-309 (1/|S|) sum_rho grad f_rho
//   value / data_fidelity:59-61, 286-301
//
// B200 design: the DCT is view-independent, so a subset of |S| views costs ONE
// forward DCT, ONE fused mask-combine kernel (all views of the subset in one
// pass over the spectrum, per-view masks as a 64-bit set per frequency) and
// ONE inverse DCT.  The DCTs are exact separable matrix transforms along each
// axis (cosine table in shared memory, one block per line batch, f64
// accumulation for f64 data), matching scipy's orthonormal DCT to ~1e-15.
#include <mutex>

#include "common.cuh"

namespace bq {
namespace {

constexpr int DCT_MAX = 512;

// One block transforms `lines` lines of length n along `axis` (stride s).
// Table C[k][m] = sqrt(2/n) c_k cos(pi k (2m+1) / (2n)),  c_0 = 1/sqrt(2).
// forward: X[k] = sum_m C[k][m] x[m];  inverse: x[m] = sum_k C[k][m] X[k].
template <typename T>
__global__ void dct_axis_kernel(const T* __restrict__ in, T* __restrict__ out, int n, long long stride,
                                long long inner, long long nlines, int inverse) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* C = reinterpret_cast<double*>(smem_raw);  // n*n (n <= 128) else computed on the fly
  const bool table = n <= 128;
  if (table) {
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
      const int k = i / n, m = i % n;
      const double ck = (k == 0) ? sqrt(1.0 / n) : sqrt(2.0 / n);
      C[i] = ck * cospi((double)k * (2 * m + 1) / (2.0 * n));
    }
  }
  __syncthreads();
  // lines are indexed by (outer, inner) with line start = outer * n * stride + inner
  for (long long line = blockIdx.x; line < nlines; line += gridDim.x) {
    const long long outer = line / inner, inn = line - outer * inner;
    const long long base = outer * (long long)n * stride + inn;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      double acc = 0.0;
      for (int m = 0; m < n; ++m) {
        const double c = table ? (inverse ? C[m * n + k] : C[k * n + m])
                               : (inverse ? ((m == 0 ? sqrt(1.0 / n) : sqrt(2.0 / n)) * cospi((double)m * (2 * k + 1) / (2.0 * n)))
                                          : ((k == 0 ? sqrt(1.0 / n) : sqrt(2.0 / n)) * cospi((double)k * (2 * m + 1) / (2.0 * n))));
        acc += c * (double)in[base + (long long)m * stride];
      }
      out[base + (long long)k * stride] = (T)acc;
    }
  }
}

// Tiled variant for n <= 128 (every axis of the reference's grids): one block
// transforms LB = 32 lines.  The orthonormal table comes precomputed from
// global memory (dct_table, one per n, built once), the tile of 32 lines is
// staged in shared memory with coalesced loads (along the lines for the x
// axis, across adjacent lines for the strided axes), and each thread forms
// n/8 outputs of one line: warps share k, so the table read is a broadcast
// and the tile read is conflict-free.  Same f64 accumulation order as
// dct_axis_kernel (m ascending), so the results are bit-identical to it.
constexpr int DLB = 32;
template <typename T>
__global__ void __launch_bounds__(256) dct_tile_kernel(const T* __restrict__ in, T* __restrict__ out,
                                                       const double* __restrict__ tab, int n, long long stride,
                                                       long long inner, long long nlines, int inverse) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* C = reinterpret_cast<double*>(smem_raw);  // n*n
  double* xs = C + n * n;                           // n rows of DLB+1 (padded)
  constexpr int LP = DLB + 1;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    const int k = i / n, m = i - k * n;
    C[i] = inverse ? tab[m * n + k] : tab[i];  // C[k][m]: the coefficient of x[m] in out[k]
  }
  const bool xaxis = stride == 1;
  for (long long l0 = (long long)blockIdx.x * DLB; l0 < nlines; l0 += (long long)gridDim.x * DLB) {
    const int nl = (int)min((long long)DLB, nlines - l0);
    __syncthreads();
    for (int e = threadIdx.x; e < DLB * n; e += blockDim.x) {
      int l, m;
      if (xaxis) l = e / n, m = e - (e / n) * n;
      else m = e / DLB, l = e - (e / DLB) * DLB;
      if (l < nl) {
        const long long line = l0 + l;
        const long long outer = line / inner, inn = line - outer * inner;
        xs[m * LP + l] = (double)in[outer * (long long)n * stride + inn + (long long)m * stride];
      }
    }
    __syncthreads();
    const int l = threadIdx.x % DLB;
    double res[16];
    int nk = 0;
    for (int k = threadIdx.x / DLB; k < n; k += blockDim.x / DLB, ++nk) {
      double acc = 0.0;
      const double* ck = C + k * n;
      for (int m = 0; m < n; ++m) acc += ck[m] * xs[m * LP + l];
      res[nk] = acc;
    }
    __syncthreads();  // every thread has read the tile: reuse it for the outputs
    nk = 0;
    for (int k = threadIdx.x / DLB; k < n; k += blockDim.x / DLB, ++nk) xs[k * LP + l] = res[nk];
    __syncthreads();
    for (int e = threadIdx.x; e < DLB * n; e += blockDim.x) {
      int ll, k;
      if (xaxis) ll = e / n, k = e - (e / n) * n;
      else k = e / DLB, ll = e - (e / DLB) * DLB;
      if (ll < nl) {
        const long long line = l0 + ll;
        const long long outer = line / inner, inn = line - outer * inner;
        out[outer * (long long)n * stride + inn + (long long)k * stride] = (T)xs[k * LP + ll];
      }
    }
  }
}

__global__ void dct_table_kernel(double* tab, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * n; i += gridDim.x * blockDim.x) {
    const int k = i / n, m = i % n;
    const double ck = (k == 0) ? sqrt(1.0 / n) : sqrt(2.0 / n);
    tab[i] = ck * cospi((double)k * (2 * m + 1) / (2.0 * n));  // the table of dct_axis_kernel
  }
}

// 3-point edge-clamped mean along an axis (forward_models.py:139-150).
template <typename T>
__global__ void smooth_axis_kernel(const T* __restrict__ in, T* __restrict__ out, int n, long long stride,
                                   long long total) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < total; j += (long long)gridDim.x * blockDim.x) {
    const int pos = (int)((j / stride) % n);
    const T c = in[j];
    const T l = pos > 0 ? in[j - stride] : c;
    const T r = pos < n - 1 ? in[j + stride] : c;
    out[j] = (l + c + r) / (T)3;  // ((p[:-2] + p[1:-1]) + p[2:]) / 3
  }
}

struct CombinePtrs {
  const void* y[64];
};

// r = scale * sum_{rho in S} M_rho (F - y_rho); cost[i] = 1/2 ||M_rho F - y_rho||^2 partials.
template <typename T>
__global__ void combine_kernel(long long n, const T* __restrict__ F, CombinePtrs Y, const unsigned long long* __restrict__ masks,
                               const int* __restrict__ views, int count, double scale, T* __restrict__ r,
                               double* __restrict__ cost_partials, int want_cost) {
  __shared__ int s_views[64];
  __shared__ double s_red[64][8];
  if (threadIdx.x < count) s_views[threadIdx.x] = views[threadIdx.x];
  __syncthreads();
  double cacc[64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = 0; i < count; ++i) cacc[i] = 0.0;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    const unsigned long long m = masks[j];
    const T f = F[j];
    T acc = 0;
    for (int i = 0; i < count; ++i) {
      const int v = s_views[i];
      const T yv = ((const T*)Y.y[i])[j];
      const T res = ((m >> v) & 1ull) ? f - yv : -yv;  // M F - y  (y vanishes off-mask up to noise M)
      if ((m >> v) & 1ull) acc += res;
      if (want_cost) cacc[i] += (double)res * (double)res;
    }
    if (r) r[j] = (T)(scale * (double)acc);
  }
  if (want_cost) {
    for (int i = 0; i < count; ++i) {
      double s = cacc[i];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) s_red[i][warp] = s;
    }
    __syncthreads();
    if (threadIdx.x < count) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x / 32); ++w) s += s_red[threadIdx.x][w];
      cost_partials[(long long)blockIdx.x * 64 + threadIdx.x] = s;
    }
  }
}

template <typename T>
__global__ void cost_finish_kernel(const double* partials, int nblocks, int count, double* out) {
  const int i = threadIdx.x;
  if (i < count) {
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += partials[(long long)b * 64 + i];
    out[i] = 0.5 * s;
  }
}

// pointwise helpers for the chain rule (forward_models.py:166-183)
//  op 0: out = x + s * a * a            (f(x), a = A x)
//  op 1: out = w + 2 s * a * b          (JVP inner, a = A x, b = A w)
//  op 2: out = a * b                    (product)
//  op 3: out = q + 2 s * b              (VJP tail, b = A(Ax . q))
//  op 4: out = alpha * x                (scale)
template <typename T>
__global__ void pointwise_kernel(int op, long long n, const T* __restrict__ x, const T* __restrict__ a,
                                 const T* __restrict__ b, double s, T* __restrict__ out) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    switch (op) {
      case 0: out[j] = x[j] + (T)s * a[j] * a[j]; break;
      case 1: out[j] = x[j] + (T)(2.0 * s) * a[j] * b[j]; break;
      case 2: out[j] = a[j] * b[j]; break;
      case 3: out[j] = x[j] + (T)(2.0 * s) * b[j]; break;
      default: out[j] = (T)s * x[j]; break;
    }
  }
}

int grid_for(bq_ctx* ctx, long long n, int nt) {
  long long want = (n + nt - 1) / nt;
  return (int)std::max<long long>(1, std::min<long long>(want, (long long)ctx->num_sms * 8));
}

// orthonormal DCT tables, one per (context, n), built once on first use
struct DctTab {
  bq_ctx* ctx;
  int n;
  double* tab;
};
DctTab g_tabs[64];
int g_ntabs = 0;
std::mutex g_tab_mu;

const double* dct_table(bq_ctx* ctx, int n, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(g_tab_mu);
  for (int i = 0; i < g_ntabs; ++i)
    if (g_tabs[i].ctx == ctx && g_tabs[i].n == n) return g_tabs[i].tab;
  if (g_ntabs == 64) return nullptr;
  double* tab = nullptr;
  if (cudaMalloc(&tab, (size_t)n * n * sizeof(double)) != cudaSuccess) return nullptr;
  dct_table_kernel<<<(n * n + 255) / 256, 256, 0, st>>>(tab, n);
  g_tabs[g_ntabs++] = DctTab{ctx, n, tab};
  return tab;
}

}  // namespace
}  // namespace bq

using namespace bq;

extern "C" int bq_dct_axis(bq_ctx* ctx, int32_t dtype, const int64_t* dims, int32_t axis, int32_t inverse,
                           const void* in, void* out, void* stream) {
  BQ_CHECK(ctx && dims && in && out && in != out, BQ_EINVAL, "bq_dct_axis: bad arguments (in-place unsupported)");
  BQ_CHECK(axis >= 0 && axis < 3, BQ_EINVAL, "bq_dct_axis: axis must be 0..2");
  const int n = (int)dims[axis];
  BQ_CHECK(n >= 1 && n <= DCT_MAX, BQ_EINVAL, "bq_dct_axis: axis length %d outside [1, %d]", n, DCT_MAX);
  long long stride = 1;
  for (int a = 0; a < axis; ++a) stride *= dims[a];
  const long long total = dims[0] * dims[1] * dims[2];
  const long long nlines = total / n;
  const long long inner = stride;
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 128 && !getenv("BQ_DCT_NAIVE")) {
    const double* tab = dct_table(ctx, n, st);
    BQ_CHECK(tab, BQ_ECUDA, "bq_dct_axis: table allocation failed");
    const size_t shm = ((size_t)n * n + (size_t)n * (DLB + 1)) * sizeof(double);
    const int G = (int)std::max<long long>(1, std::min<long long>((nlines + DLB - 1) / DLB, (long long)ctx->num_sms * 8));
    if (dtype == BQ_F32) {
      BQ_CUDA(cudaFuncSetAttribute(dct_tile_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      dct_tile_kernel<float><<<G, 256, shm, st>>>((const float*)in, (float*)out, tab, n, stride, inner, nlines, inverse);
    } else {
      BQ_CUDA(cudaFuncSetAttribute(dct_tile_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      dct_tile_kernel<double><<<G, 256, shm, st>>>((const double*)in, (double*)out, tab, n, stride, inner, nlines,
                                                   inverse);
    }
    BQ_CUDA(cudaGetLastError());
    return BQ_OK;
  }
  const size_t shm = n <= 128 ? (size_t)n * n * sizeof(double) : 0;
  const int nt = n <= 128 ? 128 : 256;
  const int G = (int)std::min<long long>(nlines, (long long)ctx->num_sms * 16);
  if (dtype == BQ_F32) {
    BQ_CUDA(cudaFuncSetAttribute(dct_axis_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    dct_axis_kernel<float><<<G, nt, shm, st>>>((const float*)in, (float*)out, n, stride, inner, nlines, inverse);
  } else {
    BQ_CUDA(cudaFuncSetAttribute(dct_axis_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    dct_axis_kernel<double><<<G, nt, shm, st>>>((const double*)in, (double*)out, n, stride, inner, nlines, inverse);
  }
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_smooth_axis(bq_ctx* ctx, int32_t dtype, const int64_t* dims, int32_t axis, const void* in,
                              void* out, void* stream) {
  BQ_CHECK(ctx && dims && in && out && in != out, BQ_EINVAL, "bq_smooth_axis: bad arguments");
  BQ_CHECK(axis >= 0 && axis < 3, BQ_EINVAL, "bq_smooth_axis: axis must be 0..2");
  long long stride = 1;
  for (int a = 0; a < axis; ++a) stride *= dims[a];
  const long long total = dims[0] * dims[1] * dims[2];
  cudaStream_t st = (cudaStream_t)stream;
  const int G = grid_for(ctx, total, 256);
  if (dtype == BQ_F32)
    smooth_axis_kernel<float><<<G, 256, 0, st>>>((const float*)in, (float*)out, (int)dims[axis], stride, total);
  else
    smooth_axis_kernel<double><<<G, 256, 0, st>>>((const double*)in, (double*)out, (int)dims[axis], stride, total);
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_views_combine(bq_ctx* ctx, int32_t dtype, int64_t n, const void* F, const void* const* ys,
                                const uint64_t* masks, const int32_t* views_dev, int32_t count, double scale,
                                void* r_out, double* cost_out, void* stream) {
  BQ_CHECK(ctx && F && ys && masks && views_dev && n > 0, BQ_EINVAL, "bq_views_combine: bad arguments");
  BQ_CHECK(count >= 1 && count <= 64, BQ_EINVAL, "bq_views_combine: 1..64 views per call");
  CombinePtrs Y{};
  for (int i = 0; i < count; ++i) Y.y[i] = ys[i];
  cudaStream_t st = (cudaStream_t)stream;
  const int G = std::min(grid_for(ctx, n, 256), 1024);
  BQ_STREAM_WS(sw, ctx, st);
  double* partials = sw->ws.partials;  // >= 1024 * 64 doubles (kMaxBlocks * kMaxVals)
  if (dtype == BQ_F32)
    combine_kernel<float><<<G, 256, 0, st>>>(n, (const float*)F, Y, (const unsigned long long*)masks, views_dev, count, scale, (float*)r_out,
                                              partials, cost_out != nullptr);
  else
    combine_kernel<double><<<G, 256, 0, st>>>(n, (const double*)F, Y, (const unsigned long long*)masks, views_dev, count, scale,
                                               (double*)r_out, partials, cost_out != nullptr);
  if (cost_out) cost_finish_kernel<double><<<1, 64, 0, st>>>(partials, G, count, cost_out);
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_pointwise(bq_ctx* ctx, int32_t dtype, int32_t op, int64_t n, const void* x, const void* a,
                            const void* b, double s, void* out, void* stream) {
  BQ_CHECK(ctx && out && n > 0 && op >= 0 && op <= 4, BQ_EINVAL, "bq_pointwise: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const int G = grid_for(ctx, n, 256);
  if (dtype == BQ_F32)
    pointwise_kernel<float><<<G, 256, 0, st>>>(op, n, (const float*)x, (const float*)a, (const float*)b, s, (float*)out);
  else
    pointwise_kernel<double><<<G, 256, 0, st>>>(op, n, (const double*)x, (const double*)a, (const double*)b, s,
                                                (double*)out);
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}
