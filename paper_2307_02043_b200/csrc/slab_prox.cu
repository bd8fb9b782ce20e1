// slab_prox.cu — one rank's passes of the z-slab-sharded weighted-TV prox.
//
// The FGP loop of dual_tv_solver.py:221-239 (and the structured projection of
// wpm.py:145-231 inside it) over a volume split along dims[2] into contiguous
// slabs, one per GPU.  Each FGP iteration is four stream-ordered passes over
// the rank's slab, with the cross-rank steps between them issued by the host
// (paper_2307_02043_b200/slab_prox.py) on the NCCL communicator:
//
//   bq_slab_div     t = D^-1 div(Pbar), s = U^T t           needs Pbar_z of plane z0-1 (halo from below)
//                   -> all-reduce(s, r doubles);  c = cap^-1 s on the host
//   bq_slab_newton  phi = U^T (w - clamp(z)), H = U_A^T D_A^-1 U_A at beta
//                   with w = v - reg (t - sign D^-1 U c), z = w - sign D^-1 U beta
//                   -> all-reduce(phi, H: r + r(r+1)/2 doubles) per Newton step
//   bq_slab_q       q = clamp(z(beta*))
//                   -> q of plane z1 from the rank above (halo)
//   bq_slab_dual    P_next = project(Pbar + step grad q), ||P_next - P||^2, ||P||^2,
//                   Pbar_next = P_next + m (P_next - P)     -> all-reduce(2 doubles)
//
// Per-block partial sums are reduced in block order by the last block
// (deterministic); every rank holds bit-identical scalars after the
// all-reduce, so the host controller (Newton accept / Levenberg / best
// residual, the FISTA t-sequence, the rel-change stop) takes the same branch
// on every rank.  Layout as the single-GPU prox: flat Fortran order over
// (K1, K2, L) for the local slab, U as rank contiguous local N-vectors, the
// dual field as 3 contiguous local N-vectors.
#include <algorithm>

#include "common.cuh"
#include "prox_common.cuh"
#include "reduce.cuh"

namespace bq {
namespace {

constexpr int NT = 256;

struct SlabArgs {
  long long N;      // local voxels K1*K2*L
  long long plane;  // K1*K2
  int K1, K2, L;
  int first, last;  // slab holds global plane 0 / K3-1
  int rank, sign, iso;
  double tau, reg, lo, hi;
  const void* d;
  const void* U;
  const void* v;
  double c[BQ_MAX_RANK];     // cap^-1 (U^T D^-1 div)  (Woodbury coefficient, global)
  double beta[BQ_MAX_RANK];  // Newton point
  const double* ctl;         // optional device control block: c and beta read from it
};

constexpr int C_DONE = 0, C_IT = 1, C_BEST = 2, C_TOTAL = 3, C_REL = 4, C_FGP = 5, C_LAST = 6, C_BETA = 8,
              C_BBETA = 16, C_COEF = 24, C_SAVED = 32, C_CHOL = 40;

// c and beta of this launch, in shared memory (from the control block when set)
template <int R>
__device__ __forceinline__ void load_cb(const SlabArgs& A, double* s_c, double* s_b) {
  if (threadIdx.x < R) {
    s_c[threadIdx.x] = A.ctl ? A.ctl[C_COEF + threadIdx.x] : A.c[threadIdx.x];
    s_b[threadIdx.x] = A.ctl ? A.ctl[C_BETA + threadIdx.x] : A.beta[threadIdx.x];
  }
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ T inv_d(const SlabArgs& A, long long j) {
  return A.d ? (T)1 / ((const T*)A.d)[j] : (T)(1.0 / A.tau);
}

// w_j = v_j - reg (t_j - sign D^-1 U c)   (dual_tv_solver.py:119-123 with the Woodbury inverse)
template <typename T, int R>
__device__ __forceinline__ T center(const SlabArgs& A, const double* cf, const T* __restrict__ t, long long j, T idj) {
  const T* U = (const T*)A.U;
  T uc = (T)0;
#pragma unroll
  for (int k = 0; k < R; ++k) uc += U[k * A.N + j] * (T)cf[k];
  const T corr = (R > 0) ? t[j] - (T)A.sign * uc * idj : t[j];
  return ((const T*)A.v)[j] - (T)A.reg * corr;
}

// ---------------------------------------------------------------------------
// t = D^-1 div(F), s = U^T t    (F = Pbar or P; halo = F_z of global plane z0-1)
// ---------------------------------------------------------------------------
template <typename T, int R>
__global__ void __launch_bounds__(NT) div_kernel(SlabArgs A, const T* __restrict__ F, const T* __restrict__ halo,
                                                 T* __restrict__ t, double* s_out, RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  constexpr int NA = R > 0 ? R : 1;
  double acc[NA];
#pragma unroll
  for (int k = 0; k < NA; ++k) acc[k] = 0.0;
  const T* Fx = F;
  const T* Fy = F + A.N;
  const T* Fz = F + 2 * A.N;
  const T* U = (const T*)A.U;
  // groups of RB whole x-rows per block step (RB = NT / K1 for short rows): the
  // coordinates come from 32-bit row arithmetic, no per-voxel 64-bit division
  const int rows = A.K2 * A.L;
  const int RB = A.K1 >= NT ? 1 : NT / A.K1;
  const int span = RB * A.K1;
  for (int row0 = blockIdx.x * RB; row0 < rows; row0 += gridDim.x * RB)
  for (int e = threadIdx.x; e < span; e += NT) {
    const int sub = e / A.K1;
    const int ix = e - sub * A.K1;
    const int row = row0 + sub;
    if (row >= rows) break;
    const int iy = row % A.K2;
    const int iz = row / A.K2;
    const long long j = (long long)row * A.K1 + ix;
    // sum_a (D^a)^T F_a, term order of tv_ops.py:129-131 per axis, axes accumulated from 0
    T dv = (T)0;
    {
      T o = (T)0;
      if (ix < A.K1 - 1) o -= Fx[j];
      if (ix >= 1) o += Fx[j - 1];
      dv += o;
    }
    {
      T o = (T)0;
      if (iy < A.K2 - 1) o -= Fy[j];
      if (iy >= 1) o += Fy[j - A.K1];
      dv += o;
    }
    {
      T o = (T)0;
      if (!(A.last && iz == A.L - 1)) o -= Fz[j];
      if (iz >= 1) o += Fz[j - A.plane];
      else if (!A.first) o += halo[j];  // plane z0-1 of the rank below
      dv += o;
    }
    const T tj = dv * inv_d<T>(A, j);
    t[j] = tj;
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] += (double)U[k * A.N + j] * (double)tj;
  }
  if (R > 0) {
    if (last_block_reduce<NT, NA>(acc, R, ws, red, scr) && threadIdx.x < R) s_out[threadIdx.x] = red[threadIdx.x];
  }
}

// ---------------------------------------------------------------------------
// Newton residual and generalized Jacobian at beta (wpm.py:150-167):
//   out[0..R)            sum_j U_c (w_j - clamp(z_j))
//   out[R + tri(c, c')]  sum_{j inside} U_c U_c' * (1/d_j or 1: the host divides by tau)
// ---------------------------------------------------------------------------
template <typename T, int R>
__global__ void __launch_bounds__(NT) newton_kernel(SlabArgs A, const T* __restrict__ t, double* out, RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  __shared__ double s_c[R], s_b[R];
  if (A.ctl && A.ctl[C_DONE] != 0.0) return;  // uniform: the Newton already stopped
  load_cb<R>(A, s_c, s_b);
  constexpr int NV = R + R * (R + 1) / 2;
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  const T* U = (const T*)A.U;
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < A.N; j += (long long)gridDim.x * NT) {
    const T idj = inv_d<T>(A, j);
    const T w = center<T, R>(A, s_c, t, j, idj);
    T u[R];
    T ub = (T)0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      u[k] = U[k * A.N + j];
      ub += u[k] * (T)s_b[k];
    }
    const T z = A.d ? w - (T)A.sign * ub * idj : w - (T)A.sign * ub / (T)A.tau;
    const T q = min(max(z, (T)A.lo), (T)A.hi);
    const T r = w - q;
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] += (double)(u[k] * r);
    if (z > (T)A.lo && z < (T)A.hi) {  // ties count as outside (wpm.py:161-167)
      const T sc = A.d ? idj : (T)1;
      int m = R;
#pragma unroll
      for (int k = 0; k < R; ++k)
#pragma unroll
        for (int k2 = 0; k2 <= k; ++k2, ++m) acc[m] += (double)(u[k] * u[k2] * sc);
    }
  }
  if (last_block_reduce<NT, NV>(acc, NV, ws, red, scr) && threadIdx.x < NV) out[threadIdx.x] = red[threadIdx.x];
}

// q = clamp(z(beta))   (wpm.py:246-253)
template <typename T, int R>
__global__ void __launch_bounds__(NT) q_kernel(SlabArgs A, const T* __restrict__ t, T* __restrict__ q) {
  constexpr int RR = R > 0 ? R : 1;
  __shared__ double s_c[RR], s_b[RR];
  load_cb<R>(A, s_c, s_b);
  const T* U = (const T*)A.U;
  for (long long j = (long long)blockIdx.x * NT + threadIdx.x; j < A.N; j += (long long)gridDim.x * NT) {
    const T idj = inv_d<T>(A, j);
    const T w = center<T, R>(A, s_c, t, j, idj);
    T ub = (T)0;
#pragma unroll
    for (int k = 0; k < R; ++k) ub += U[k * A.N + j] * (T)s_b[k];
    const T z = (R == 0) ? w : (A.d ? w - (T)A.sign * ub * idj : w - (T)A.sign * ub / (T)A.tau);
    q[j] = min(max(z, (T)A.lo), (T)A.hi);
  }
}

// ---------------------------------------------------------------------------
// dual update (dual_tv_solver.py:227-239): P_next = project(Pbar + step grad q)
// norms: ||P_next - P||^2, ||P||^2 ; Pbar_next = P_next + m (P_next - P)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(NT) dual_kernel(SlabArgs A, const T* __restrict__ pbar, const T* __restrict__ p,
                                                  const T* __restrict__ q, const T* __restrict__ halo_q,
                                                  double step, double mom, T* __restrict__ pn,
                                                  T* __restrict__ pbn, double* norms, RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  double acc[2] = {0.0, 0.0};
  const long long N = A.N;
  // groups of RB whole x-rows per block step (RB = NT / K1 for short rows): the
  // coordinates come from 32-bit row arithmetic, no per-voxel 64-bit division
  const int rows = A.K2 * A.L;
  const int RB = A.K1 >= NT ? 1 : NT / A.K1;
  const int span = RB * A.K1;
  for (int row0 = blockIdx.x * RB; row0 < rows; row0 += gridDim.x * RB)
  for (int e = threadIdx.x; e < span; e += NT) {
    const int sub = e / A.K1;
    const int ix = e - sub * A.K1;
    const int row = row0 + sub;
    if (row >= rows) break;
    const int iy = row % A.K2;
    const int iz = row / A.K2;
    const long long j = (long long)row * A.K1 + ix;
    const T qj = q[j];
    T g[3];
    g[0] = ix < A.K1 - 1 ? q[j + 1] - qj : (T)0;
    g[1] = iy < A.K2 - 1 ? q[j + A.K1] - qj : (T)0;
    if (iz < A.L - 1)
      g[2] = q[j + A.plane] - qj;
    else
      g[2] = A.last ? (T)0 : halo_q[j - (long long)(A.L - 1) * A.plane] - qj;
    T w[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) w[a] = pbar[a * N + j] + (T)step * g[a];
    if (A.iso) {
      const T den = max(sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]), (T)1);  // tv_ops.py:177-179
#pragma unroll
      for (int a = 0; a < 3; ++a) w[a] = w[a] / den;
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a) w[a] = min(max(w[a], (T)-1), (T)1);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const T pa = p[a * N + j];
      const T dlt = w[a] - pa;
      acc[0] += (double)dlt * (double)dlt;
      acc[1] += (double)pa * (double)pa;
      pn[a * N + j] = w[a];
      pbn[a * N + j] = w[a] + (T)mom * dlt;
    }
  }
  if (last_block_reduce<NT, 2>(acc, 2, ws, red, scr) && threadIdx.x < 2) norms[threadIdx.x] = red[threadIdx.x];
}

// ---------------------------------------------------------------------------
// The same four passes on 4 consecutive x-voxels per thread (16-byte accesses;
// K1 % 4 == 0 and 16-byte aligned fields), the per-voxel arithmetic unchanged.
// At 256^3 on one slab the scalar passes ran at 2.5-4 TB/s of DRAM traffic.
// ---------------------------------------------------------------------------
using prox::Vec4;

// row / quad coordinates of work item e of a block step (RB rows of K1 / 4 quads)
struct QuadPos {
  int ix, iy, iz;
  long long j;
  bool ok;
};
__device__ __forceinline__ QuadPos quad_pos(const SlabArgs& A, int row0, int e, int rows) {
  const int qpr = A.K1 >> 2;
  const int sub = e / qpr;
  QuadPos q;
  q.ix = (e - sub * qpr) << 2;
  const int row = row0 + sub;
  q.ok = row < rows;
  q.iy = row % A.K2;
  q.iz = row / A.K2;
  q.j = (long long)row * A.K1 + q.ix;
  return q;
}

template <typename T>
__device__ __forceinline__ void inv_d4(const SlabArgs& A, long long j, T (&id)[4]) {
  if (A.d) {
    T dd[4];
    Vec4<T>::ro((const T*)A.d + j, dd);
#pragma unroll
    for (int k = 0; k < 4; ++k) id[k] = (T)1 / dd[k];
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) id[k] = (T)(1.0 / A.tau);
  }
}

template <typename T, int R>
__global__ void __launch_bounds__(NT) div_kernel4(SlabArgs A, const T* __restrict__ F, const T* __restrict__ halo,
                                                  T* __restrict__ t, double* s_out, RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  constexpr int NA = R > 0 ? R : 1;
  double acc[NA];
#pragma unroll
  for (int k = 0; k < NA; ++k) acc[k] = 0.0;
  const T* Fx = F;
  const T* Fy = F + A.N;
  const T* Fz = F + 2 * A.N;
  const T* U = (const T*)A.U;
  const int rows = A.K2 * A.L;
  const int qpr = A.K1 >> 2;
  const int RB = qpr >= NT ? 1 : NT / qpr;
  const int span = RB * qpr;
  for (int row0 = blockIdx.x * RB; row0 < rows; row0 += gridDim.x * RB)
    for (int e = threadIdx.x; e < span; e += NT) {
      const QuadPos P = quad_pos(A, row0, e, rows);
      if (!P.ok) break;
      const long long j = P.j;
      T fx[4], fy[4], fz[4], ym[4], zm[4], id[4];
      Vec4<T>::rw(Fx + j, fx);
      Vec4<T>::rw(Fy + j, fy);
      Vec4<T>::rw(Fz + j, fz);
      const T xm = P.ix >= 1 ? Fx[j - 1] : (T)0;
      const bool has_ym = P.iy >= 1, has_zm = P.iz >= 1, has_halo = !has_zm && !A.first;
      if (has_ym) Vec4<T>::rw(Fy + j - A.K1, ym);
      if (has_zm) Vec4<T>::rw(Fz + j - A.plane, zm);
      else if (has_halo) Vec4<T>::rw(halo + j, zm);  // plane z0-1 of the rank below
      inv_d4<T>(A, j, id);
      T tj[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // sum_a (D^a)^T F_a, term order of tv_ops.py:129-131 per axis, axes accumulated from 0
        T dv = (T)0;
        {
          T o = (T)0;
          if (P.ix + k < A.K1 - 1) o -= fx[k];
          if (P.ix + k >= 1) o += k == 0 ? xm : fx[k - 1];
          dv += o;
        }
        {
          T o = (T)0;
          if (P.iy < A.K2 - 1) o -= fy[k];
          if (has_ym) o += ym[k];
          dv += o;
        }
        {
          T o = (T)0;
          if (!(A.last && P.iz == A.L - 1)) o -= fz[k];
          if (has_zm || has_halo) o += zm[k];
          dv += o;
        }
        tj[k] = dv * id[k];
      }
      Vec4<T>::st(t + j, tj);
#pragma unroll
      for (int c = 0; c < R; ++c) {
        T u[4];
        Vec4<T>::ro(U + c * A.N + j, u);
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[c] += (double)u[k] * (double)tj[k];
      }
    }
  if (R > 0) {
    if (last_block_reduce<NT, NA>(acc, R, ws, red, scr) && threadIdx.x < R) s_out[threadIdx.x] = red[threadIdx.x];
  }
}

// w (center) and z(beta) of 4 voxels; u returned for the Newton sums
template <typename T, int R>
__device__ __forceinline__ void center_z4(const SlabArgs& A, const double* s_c, const double* s_b,
                                          const T* __restrict__ t, long long j, T (&w)[4], T (&z)[4], T (&id)[4],
                                          T (&u)[R > 0 ? R : 1][4]) {
  const T* U = (const T*)A.U;
  T tv[4], vv[4];
  Vec4<T>::rw(t + j, tv);
  Vec4<T>::ro((const T*)A.v + j, vv);
  inv_d4<T>(A, j, id);
#pragma unroll
  for (int c = 0; c < R; ++c) Vec4<T>::ro(U + c * A.N + j, u[c]);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    T uc = (T)0, ub = (T)0;
#pragma unroll
    for (int c = 0; c < R; ++c) uc += u[c][k] * (T)s_c[c];
#pragma unroll
    for (int c = 0; c < R; ++c) ub += u[c][k] * (T)s_b[c];
    const T corr = (R > 0) ? tv[k] - (T)A.sign * uc * id[k] : tv[k];
    w[k] = vv[k] - (T)A.reg * corr;
    z[k] = (R == 0) ? w[k] : (A.d ? w[k] - (T)A.sign * ub * id[k] : w[k] - (T)A.sign * ub / (T)A.tau);
  }
}

template <typename T, int R>
__global__ void __launch_bounds__(NT) newton_kernel4(SlabArgs A, const T* __restrict__ t, double* out, RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  __shared__ double s_c[R], s_b[R];
  if (A.ctl && A.ctl[C_DONE] != 0.0) return;  // uniform: the Newton already stopped
  load_cb<R>(A, s_c, s_b);
  constexpr int NV = R + R * (R + 1) / 2;
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  for (long long j = 4 * ((long long)blockIdx.x * NT + threadIdx.x); j < A.N; j += 4LL * gridDim.x * NT) {
    T w[4], z[4], id[4], u[R][4];
    center_z4<T, R>(A, s_c, s_b, t, j, w, z, id, u);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const T q = min(max(z[k], (T)A.lo), (T)A.hi);
      const T r = w[k] - q;
#pragma unroll
      for (int c = 0; c < R; ++c) acc[c] += (double)(u[c][k] * r);
      if (z[k] > (T)A.lo && z[k] < (T)A.hi) {  // ties count as outside (wpm.py:161-167)
        const T sc = A.d ? id[k] : (T)1;
        int m = R;
#pragma unroll
        for (int c = 0; c < R; ++c)
#pragma unroll
          for (int c2 = 0; c2 <= c; ++c2, ++m) acc[m] += (double)(u[c][k] * u[c2][k] * sc);
      }
    }
  }
  if (last_block_reduce<NT, NV>(acc, NV, ws, red, scr) && threadIdx.x < NV) out[threadIdx.x] = red[threadIdx.x];
}

template <typename T, int R>
__global__ void __launch_bounds__(NT) q_kernel4(SlabArgs A, const T* __restrict__ t, T* __restrict__ q) {
  constexpr int RR = R > 0 ? R : 1;
  __shared__ double s_c[RR], s_b[RR];
  load_cb<R>(A, s_c, s_b);
  for (long long j = 4 * ((long long)blockIdx.x * NT + threadIdx.x); j < A.N; j += 4LL * gridDim.x * NT) {
    T w[4], z[4], id[4], u[RR][4];
    center_z4<T, R>(A, s_c, s_b, t, j, w, z, id, u);
#pragma unroll
    for (int k = 0; k < 4; ++k) z[k] = min(max(z[k], (T)A.lo), (T)A.hi);
    Vec4<T>::st(q + j, z);
  }
}

template <typename T>
__global__ void __launch_bounds__(NT) dual_kernel4(SlabArgs A, const T* __restrict__ pbar, const T* __restrict__ p,
                                                   const T* __restrict__ q, const T* __restrict__ halo_q,
                                                   double step, double mom, T* __restrict__ pn,
                                                   T* __restrict__ pbn, double* norms, RedWs ws) {
  __shared__ double red[kMaxVals];
  __shared__ double scr[(NT / 32) * kMaxVals];
  double acc[2] = {0.0, 0.0};
  const long long N = A.N;
  const int rows = A.K2 * A.L;
  const int qpr = A.K1 >> 2;
  const int RB = qpr >= NT ? 1 : NT / qpr;
  const int span = RB * qpr;
  for (int row0 = blockIdx.x * RB; row0 < rows; row0 += gridDim.x * RB)
    for (int e = threadIdx.x; e < span; e += NT) {
      const QuadPos P = quad_pos(A, row0, e, rows);
      if (!P.ok) break;
      const long long j = P.j;
      T qj[4], qy[4], qz[4], pb[3][4], pp[3][4];
      Vec4<T>::rw(q + j, qj);
      const bool has_x = P.ix + 4 < A.K1, has_y = P.iy < A.K2 - 1, in_z = P.iz < A.L - 1, has_z = in_z || !A.last;
      const T qx = has_x ? q[j + 4] : (T)0;
      if (has_y) Vec4<T>::rw(q + j + A.K1, qy);
      if (in_z) Vec4<T>::rw(q + j + A.plane, qz);
      else if (has_z) Vec4<T>::rw(halo_q + j - (long long)(A.L - 1) * A.plane, qz);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        Vec4<T>::rw(pbar + a * N + j, pb[a]);
        Vec4<T>::rw(p + a * N + j, pp[a]);
      }
      T wn[3][4], wb[3][4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        T g[3];
        g[0] = (k < 3 || has_x) ? (k < 3 ? qj[k + 1] : qx) - qj[k] : (T)0;
        g[1] = has_y ? qy[k] - qj[k] : (T)0;
        g[2] = has_z ? qz[k] - qj[k] : (T)0;
        T w[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) w[a] = pb[a][k] + (T)step * g[a];
        if (A.iso) {
          const T den = max(sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]), (T)1);  // tv_ops.py:177-179
#pragma unroll
          for (int a = 0; a < 3; ++a) w[a] = w[a] / den;
        } else {
#pragma unroll
          for (int a = 0; a < 3; ++a) w[a] = min(max(w[a], (T)-1), (T)1);
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const T pa = pp[a][k];
          const T dlt = w[a] - pa;
          acc[0] += (double)dlt * (double)dlt;
          acc[1] += (double)pa * (double)pa;
          wn[a][k] = w[a];
          wb[a][k] = w[a] + (T)mom * dlt;
        }
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        Vec4<T>::st(pn + a * N + j, wn[a]);
        Vec4<T>::st(pbn + a * N + j, wb[a]);
      }
    }
  if (last_block_reduce<NT, 2>(acc, 2, ws, red, scr) && threadIdx.x < 2) norms[threadIdx.x] = red[threadIdx.x];
}

inline bool al16(const void* q) { return q == nullptr || ((uintptr_t)q & 15u) == 0; }
// 4 voxels per thread: whole quads per x-row and 16-byte aligned fields
inline bool quad_ok(const SlabArgs& A, std::initializer_list<const void*> ptrs) {
  static const bool off = [] {
    const char* e = getenv("BQ_SLAB_SCALAR");
    return e && e[0] == '1';
  }();
  if (off || (A.K1 & 3)) return false;
  for (const void* q : ptrs)
    if (!al16(q)) return false;
  return al16(A.d) && al16(A.U) && al16(A.v);
}

// ---------------------------------------------------------------------------
// device control (bq_slab_ctl): one thread, the reference's scalar logic
// ---------------------------------------------------------------------------
__device__ bool lu_solve(double* h, double* b, int r) {
  for (int k = 0; k < r; ++k) {  // partial pivoting; an exactly zero pivot = singular (LinAlgError)
    int p = k;
    for (int i = k + 1; i < r; ++i)
      if (fabs(h[i * r + k]) > fabs(h[p * r + k])) p = i;
    if (h[p * r + k] == 0.0) return false;
    if (p != k) {
      for (int j = 0; j < r; ++j) {
        const double tmp = h[k * r + j];
        h[k * r + j] = h[p * r + j];
        h[p * r + j] = tmp;
      }
      const double tb = b[k];
      b[k] = b[p];
      b[p] = tb;
    }
    for (int i = k + 1; i < r; ++i) {
      const double f = h[i * r + k] / h[k * r + k];
      for (int j = k; j < r; ++j) h[i * r + j] -= f * h[k * r + j];
      b[i] -= f * b[k];
    }
  }
  for (int i = r - 1; i >= 0; --i) {
    double s = b[i];
    for (int j = i + 1; j < r; ++j) s -= h[i * r + j] * b[j];
    b[i] = s / h[i * r + i];
  }
  return true;
}

__global__ void slab_ctl_kernel(int op, int r, int sign, double tau, int scalar, const double* in, double neps,
                                int nmax, double eps, double* c) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  switch (op) {
    case 0: {  // INIT
      for (int i = 0; i < r * r; ++i) c[C_CHOL + i] = in[i];
      for (int i = 0; i < r; ++i) c[C_BETA + i] = in[64 + i];
      c[C_TOTAL] = 0.0;
      c[C_FGP] = 0.0;
      c[C_REL] = INFINITY;
      c[C_DONE] = (r == 0) ? 1.0 : 0.0;
      return;
    }
    case 1: {  // COEF: c = cap^-1 s (L L^T solve), Newton reset
      const double* L = c + C_CHOL;
      double b[8];
      for (int i = 0; i < r; ++i) b[i] = in[i];
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
      for (int i = 0; i < r; ++i) {
        c[C_COEF + i] = b[i];
        c[C_SAVED + i] = c[C_BETA + i];
        c[C_BBETA + i] = c[C_BETA + i];
      }
      c[C_BEST] = INFINITY;
      c[C_IT] = 0.0;
      c[C_LAST] = 0.0;
      c[C_DONE] = (r == 0) ? 1.0 : 0.0;
      return;
    }
    case 2: {  // NEWTON step on the all-reduced residual / Jacobian
      if (c[C_DONE] != 0.0) return;
      double phi[8], res2 = 0.0;
      for (int i = 0; i < r; ++i) {
        phi[i] = in[i] + c[C_BETA + i];
        res2 += phi[i] * phi[i];
      }
      const double res = sqrt(res2);
      if (res < c[C_BEST]) {
        c[C_BEST] = res;
        for (int i = 0; i < r; ++i) c[C_BBETA + i] = c[C_BETA + i];
      }
      const int it = (int)c[C_IT];
      bool stop = res <= neps || it == nmax;
      if (!stop) {
        double h[64], hs[64], st[8];
        int k = r;
        for (int i = 0; i < r; ++i)
          for (int j = 0; j <= i; ++j, ++k) {
            const double g = scalar ? in[k] / tau : in[k];
            h[i * r + j] = h[j * r + i] = (i == j ? 1.0 : 0.0) + sign * g;
          }
        for (int i = 0; i < r * r; ++i) hs[i] = h[i];
        for (int i = 0; i < r; ++i) st[i] = phi[i];
        if (!lu_solve(hs, st, r)) {  // Levenberg fallback, wpm.py:219-223
          double ninf = 0.0;
          for (int i = 0; i < r; ++i) {
            double rs = 0.0;
            for (int j = 0; j < r; ++j) rs += fabs(h[i * r + j]);
            ninf = fmax(ninf, rs);
          }
          for (int i = 0; i < r * r; ++i) hs[i] = h[i];
          for (int i = 0; i < r; ++i) hs[i * r + i] += 1e-8 * ninf, st[i] = phi[i];
          lu_solve(hs, st, r);
        }
        for (int i = 0; i < r; ++i) c[C_BETA + i] -= st[i];
        c[C_IT] = it + 1;
      } else {
        for (int i = 0; i < r; ++i) c[C_BETA + i] = c[C_BBETA + i];
        c[C_LAST] = it;
        c[C_TOTAL] += it;
        c[C_DONE] = 1.0;
      }
      return;
    }
    case 3: {  // NORMS
      const double num = sqrt(in[0]), den = sqrt(in[1]);
      const double rel = (num == 0.0) ? 0.0 : (den > 0.0 ? num / den : INFINITY);
      c[C_REL] = rel;
      c[C_FGP] = rel < eps ? 1.0 : 0.0;
      return;
    }
    case 4: {  // UNDO a speculative iteration's Newton
      for (int i = 0; i < r; ++i) c[C_BETA + i] = c[C_SAVED + i];
      if (c[C_DONE] != 0.0) c[C_TOTAL] -= c[C_LAST];
      return;
    }
  }
}

template <typename T, int R>
void launch_newton(int G, cudaStream_t st, const SlabArgs& A, const T* t, double* out, RedWs ws, bool quad) {
  if constexpr (R > 0) {
    if (quad) newton_kernel4<T, R><<<G, NT, 0, st>>>(A, t, out, ws);
    else newton_kernel<T, R><<<G, NT, 0, st>>>(A, t, out, ws);
  }
}

#define SLAB_RANK_SWITCH(r, BODY)                  \
  switch (r) {                                     \
    case 0: { constexpr int R = 0; BODY; } break;  \
    case 1: { constexpr int R = 1; BODY; } break;  \
    case 2: { constexpr int R = 2; BODY; } break;  \
    case 3: { constexpr int R = 3; BODY; } break;  \
    case 4: { constexpr int R = 4; BODY; } break;  \
    case 5: { constexpr int R = 5; BODY; } break;  \
    case 6: { constexpr int R = 6; BODY; } break;  \
    case 7: { constexpr int R = 7; BODY; } break;  \
    case 8: { constexpr int R = 8; BODY; } break;  \
    default: set_error("rank %d outside [0, 8]", r); return BQ_EINVAL; \
  }

int make_args(const bq_slab_desc* D, const double* c, const double* beta, SlabArgs& A) {
  BQ_CHECK(D && D->K1 >= 1 && D->K2 >= 1 && D->L >= 1, BQ_EINVAL, "bq_slab: bad slab geometry");
  BQ_CHECK(D->rank >= 0 && D->rank <= BQ_MAX_RANK, BQ_EINVAL, "bq_slab: rank %d outside [0, 8]", D->rank);
  BQ_CHECK(D->rank == 0 || D->U, BQ_EINVAL, "bq_slab: U required for rank > 0");
  BQ_CHECK(D->d || D->tau > 0, BQ_EINVAL, "bq_slab: tau must be positive");
  BQ_CHECK(D->sign == 1 || D->sign == -1, BQ_EINVAL, "bq_slab: sign must be +/-1");
  BQ_CHECK(D->dtype == BQ_F32 || D->dtype == BQ_F64, BQ_EINVAL, "bq_slab: bad dtype");
  A = SlabArgs{};
  A.K1 = (int)D->K1;
  A.K2 = (int)D->K2;
  A.L = (int)D->L;
  A.plane = D->K1 * D->K2;
  A.N = A.plane * D->L;
  A.first = D->first;
  A.last = D->last;
  A.rank = D->rank;
  A.sign = D->sign;
  A.iso = D->mode == BQ_TV_ISO;
  A.tau = D->tau;
  A.reg = D->reg;
  A.lo = D->lo;
  A.hi = D->hi;
  A.d = D->d;
  A.U = D->U;
  A.v = D->v;
  A.ctl = D->ctl;
  for (int k = 0; k < D->rank; ++k) {
    A.c[k] = c ? c[k] : 0.0;
    A.beta[k] = beta ? beta[k] : 0.0;
  }
  return BQ_OK;
}

int blocks(bq_ctx* ctx, long long n) {
  long long want = (n + 4LL * NT - 1) / (4LL * NT);
  return (int)std::max<long long>(1, std::min<long long>(want, std::min(1184, ctx->num_sms * 8)));
}
// row-mapped passes (div, dual): one block per x-row step (vox = voxels per thread)
int row_blocks(bq_ctx* ctx, const SlabArgs& A, int vox = 1) {
  const long long per_row = A.K1 / vox;
  const long long rb = per_row >= NT ? 1 : NT / per_row;
  const long long groups = ((long long)A.K2 * A.L + rb - 1) / rb;
  return (int)std::max<long long>(1, std::min<long long>(groups, std::min(1184, ctx->num_sms * 8)));
}

}  // namespace
}  // namespace bq

using namespace bq;

extern "C" int bq_slab_div(bq_ctx* ctx, const bq_slab_desc* desc, const void* field, const void* halo_below,
                           void* t_out, double* s_out, void* stream) {
  SlabArgs A;
  int rc = make_args(desc, nullptr, nullptr, A);
  if (rc) return rc;
  BQ_CHECK(ctx && field && t_out && (A.first || halo_below) && (A.rank == 0 || s_out), BQ_EINVAL,
           "bq_slab_div: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  BQ_STREAM_WS(sw, ctx, st);
  RedWs ws = red_ws(sw);
  const bool quad = quad_ok(A, {field, halo_below, t_out});
  const int G = row_blocks(ctx, A, quad ? 4 : 1);
  if (desc->dtype == BQ_F32) {
    if (quad) {
      SLAB_RANK_SWITCH(A.rank, (div_kernel4<float, R><<<G, NT, 0, st>>>(A, (const float*)field,
                                                                         (const float*)halo_below, (float*)t_out,
                                                                         s_out, ws)));
    } else {
      SLAB_RANK_SWITCH(A.rank, (div_kernel<float, R><<<G, NT, 0, st>>>(A, (const float*)field,
                                                                        (const float*)halo_below, (float*)t_out,
                                                                        s_out, ws)));
    }
  } else {
    if (quad) {
      SLAB_RANK_SWITCH(A.rank, (div_kernel4<double, R><<<G, NT, 0, st>>>(A, (const double*)field,
                                                                          (const double*)halo_below, (double*)t_out,
                                                                          s_out, ws)));
    } else {
      SLAB_RANK_SWITCH(A.rank, (div_kernel<double, R><<<G, NT, 0, st>>>(A, (const double*)field,
                                                                         (const double*)halo_below, (double*)t_out,
                                                                         s_out, ws)));
    }
  }
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_slab_newton(bq_ctx* ctx, const bq_slab_desc* desc, const void* t, const double* c,
                              const double* beta, double* out, void* stream) {
  SlabArgs A;
  int rc = make_args(desc, c, beta, A);
  if (rc) return rc;
  BQ_CHECK(ctx && t && out && A.rank >= 1 && ((c && beta) || A.ctl), BQ_EINVAL, "bq_slab_newton: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  BQ_STREAM_WS(sw, ctx, st);
  RedWs ws = red_ws(sw);
  const bool quad = quad_ok(A, {t});
  const int G = blocks(ctx, quad ? A.N / 4 : A.N);
  if (desc->dtype == BQ_F32) {
    SLAB_RANK_SWITCH(A.rank, (launch_newton<float, R>(G, st, A, (const float*)t, out, ws, quad)));
  } else {
    SLAB_RANK_SWITCH(A.rank, (launch_newton<double, R>(G, st, A, (const double*)t, out, ws, quad)));
  }
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_slab_q(bq_ctx* ctx, const bq_slab_desc* desc, const void* t, const double* c, const double* beta,
                         void* q_out, void* stream) {
  SlabArgs A;
  int rc = make_args(desc, c, beta, A);
  if (rc) return rc;
  BQ_CHECK(ctx && t && q_out && (A.rank == 0 || (c && beta) || A.ctl), BQ_EINVAL, "bq_slab_q: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const bool quad = quad_ok(A, {t, q_out});
  const int G = blocks(ctx, quad ? A.N / 4 : A.N);
  if (desc->dtype == BQ_F32) {
    if (quad) {
      SLAB_RANK_SWITCH(A.rank, (q_kernel4<float, R><<<G, NT, 0, st>>>(A, (const float*)t, (float*)q_out)));
    } else {
      SLAB_RANK_SWITCH(A.rank, (q_kernel<float, R><<<G, NT, 0, st>>>(A, (const float*)t, (float*)q_out)));
    }
  } else {
    if (quad) {
      SLAB_RANK_SWITCH(A.rank, (q_kernel4<double, R><<<G, NT, 0, st>>>(A, (const double*)t, (double*)q_out)));
    } else {
      SLAB_RANK_SWITCH(A.rank, (q_kernel<double, R><<<G, NT, 0, st>>>(A, (const double*)t, (double*)q_out)));
    }
  }
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_slab_dual(bq_ctx* ctx, const bq_slab_desc* desc, const void* pbar, const void* p, const void* q,
                            const void* halo_above, double step, double momentum, void* p_next, void* pbar_next,
                            double* norms_out, void* stream) {
  SlabArgs A;
  int rc = make_args(desc, nullptr, nullptr, A);
  if (rc) return rc;
  BQ_CHECK(ctx && pbar && p && q && p_next && pbar_next && norms_out && (A.last || halo_above), BQ_EINVAL,
           "bq_slab_dual: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  BQ_STREAM_WS(sw, ctx, st);
  RedWs ws = red_ws(sw);
  // (the dual field's 3 components are N apart: N % 4 == 0 with K1 % 4 == 0; f64 needs N even for 16 bytes)
  const bool quad = quad_ok(A, {pbar, p, q, halo_above, p_next, pbar_next});
  const int G = row_blocks(ctx, A, quad ? 4 : 1);
  if (desc->dtype == BQ_F32) {
    if (quad)
      dual_kernel4<float><<<G, NT, 0, st>>>(A, (const float*)pbar, (const float*)p, (const float*)q,
                                            (const float*)halo_above, step, momentum, (float*)p_next,
                                            (float*)pbar_next, norms_out, ws);
    else
      dual_kernel<float><<<G, NT, 0, st>>>(A, (const float*)pbar, (const float*)p, (const float*)q,
                                           (const float*)halo_above, step, momentum, (float*)p_next,
                                           (float*)pbar_next, norms_out, ws);
  } else {
    if (quad)
      dual_kernel4<double><<<G, NT, 0, st>>>(A, (const double*)pbar, (const double*)p, (const double*)q,
                                             (const double*)halo_above, step, momentum, (double*)p_next,
                                             (double*)pbar_next, norms_out, ws);
    else
      dual_kernel<double><<<G, NT, 0, st>>>(A, (const double*)pbar, (const double*)p, (const double*)q,
                                            (const double*)halo_above, step, momentum, (double*)p_next,
                                            (double*)pbar_next, norms_out, ws);
  }
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

extern "C" int bq_slab_ctl(bq_ctx* ctx, const bq_slab_desc* desc, int32_t op, const double* in, double newton_eps,
                           int32_t newton_max_iter, double eps, void* stream) {
  SlabArgs A;
  int rc = make_args(desc, nullptr, nullptr, A);
  if (rc) return rc;
  BQ_CHECK(ctx && A.ctl && op >= 0 && op <= 4 && (in || op == 4), BQ_EINVAL, "bq_slab_ctl: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  slab_ctl_kernel<<<1, 32, 0, st>>>(op, A.rank, A.sign, desc->tau, desc->d == nullptr, in, newton_eps,
                                    newton_max_iter, eps, desc->ctl);
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}
