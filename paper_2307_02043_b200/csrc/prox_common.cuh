// prox_common.cuh — device helpers shared by the prox kernels.
#pragma once

#include "common.cuh"

namespace bq {
namespace prox {

template <typename T>
__device__ __forceinline__ T clampv(T z, T lo, T hi) {
  return fmin(fmax(z, lo), hi);  // np.clip == minimum(maximum(z, lo), hi)
}

// Reciprocal: correctly rounded MUFU-based sequence in f32 (no IEEE division
// subroutine on the hot path); exact division in f64.
__device__ __forceinline__ float rcp(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double rcp(double x) { return 1.0 / x; }

// Isotropic dual-ball projection p / max(||p||, 1) (tv_ops.py:177-179).
// f32: branch-free, s = min(1/sqrt(ss), 1) is 1 exactly when ss <= 1 (also
// for ss == 0 or a denormal ss, whose ftz reciprocal root is +inf).
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ball_scale(float ss) { return fminf(rsqrt_ftz(ss), 1.0f); }
__device__ __forceinline__ void ball(float (&w)[3], float ss) {
  const float s = ball_scale(ss);
  w[0] *= s, w[1] *= s, w[2] *= s;
}
__device__ __forceinline__ void ball(double (&w)[3], double ss) {
  const double den = fmax(sqrt(ss), 1.0);
  w[0] /= den, w[1] /= den, w[2] /= den;
}

// 4 consecutive elements; 16-byte vector accesses (f32) / 2 x 16 (f64).
// ro: read-only for the kernel's lifetime (non-coherent path); rw: plain.
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

// ---- voxel pairs: sm_100 packed fp32x2 arithmetic (FADD2/FMUL2/FFMA2) ----
// One instruction serves two adjacent voxels in f32 (the x-vector of a lane
// is held as two pairs); f64 pairs are two scalar operations.  Negation and
// |x| of an operand fold into the packed instruction's operand modifiers.
template <typename T>
struct Pair;
template <>
struct Pair<float> {
  using t = float2;
};
template <>
struct Pair<double> {
  using t = double2;
};
template <typename T>
using pair_t = typename Pair<T>::t;

__device__ __forceinline__ float2 mk2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ double2 mk2(double a, double b) { return make_double2(a, b); }
__device__ __forceinline__ float2 bc2(float a) { return make_float2(a, a); }
__device__ __forceinline__ double2 bc2(double a) { return make_double2(a, a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 abs2(float2 a) { return make_float2(fabsf(a.x), fabsf(a.y)); }
__device__ __forceinline__ double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sub2(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul2(double2 a, double2 b) { return make_double2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ double2 fma2(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y));
}
__device__ __forceinline__ double2 abs2(double2 a) { return make_double2(fabs(a.x), fabs(a.y)); }
// element e (compile-time under unrolling) of a 2-pair x-vector
template <typename P>
__device__ __forceinline__ auto& el(P (&a)[2], int e) {
  return (e & 1) ? a[e >> 1].y : a[e >> 1].x;
}
template <typename P>
__device__ __forceinline__ const auto& el(const P (&a)[2], int e) {
  return (e & 1) ? a[e >> 1].y : a[e >> 1].x;
}
// 4 consecutive elements as two pairs (16-byte f32 / 2 x 16-byte f64 accesses)
__device__ __forceinline__ void ld2(const float* p, float2 (&o)[2]) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  o[0] = make_float2(v.x, v.y), o[1] = make_float2(v.z, v.w);
}
__device__ __forceinline__ void ld2(const double* p, double2 (&o)[2]) {
  o[0] = reinterpret_cast<const double2*>(p)[0];
  o[1] = reinterpret_cast<const double2*>(p)[1];
}
// read-only for the kernel's lifetime (non-coherent path)
__device__ __forceinline__ void ld2ro(const float* p, float2 (&o)[2]) {
  const float4 v = __ldg(reinterpret_cast<const float4*>(p));
  o[0] = make_float2(v.x, v.y), o[1] = make_float2(v.z, v.w);
}
__device__ __forceinline__ void ld2ro(const double* p, double2 (&o)[2]) {
  o[0] = __ldg(reinterpret_cast<const double2*>(p));
  o[1] = __ldg(reinterpret_cast<const double2*>(p) + 1);
}
__device__ __forceinline__ void st2(float* p, const float2 (&o)[2]) {
  *reinterpret_cast<float4*>(p) = make_float4(o[0].x, o[0].y, o[1].x, o[1].y);
}
__device__ __forceinline__ void st2(double* p, const double2 (&o)[2]) {
  reinterpret_cast<double2*>(p)[0] = o[0];
  reinterpret_cast<double2*>(p)[1] = o[1];
}
// pass accumulators: a pair (packed multiply-add, folded at flush time) or a
// scalar that takes both products of the pair at once (x first, then y)
__device__ __forceinline__ void accf(float2& a, float2 x, float2 y) { a = fma2(x, y, a); }
__device__ __forceinline__ void accf(double2& a, double2 x, double2 y) { a = fma2(x, y, a); }
__device__ __forceinline__ void accf(float& a, float2 x, float2 y) { a = fmaf(x.y, y.y, fmaf(x.x, y.x, a)); }
__device__ __forceinline__ void accf(double& a, double2 x, double2 y) { a = fma(x.y, y.y, fma(x.x, y.x, a)); }
__device__ __forceinline__ void acc_zero(float2& a) { a = make_float2(0.f, 0.f); }
__device__ __forceinline__ void acc_zero(double2& a) { a = make_double2(0.0, 0.0); }
__device__ __forceinline__ void acc_zero(float& a) { a = 0.f; }
__device__ __forceinline__ void acc_zero(double& a) { a = 0.0; }
__device__ __forceinline__ double acc_fold(float2 a) { return (double)a.x + (double)a.y; }
__device__ __forceinline__ double acc_fold(double2 a) { return a.x + a.y; }
__device__ __forceinline__ double acc_fold(float a) { return (double)a; }
__device__ __forceinline__ double acc_fold(double a) { return a; }

// dual-ball projection of two voxels' (w0, w1, w2) given ss = ||w||^2 per voxel
__device__ __forceinline__ void ball2(float2 (&w)[3], float2 ss) {
  const float2 s = make_float2(ball_scale(ss.x), ball_scale(ss.y));
  w[0] = mul2(w[0], s), w[1] = mul2(w[1], s), w[2] = mul2(w[2], s);
}
__device__ __forceinline__ void ball2(double2 (&w)[3], double2 ss) {
  const double dx = fmax(sqrt(ss.x), 1.0), dy = fmax(sqrt(ss.y), 1.0);
#pragma unroll
  for (int n = 0; n < 3; ++n) w[n].x /= dx, w[n].y /= dy;
}

// ---- small dense linear algebra for the controller (r <= 8), unrolled ----
// cap/H are symmetric; packed lower index k(i, j) = i (i + 1) / 2 + j, j <= i.
template <int R>
__device__ __forceinline__ bool chol(double (&a)[R > 0 ? R * R : 1]) {
#pragma unroll
  for (int j = 0; j < R; ++j) {
    double s = a[j * R + j];
#pragma unroll
    for (int k = 0; k < j; ++k) s -= a[j * R + k] * a[j * R + k];
    if (!(s > 0.0)) return false;
    const double l = sqrt(s);
    a[j * R + j] = l;
#pragma unroll
    for (int i = j + 1; i < R; ++i) {
      double t = a[i * R + j];
#pragma unroll
      for (int k = 0; k < j; ++k) t -= a[i * R + k] * a[j * R + k];
      a[i * R + j] = t / l;
    }
  }
  return true;
}
// chol_solve with the reciprocal diagonal precomputed (multiplies, no divisions)
template <int R>
__device__ __forceinline__ void chol_solve_rd(const double* l, const double* rd, double (&b)[R > 0 ? R : 1]) {
#pragma unroll
  for (int i = 0; i < R; ++i) {
    double s = b[i];
#pragma unroll
    for (int k = 0; k < i; ++k) s -= l[i * R + k] * b[k];
    b[i] = s * rd[i];
  }
#pragma unroll
  for (int i = R - 1; i >= 0; --i) {
    double s = b[i];
#pragma unroll
    for (int k = i + 1; k < R; ++k) s -= l[k * R + i] * b[k];
    b[i] = s * rd[i];
  }
}
template <int R>
__device__ __forceinline__ void chol_solve(const double* l, double (&b)[R > 0 ? R : 1]) {
#pragma unroll
  for (int i = 0; i < R; ++i) {
    double s = b[i];
#pragma unroll
    for (int k = 0; k < i; ++k) s -= l[i * R + k] * b[k];
    b[i] = s / l[i * R + i];
  }
#pragma unroll
  for (int i = R - 1; i >= 0; --i) {
    double s = b[i];
#pragma unroll
    for (int k = i + 1; k < R; ++k) s -= l[k * R + i] * b[k];
    b[i] = s / l[i * R + i];
  }
}
// LU with partial pivoting (numpy.linalg.solve / LAPACK gesv); false on an
// exactly-zero pivot (LinAlgError in the reference).
template <int R>
__device__ __forceinline__ bool lu(double (&a)[R > 0 ? R * R : 1], double (&b)[R > 0 ? R : 1]) {
#pragma unroll
  for (int k = 0; k < R; ++k) {
    int piv = k;
    double best = fabs(a[k * R + k]);
#pragma unroll
    for (int i = k + 1; i < R; ++i)
      if (fabs(a[i * R + k]) > best) best = fabs(a[i * R + k]), piv = i;
    if (best == 0.0) return false;
    if (piv != k) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double t = a[k * R + j];
        a[k * R + j] = a[piv * R + j];
        a[piv * R + j] = t;
      }
      const double t = b[k];
      b[k] = b[piv];
      b[piv] = t;
    }
#pragma unroll
    for (int i = k + 1; i < R; ++i) {
      const double f = a[i * R + k] / a[k * R + k];
#pragma unroll
      for (int j = k; j < R; ++j) a[i * R + j] -= f * a[k * R + j];
      b[i] -= f * b[k];
    }
  }
#pragma unroll
  for (int i = R - 1; i >= 0; --i) {
    double s = b[i];
#pragma unroll
    for (int j = i + 1; j < R; ++j) s -= a[i * R + j] * b[j];
    b[i] = s / a[i * R + i];
  }
  return true;
}

// ---- device-wide barrier primitives (release/acquire, no SC fences) -------
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

}  // namespace prox
}  // namespace bq

namespace bq {
namespace prox {
// ---- bulk async copy (TMA engine) + mbarrier, raw PTX for sm_100a ---------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy, completion counted on `bar` (bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// order earlier generic-proxy accesses before later async-proxy ones
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// named barrier over a subset of the block's warps (ids 1..15; 0 = __syncthreads)
__device__ __forceinline__ void named_sync(unsigned id, unsigned nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
}  // namespace prox
}  // namespace bq
