// ls_fft.cu — pruned, fused padded-Green convolution for the Born/LS views.
//
// Computes exactly what oracle/physics.py Green.apply_full does -- the aperiodic
// convolution of a field on the n^3 domain with the Green kernel K on the
// (2n)^3 padded grid, via K_hat = FFT(K) -- but never materialises the padded
// grid.  The 3-D transform is split into five batched line passes:
//
//   XF  rows  (z<nz_in, y<n)  : x-DFT of the n inputs (zero-padded to m)  -> Hx [z][y<n][x<m]
//   YF  cols  (z<nz_in, x<m)  : y-DFT of the n inputs                      -> Q  [z][y<m][x<m]
//   ZC  cols  (y<m,   x<m)    : z-DFT of the nz_in inputs, * K_hat (or conj), inverse z-DFT,
//                               keep the nz_out output planes (in place)    -> Q
//   YI  cols  (z<nz_out, x<m) : inverse y-DFT, keep y < n                   -> Hx
//   XI  rows  (z<nz_out, y<n) : inverse x-DFT, keep x < n, fused epilogue   -> out
//
// so the zero half of every line is neither read nor transformed, the two
// z-transforms and the spectral multiply share registers, and the padded
// grid's 8N values are only ever touched as the 4N (y,x)-padded planes of Q.
// HBM traffic per view drops from ~130N to ~28N complex words.
// K is even in every axis (offsets i and m-i have the same length), so K_hat
// is read through the folded index min(k, m-k): only its (n+1)^3 octant is
// touched and it stays L2-resident across the views of a batch.
//
// Each line of length m = R1*R2 is a four-step DFT held by C threads:
//   step 1: thread t owns n1 = t + C s; DFT-R2 over n2 of x[n1 + R1 n2] in
//           registers, twiddle w_m^(n1 k2), exchange through shared memory;
//   step 3: thread t owns k2 = t + C s; DFT-R1 over n1 -> X[k2 + R2 k1].
// In ZC the forward result is exactly the register layout the inverse
// (R1' = R2, R2' = R1) needs for its own step 1, so the spectral multiply and
// the inverse's first DFT happen without touching shared memory.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "ls_twiddle.cuh"

namespace bq {
namespace lsfft {

template <typename T>
struct CV;
template <>
struct CV<float> {
  using V = float2;
};
template <>
struct CV<double> {
  using V = double2;
};

template <typename V>
__device__ __forceinline__ V cadd(V a, V b) {
  a.x += b.x;
  a.y += b.y;
  return a;
}
template <typename V>
__device__ __forceinline__ V csub(V a, V b) {
  a.x -= b.x;
  a.y -= b.y;
  return a;
}
template <typename V>
__device__ __forceinline__ V cmul(V a, V b) {
  V r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}

// complex64 on sm_100's packed fp32x2 pipe: an add is one FADD2, a product
// two instructions (FMUL2 of the rotated operand (-a.y, a.x) by b.y -- the
// rotation folds into the operand's swap/negate modifiers -- then FFMA2 by
// b.x), against 2 and 4 scalar instructions.
__device__ __forceinline__ float2 rot90(float2 a) { return make_float2(-a.y, a.x); }  // i a
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return __ffma2_rn(a, make_float2(b.x, b.x), __fmul2_rn(rot90(a), make_float2(b.y, b.y)));
}
// a * (c + i s) for scalar c, s
__device__ __forceinline__ float2 cmul_cs(float2 a, float c, float s) {
  return __ffma2_rn(a, make_float2(c, c), __fmul2_rn(rot90(a), make_float2(s, s)));
}
template <typename V, typename T>
__device__ __forceinline__ V cmul_cs(V a, T c, T s) {
  V r;
  r.x = a.x * c - a.y * s;
  r.y = a.x * s + a.y * c;
  return r;
}
// complex64 held as two scalars (scalar FADD/FMUL/FFMA arithmetic).  ZC used it
// while the packed code's register pairs cost it a resident block (96 registers,
// 12-16% slower); since the next view's column is loaded into the registers
// step 1 frees, ptxas fits the packed ZC into the same 80 / 126 registers and
// it is 1-2.5% faster (LS_ZC_SCALAR selects this form for A/B)
struct __align__(8) F2S {
  float x, y;
};
template <typename T>
struct CVS {
  using V = typename CV<T>::V;
};
template <>
struct CVS<float> {
  using V = F2S;
};

// a * exp(DIR 2 pi i k / 32); k is a compile-time constant after unrolling
template <int DIR, typename V>
__device__ __forceinline__ V tw32(V a, int k) {
  using T = decltype(a.x);
  k &= 31;
  if (k == 0) return a;
  V r;
  if (k == 16) {
    r.x = -a.x;
    r.y = -a.y;
    return r;
  }
  if (k == 8) {  // * (DIR i)
    r.x = DIR > 0 ? -a.y : a.y;
    r.y = DIR > 0 ? a.x : -a.x;
    return r;
  }
  if (k == 24) {  // * (-DIR i)
    r.x = DIR > 0 ? a.y : -a.y;
    r.y = DIR > 0 ? -a.x : a.x;
    return r;
  }
  const T c = (T)cos32(k), s = (T)(DIR > 0 ? sin32(k) : -sin32(k));
  return cmul_cs(a, c, s);
}

template <int R>
__host__ __device__ constexpr int brev(int k) {
  int r = 0;
  for (int b = 1; b < R; b <<= 1) {
    r = (r << 1) | (k & 1);
    k >>= 1;
  }
  return r;
}

// in-register DFT of length R (power of two <= 32), natural order in and out,
// X[k] = sum_n a[n] exp(DIR 2 pi i n k / R)   (radix-2 decimation in frequency)
template <int R, int DIR, typename V>
__device__ __forceinline__ void dft(V (&a)[R]) {
#pragma unroll
  for (int half = R / 2; half >= 1; half >>= 1) {
#pragma unroll
    for (int base = 0; base < R; base += 2 * half) {
#pragma unroll
      for (int j = 0; j < half; ++j) {
        const V u = a[base + j], v = a[base + j + half];
        a[base + j] = cadd(u, v);
        a[base + j + half] = tw32<DIR>(csub(u, v), j * (32 / (2 * half)));
      }
    }
  }
  V t[R];
#pragma unroll
  for (int k = 0; k < R; ++k) t[k] = a[brev<R>(k)];
#pragma unroll
  for (int k = 0; k < R; ++k) a[k] = t[k];
}

// dft with pruning: HIN -- inputs a[R/2 .. R) are zero (the first DIF stage
// is a twiddle only); HOUT -- only the outputs k < R/2 are needed (the last
// stage keeps its even positions, which are the bit-reversed k < R/2).
template <int R, int DIR, bool HIN, bool HOUT, typename V>
__device__ __forceinline__ void dft_p(V (&a)[R]) {
#pragma unroll
  for (int half = R / 2; half >= 1; half >>= 1) {
#pragma unroll
    for (int base = 0; base < R; base += 2 * half) {
#pragma unroll
      for (int j = 0; j < half; ++j) {
        const V u = a[base + j], v = a[base + j + half];
        if (HIN && half == R / 2) {
          a[base + j + half] = tw32<DIR>(u, j * (32 / (2 * half)));
        } else if (HOUT && half == 1) {
          a[base + j] = cadd(u, v);
        } else {
          a[base + j] = cadd(u, v);
          a[base + j + half] = tw32<DIR>(csub(u, v), j * (32 / (2 * half)));
        }
      }
    }
  }
  V t[R];
#pragma unroll
  for (int k = 0; k < (HOUT ? R / 2 : R); ++k) t[k] = a[brev<R>(k)];
#pragma unroll
  for (int k = 0; k < (HOUT ? R / 2 : R); ++k) a[k] = t[k];
}

// shared-memory position of Y[n1][k2] for line l.  COL: lines are adjacent
// columns and l is the fastest index; rows: each line's slab is padded so the
// step-3 reads (stride R1+1) are bank-conflict free.
template <int R1, int R2, int L, bool COL>
__device__ __forceinline__ int spos(int l, int n1, int k2) {
  return COL ? (k2 * R1 + n1) * L + l : l * (R2 * (R1 + 1)) + k2 * (R1 + 1) + n1;
}

template <int R1, int R2, int L, bool COL>
constexpr int smem_elems() {
  return COL ? R1 * R2 * L : L * R2 * (R1 + 1);
}

// step 1: a[s][n2] = x[n1 + R1 n2] (n1 = t + C s) -> smem Y[n1][k2] w_m^(DIR n1 k2)
template <int R1, int R2, int C, int L, bool COL, int DIR, bool HIN = false, typename V>
__device__ __forceinline__ void step1(V (&a)[R1 / C][R2], V* sm, const V* tw, int l, int t) {
  constexpr int M = R1 * R2;
#pragma unroll
  for (int s = 0; s < R1 / C; ++s) {
    dft_p<R2, DIR, HIN, false>(a[s]);
    const int n1 = t + C * s;
#pragma unroll
    for (int k2 = 0; k2 < R2; ++k2) {
      V w = tw[(n1 * k2) & (M - 1)];
      if (DIR > 0) w.y = -w.y;
      sm[spos<R1, R2, L, COL>(l, n1, k2)] = cmul(a[s][k2], w);
    }
  }
}

// step 3: b[s][k1] = X[k2 + R2 k1], k2 = t + C s
template <int R1, int R2, int C, int L, bool COL, int DIR, bool HOUT = false, typename V>
__device__ __forceinline__ void step3(V (&b)[R2 / C][R1], const V* sm, int l, int t) {
#pragma unroll
  for (int s = 0; s < R2 / C; ++s) {
    const int k2 = t + C * s;
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) b[s][n1] = sm[spos<R1, R2, L, COL>(l, n1, k2)];
    dft_p<R1, DIR, false, HOUT>(b[s]);
  }
}

template <typename V, int M>
__device__ __forceinline__ void load_twiddles(V* tw, int tid, int nt) {
  for (int i = tid; i < M; i += nt) {
    const double2 w = g_tw512[i * (512 / M)];
    V v;
    v.x = (decltype(v.x))w.x;
    v.y = (decltype(v.x))w.y;
    tw[i] = v;
  }
}

template <typename V>
__device__ __forceinline__ V czero() {
  V v;
  v.x = 0;
  v.y = 0;
  return v;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// ---------------------------------------------------------------------------
// XF: forward x pass over rows (row = z*n + y, rows = nz_in*n) of the compact
// input (f .* v, or the detector residual plane), zero-padded to m.
// ---------------------------------------------------------------------------
template <typename T, int R1, int R2, int C, int L>
__global__ void __launch_bounds__(C* L) xf_kernel(int n_rt, int rows, const T* __restrict__ f,
                                                  const typename CV<T>::V* __restrict__ v,
                                                  typename CV<T>::V* __restrict__ hx, const int* __restrict__ active) {
  using V = typename CV<T>::V;
  constexpr int M = R1 * R2;
  constexpr int n = M / 2;  // the pruned passes serve n = m/2 only (dispatch on 2n)
  (void)n_rt;
  extern __shared__ __align__(16) unsigned char smraw[];
  V* tw = (V*)smraw;
  V* sm = tw + M;
  const int tid = threadIdx.x, l = tid / C, t = tid % C;
  const int b = blockIdx.x, row = blockIdx.y * L + l;
  if (active && !active[b]) return;  // converged view of a batched solve: nothing to do
  const bool ok = row < rows;
  load_twiddles<V, M>(tw, tid, C * L);
  const V* src = v + ((long long)b * rows + row) * n;
  const T* fr = f ? f + (long long)row * n : nullptr;
  V a[R1 / C][R2];
#pragma unroll
  for (int s = 0; s < R1 / C; ++s)
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) {
      const int e = t + C * s + R1 * n2;
      V x = czero<V>();
      if (ok && e < n) {
        x = src[e];
        if (fr) {
          const T g = fr[e];
          x.x *= g;
          x.y *= g;
        }
      }
      a[s][n2] = x;
    }
  __syncthreads();
  step1<R1, R2, C, L, false, -1, true>(a, sm, tw, l, t);
  __syncthreads();
  V c[R2 / C][R1];
  step3<R1, R2, C, L, false, -1>(c, sm, l, t);
  if (ok) {
    V* dst = hx + ((long long)b * n * n + row) * M;
#pragma unroll
    for (int s = 0; s < R2 / C; ++s)
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) dst[t + C * s + R2 * k1] = c[s][k1];
  }
}

// ---------------------------------------------------------------------------
// YF: forward y pass over columns (z < nz_in, x < m): Hx[z][y<n][x] -> Q[z][y<m][x]
// ---------------------------------------------------------------------------
template <typename T, int R1, int R2, int C, int L>
__global__ void __launch_bounds__(C* L) yf_kernel(int n_rt, const typename CV<T>::V* __restrict__ hx,
                                                  typename CV<T>::V* __restrict__ q, const int* __restrict__ active) {
  if (active && !active[blockIdx.x]) return;
  using V = typename CV<T>::V;
  constexpr int M = R1 * R2, XT = M / L;
  constexpr int n = M / 2;  // the pruned passes serve n = m/2 only (dispatch on 2n)
  (void)n_rt;
  extern __shared__ __align__(16) unsigned char smraw[];
  V* tw = (V*)smraw;
  V* sm = tw + M;
  const int tid = threadIdx.x, l = tid % L, t = tid / L;
  const int b = blockIdx.x, z = blockIdx.y / XT, x = (blockIdx.y % XT) * L + l;
  load_twiddles<V, M>(tw, tid, C * L);
  const V* src = hx + ((long long)b * n + z) * n * M + x;
  V a[R1 / C][R2];
#pragma unroll
  for (int s = 0; s < R1 / C; ++s)
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) {
      const int e = t + C * s + R1 * n2;
      a[s][n2] = e < n ? src[(long long)e * M] : czero<V>();
    }
  __syncthreads();
  step1<R1, R2, C, L, true, -1, true>(a, sm, tw, l, t);
  __syncthreads();
  V c[R2 / C][R1];
  step3<R1, R2, C, L, true, -1>(c, sm, l, t);
  V* dst = q + ((long long)b * n + z) * M * M + x;
#pragma unroll
  for (int s = 0; s < R2 / C; ++s)
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) dst[(long long)(t + C * s + R2 * k1) * M] = c[s][k1];
}

// ---------------------------------------------------------------------------
// ZC: z pass over columns (y < m, x < m), in place in Q:
//   forward z-DFT of planes [z0, z0+nzi), * K_hat (conj if adj),
//   inverse z-DFT, keep planes [zo0, zo0+nzo) -> Q slots 0..nzo-1.
// One block owns one (y, x-chunk) column group and walks the B views of the
// batch: the twiddles and the block's K_hat columns (folded z index, n+1
// values per line) are staged into shared memory once (cp.async, overlapping
// the first view's loads and forward DFT) and reused by every view, and the
// next active view's column is prefetched into L2 while this one computes.
// ---------------------------------------------------------------------------
#ifndef LS_ZC_PF
#define LS_ZC_PF 512  // ZC: prefetch the next view's column into L2 for m >= LS_ZC_PF (helps at 512, not 256)
#endif

#ifndef LS_ZC_MINB
#define LS_ZC_MINB 3  // ZC at m <= 256: minimum resident blocks per SM requested from ptxas (register cap; 2 at m = 512)
#endif
#ifndef LS_ZC_RPF
#define LS_ZC_RPF 1  // ZC at m <= 256: register prefetch of the next view's column (A/B hook)
#endif
#ifndef LS_ZC_RPF_MAXM
#define LS_ZC_RPF_MAXM 256
#endif
#ifndef LS_LR512
#define LS_LR512 8  // rows per block of the row passes at m = 512 (views_ls.cu bg_conv_blocks must agree)
#endif
#ifndef LS_ZC_VG
#define LS_ZC_VG 1  // ZC view groups per column group (grid.y); measured: 2 and 4 are no faster at m = 256 / 512
#endif
template <int R1, int R2, int L>
constexpr int zc_smem_elems(int n) {
  return R1 * R2 + R1 * R2 * L + (n + 1) * L;
}

// STD: the volume-to-volume case (z0 = zo0 = 0, nzi = nzo = n = m/2): the
// zero half of the input and the dropped half of the output are compile-time
// (no bounds tests, pruned first forward / last inverse DFT stages).
template <typename T, int R1, int R2, int C, int L, bool STD>
__global__ void __launch_bounds__(C* L, (R1 * R2 <= 256 ? LS_ZC_MINB : 2)) zc_kernel(int n, int B, int z0, int nzi, int zo0, int nzo, int adj,
                                                  const typename CV<T>::V* __restrict__ khat,
                                                  typename CV<T>::V* __restrict__ q_, const int* __restrict__ active) {
#ifdef LS_ZC_SCALAR  // A/B hook: scalar complex arithmetic (F2S), the form ZC had before the register prefetch
  using V = typename CVS<T>::V;
#else
  using V = typename CV<T>::V;
#endif
  V* __restrict__ q = reinterpret_cast<V*>(q_);
  constexpr int M = R1 * R2, XT = M / L, NT = C * L;
  extern __shared__ __align__(16) unsigned char smraw[];
  V* tw = (V*)smraw;
  V* sm = tw + M;
  V* ks = sm + M * L;  // [fz <= n][l]: K_hat of this block's columns, folded z
  const int tid = threadIdx.x, l = tid % L, t = tid / L;
  const int y = blockIdx.x / XT, xc = blockIdx.x % XT, x = xc * L + l;
  const long long zs = (long long)M * M;
  const long long vstride = (long long)n * zs;  // one view's Q
  const int fy = y <= n ? y : M - y;
  {
    const V* kb = reinterpret_cast<const V*>(khat) + (long long)fy * M;
    const int nk = (n + 1) * L;
    for (int i = tid; i < nk; i += NT) {
      const int fz = i / L, xx = xc * L + i % L;
      const int fx = xx <= n ? xx : M - xx;
      if (sizeof(V) == 8) cp_async8(&ks[i], kb + fz * zs + fx);
      else cp_async16(&ks[i], kb + fz * zs + fx);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  load_twiddles<V, M>(tw, tid, NT);
  // blockIdx.y: view group -- the block walks views [b_lo, b_hi) of the batch
  const int b_lo = (int)(((long long)B * blockIdx.y) / gridDim.y);
  const int b_hi = (int)(((long long)B * (blockIdx.y + 1)) / gridDim.y);
  B = b_hi;
  auto next_active = [&](int b) {
    while (b < B && active && !active[b]) ++b;
    return b;
  };
  bool first = true;
  constexpr int ZS = M * M;  // plane stride (32-bit offsets within one view's Q)
  // RPF: the next active view's column is loaded into the registers of `a` as
  // soon as step 1 has consumed them, so its DRAM latency runs under this
  // view's transforms (volume-to-volume case, one line segment per thread)
  constexpr bool RPF = LS_ZC_RPF && STD && M <= LS_ZC_RPF_MAXM;
  V a[R1 / C][R2];
  auto load_col = [&](const V* col) {
#pragma unroll
    for (int s = 0; s < R1 / C; ++s)
#pragma unroll
      for (int n2 = 0; n2 < R2; ++n2) {
        const int e = t + C * s + R1 * n2;
        if (STD) a[s][n2] = n2 < R2 / 2 ? col[e * ZS] : czero<V>();
        else a[s][n2] = (e >= z0 && e < z0 + nzi) ? col[(e - z0) * zs] : czero<V>();
      }
  };
  int b = next_active(b_lo);
  if (RPF && b < B) load_col(q + (long long)b * vstride + (long long)y * M + x);
  for (; b < B;) {
    V* col = q + (long long)b * vstride + (long long)y * M + x;
    const int bn = next_active(b + 1);
    if (!RPF) load_col(col);
    // the next active view's column into L2 while this one computes
    if (M >= LS_ZC_PF && bn < B) {
      const V* nc = q + (long long)bn * vstride + (long long)y * M + x;
      for (int e = t; e < nzi; e += C) prefetch_l2(nc + e * zs);
    }
    if (first) cp_async_wait_all();
    __syncthreads();  // twiddles + K_hat staged (first view); previous view's reads of sm done
    step1<R1, R2, C, L, true, -1, STD>(a, sm, tw, l, t);
    if (RPF && bn < B) load_col(q + (long long)bn * vstride + (long long)y * M + x);
    __syncthreads();
    V c[R2 / C][R1];
    step3<R1, R2, C, L, true, -1>(c, sm, l, t);
    // spectral multiply: c[s][k1] = X[kz], kz = k2 + R2 k1, k2 = t + C s.
    // Folded index (n = M/2 here): kz <= n exactly when k1 < R1/2 or kz == n,
    // and M - kz == n at kz == n, so fz = k1 < R1/2 ? kz : M - kz -- a
    // compile-time choice per unrolled k1 (immediate offsets from two bases);
    // adj is block-uniform, so it selects a whole loop
    auto kmul = [&](auto conj) {
#pragma unroll
      for (int s = 0; s < R2 / C; ++s) {
        const int k2 = t + C * s;
        const V* kp = ks + k2 * L + l;            // k1 <  R1/2: fz = k2 + R2 k1
        const V* km = ks + (M - k2) * L + l;      // k1 >= R1/2: fz = M - k2 - R2 k1
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) {
          V k = k1 < R1 / 2 ? kp[R2 * k1 * L] : km[-R2 * k1 * L];
          if (decltype(conj)::value) k.y = -k.y;
          c[s][k1] = cmul(c[s][k1], k);
        }
      }
    };
    if (adj) kmul(std::true_type{});
    else kmul(std::false_type{});
    __syncthreads();  // step-3 reads of sm are done before it is rewritten
    // inverse with (R1', R2') = (R2, R1): c[s][n2'] = x'[n1' + R2 n2'], n1' = t + C s
    step1<R2, R1, C, L, true, 1>(c, sm, tw, l, t);
    __syncthreads();
    V o[R1 / C][R2];
    step3<R2, R1, C, L, true, 1, STD>(o, sm, l, t);
#pragma unroll
    for (int s = 0; s < R1 / C; ++s)
#pragma unroll
      for (int k1 = 0; k1 < R2; ++k1) {
        const int z = t + C * s + R1 * k1;
        if (STD) {
          if (k1 < R2 / 2) col[z * ZS] = o[s][k1];
        } else if (z >= zo0 && z < zo0 + nzo) {
          col[(z - zo0) * zs] = o[s][k1];
        }
      }
    first = false;
    b = bn;
  }
  if (first) cp_async_wait_all();  // no active view: retire the staging copies
}

// ---------------------------------------------------------------------------
// YI: inverse y pass over columns (z < nz_out, x < m): Q[z][y<m][x] -> Hx[z][y<n][x]
// ---------------------------------------------------------------------------
template <typename T, int R1, int R2, int C, int L>
__global__ void __launch_bounds__(C* L) yi_kernel(int n_rt, const typename CV<T>::V* __restrict__ q,
                                                  typename CV<T>::V* __restrict__ hx, const int* __restrict__ active) {
  if (active && !active[blockIdx.x]) return;
  using V = typename CV<T>::V;
  constexpr int M = R1 * R2, XT = M / L;
  constexpr int n = M / 2;  // the pruned passes serve n = m/2 only (dispatch on 2n)
  (void)n_rt;
  extern __shared__ __align__(16) unsigned char smraw[];
  V* tw = (V*)smraw;
  V* sm = tw + M;
  const int tid = threadIdx.x, l = tid % L, t = tid / L;
  const int b = blockIdx.x, z = blockIdx.y / XT, x = (blockIdx.y % XT) * L + l;
  load_twiddles<V, M>(tw, tid, C * L);
  const V* src = q + ((long long)b * n + z) * M * M + x;
  V a[R1 / C][R2];
#pragma unroll
  for (int s = 0; s < R1 / C; ++s)
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) a[s][n2] = src[(long long)(t + C * s + R1 * n2) * M];
  __syncthreads();
  step1<R1, R2, C, L, true, 1>(a, sm, tw, l, t);
  __syncthreads();
  V c[R2 / C][R1];
  step3<R1, R2, C, L, true, 1, true>(c, sm, l, t);
  V* dst = hx + ((long long)b * n + z) * n * M + x;
#pragma unroll
  for (int s = 0; s < R2 / C; ++s)
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      const int k = t + C * s + R2 * k1;
      if (k < n) dst[(long long)k * M] = c[s][k1];
    }
}

// ---------------------------------------------------------------------------
// XI: inverse x pass over rows (rows = nz_out*n), keep x < n, fused epilogue
// (views_ls.cu crop_kernel / det_kernel semantics):
//   out = beta * scale * (fconj .* G) + alpha * v + addend
// ---------------------------------------------------------------------------
template <typename T, int R1, int R2, int C, int L>
__global__ void __launch_bounds__(C* L) xi_kernel(int n_rt, int rows, const typename CV<T>::V* __restrict__ hx,
                                                  double scale, const T* __restrict__ fconj,
                                                  const typename CV<T>::V* __restrict__ v, double alpha, double beta,
                                                  const typename CV<T>::V* __restrict__ addend,
                                                  typename CV<T>::V* __restrict__ out, const int* __restrict__ active,
                                                  const typename CV<T>::V* __restrict__ da, double* __restrict__ dotp) {
  using V = typename CV<T>::V;
  constexpr int M = R1 * R2;
  constexpr int n = M / 2;  // the pruned passes serve n = m/2 only (dispatch on 2n)
  (void)n_rt;
  extern __shared__ __align__(16) unsigned char smraw[];
  V* tw = (V*)smraw;
  V* sm = tw + M;
  const int tid = threadIdx.x, l = tid / C, t = tid % C;
  const int b = blockIdx.x, row = blockIdx.y * L + l;
  if (active && !active[b]) return;
  const bool ok = row < rows;
  load_twiddles<V, M>(tw, tid, C * L);
  const V* src = hx + ((long long)b * n * n + (ok ? row : 0)) * M;
  V a[R1 / C][R2];
#pragma unroll
  for (int s = 0; s < R1 / C; ++s)
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) a[s][n2] = ok ? src[t + C * s + R1 * n2] : czero<V>();
  if (ok) {  // the epilogue's inputs into L2 while the transform runs
    constexpr int LINE = 128 / sizeof(V);
    const long long ob = ((long long)b * rows + row) * n;
    for (int e = t * LINE; e < n; e += C * LINE) {
      if (v && alpha != 0.0) prefetch_l2(v + ob + e);
      if (addend) prefetch_l2(addend + ob + e);
      if (dotp) prefetch_l2(da + ob + e);
    }
  }
  __syncthreads();
  step1<R1, R2, C, L, false, 1>(a, sm, tw, l, t);
  __syncthreads();
  V c[R2 / C][R1];
  step3<R1, R2, C, L, false, 1, true>(c, sm, l, t);
  // fused per-view dot partials of the result: (sum conj(da) out, sum |out|^2)
  double dre = 0.0, dim = 0.0, dnn = 0.0;
  if (ok) {
    const long long ob = ((long long)b * rows + row) * n;
    const long long fb = (long long)row * n;
    const bool use_v = v && alpha != 0.0;
#pragma unroll
    for (int s = 0; s < R2 / C; ++s)
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) {
        const int k = t + C * s + R2 * k1;
        if (k < n) {
          V p = c[s][k1];
          p.x *= (T)scale;
          p.y *= (T)scale;
          if (fconj) {
            const T g = fconj[fb + k];
            p.x *= g;
            p.y *= g;
          }
          V r;
          r.x = (T)beta * p.x;
          r.y = (T)beta * p.y;
          if (use_v) {
            const V vv = v[ob + k];
            r.x += (T)alpha * vv.x;
            r.y += (T)alpha * vv.y;
          }
          if (addend) {
            const V ad = addend[ob + k];
            r.x += ad.x;
            r.y += ad.y;
          }
          out[ob + k] = r;
          if (dotp) {
            const V a = da[ob + k];
            dre += (double)a.x * r.x + (double)a.y * r.y;
            dim += (double)a.x * r.y - (double)a.y * r.x;
            dnn += (double)r.x * r.x + (double)r.y * r.y;
          }
        }
      }
  }
  if (dotp) {  // fixed-order block reduction (deterministic)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dre += __shfl_down_sync(0xffffffffu, dre, o);
      dim += __shfl_down_sync(0xffffffffu, dim, o);
      dnn += __shfl_down_sync(0xffffffffu, dnn, o);
    }
    __shared__ double red[3][32];
    const int lane = tid & 31, w = tid >> 5;
    if (lane == 0) red[0][w] = dre, red[1][w] = dim, red[2][w] = dnn;
    __syncthreads();
    if (tid == 0) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      for (int q = 0; q < (C * L) / 32; ++q) a0 += red[0][q], a1 += red[1][q], a2 += red[2][q];
      double* dp = dotp + ((long long)b * gridDim.y + blockIdx.y) * 3;
      dp[0] = a0;
      dp[1] = a1;
      dp[2] = a2;
    }
  }
}

template <typename K>
int prep(K kernel, size_t smem) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      set_error("ls_fft: cudaFuncSetAttribute(%zu B) failed: %s", smem, cudaGetErrorString(e));
      return BQ_ECUDA;
    }
  }
  return BQ_OK;
}

template <typename T, int R1, int R2, int C>
int run(int n, int B, int op, const void* khat, const void* f, const void* v, double alpha, double beta,
        const void* addend, void* scratch, void* out, const int* active, const void* da, double* dotp, int* nblk,
        cudaStream_t st) {
  using V = typename CV<T>::V;
  constexpr int M = R1 * R2;
  constexpr int L = (256 / C) < M ? (256 / C) : M;
  constexpr int NT = C * L;
  // row passes (XF, XI): rows per block.  Rows are contiguous whatever LR is, and
  // at m = 512 a 16-row block's exchange buffer (68 KB) allows 3 blocks per SM:
  // 8-row blocks (36 KB, 6 per SM) overlap their load / transform / store phases better
  constexpr int LR = M == 512 ? LS_LR512 : L;
  constexpr int NTR = C * LR;
  const size_t sm_row = sizeof(V) * (M + smem_elems<R1, R2, LR, false>());
  const size_t sm_col = sizeof(V) * (M + smem_elems<R1, R2, L, true>());
  const size_t sm_zc = sizeof(V) * zc_smem_elems<R1, R2, L>(n);
  const long long N = (long long)n * n * n;
  V* q = (V*)scratch;                 // B x n x m x m
  V* hx = q + (long long)B * 4 * N;   // B x n x n x m
  const int nzi = op == 3 ? 1 : n, z0 = op == 3 ? n : 0;
  const int nzo = op == 2 ? 1 : n, zo0 = op == 2 ? n : 0;
  const bool adj = op == 1 || op == 3;
  int rc;
  if ((rc = prep(xf_kernel<T, R1, R2, C, LR>, sm_row)) || (rc = prep(yf_kernel<T, R1, R2, C, L>, sm_col)) ||
      (rc = prep(zc_kernel<T, R1, R2, C, L, true>, sm_zc)) || (rc = prep(zc_kernel<T, R1, R2, C, L, false>, sm_zc)) || (rc = prep(yi_kernel<T, R1, R2, C, L>, sm_col)) ||
      (rc = prep(xi_kernel<T, R1, R2, C, LR>, sm_row)))
    return rc;
  const int rows_in = nzi * n, rows_out = nzo * n;
  xf_kernel<T, R1, R2, C, LR><<<dim3(B, (rows_in + LR - 1) / LR), NTR, sm_row, st>>>(
      n, rows_in, (op == 0 || op == 2) ? (const T*)f : nullptr, (const V*)v, hx, active);
  yf_kernel<T, R1, R2, C, L><<<dim3(B, nzi * (M / L)), NT, sm_col, st>>>(n, hx, q, active);
  const int zvg = B < LS_ZC_VG ? (B > 0 ? B : 1) : LS_ZC_VG;
  if (nzi == n && nzo == n && z0 == 0 && zo0 == 0)
    zc_kernel<T, R1, R2, C, L, true><<<dim3(M * (M / L), zvg), NT, sm_zc, st>>>(n, B, z0, nzi, zo0, nzo, adj ? 1 : 0,
                                                                        (const V*)khat, q, active);
  else
    zc_kernel<T, R1, R2, C, L, false><<<dim3(M * (M / L), zvg), NT, sm_zc, st>>>(n, B, z0, nzi, zo0, nzo, adj ? 1 : 0,
                                                                         (const V*)khat, q, active);
  yi_kernel<T, R1, R2, C, L><<<dim3(B, nzo * (M / L)), NT, sm_col, st>>>(n, q, hx, active);
  if (nblk) *nblk = (rows_out + LR - 1) / LR;
  const bool crop = op != 2;
  xi_kernel<T, R1, R2, C, LR><<<dim3(B, (rows_out + LR - 1) / LR), NTR, sm_row, st>>>(
      n, rows_out, hx, 1.0 / (8.0 * (double)N), op == 1 ? (const T*)f : nullptr,
      (crop && op != 3) ? (const V*)v : nullptr, (crop && op != 3) ? alpha : 0.0, crop && op != 3 ? beta : 1.0,
      crop ? (const V*)addend : nullptr, (V*)out, active, (const V*)da, dotp);
  BQ_CUDA(cudaGetLastError());
  return BQ_OK;
}

template <typename T>
int dispatch(int n, int B, int op, const void* khat, const void* f, const void* v, double alpha, double beta,
             const void* addend, void* scratch, void* out, const int* active, const void* da, double* dotp,
             int* nblk, cudaStream_t st) {
  switch (2 * n) {
    case 16: return run<T, 4, 4, 4>(n, B, op, khat, f, v, alpha, beta, addend, scratch, out, active, da, dotp, nblk, st);
    case 32: return run<T, 8, 4, 4>(n, B, op, khat, f, v, alpha, beta, addend, scratch, out, active, da, dotp, nblk, st);
    case 64: return run<T, 8, 8, 8>(n, B, op, khat, f, v, alpha, beta, addend, scratch, out, active, da, dotp, nblk, st);
    case 128: return run<T, 16, 8, 8>(n, B, op, khat, f, v, alpha, beta, addend, scratch, out, active, da, dotp, nblk, st);
    case 256: return run<T, 16, 16, 16>(n, B, op, khat, f, v, alpha, beta, addend, scratch, out, active, da, dotp, nblk, st);
    case 512: return run<T, 32, 16, 16>(n, B, op, khat, f, v, alpha, beta, addend, scratch, out, active, da, dotp, nblk, st);
    default: return 1;  // not handled: the caller uses the cuFFT path
  }
}

}  // namespace lsfft

// Returns 1 when (n) has no pruned-pass instantiation (or BQ_LS_CUFFT=1 forces
// the cuFFT path); otherwise a BQ status.  Scratch: 6N complex per view.
int ls_conv_pruned(bq_ctx* ctx, int dtype, int n, int B, int op, const void* khat, const void* f, const void* v,
                   double alpha, double beta, const void* addend, void* scratch, void* out, cudaStream_t st,
                   const int* active, const void* da, double* dotp, int* nblk) {
  (void)ctx;
  static const bool force_cufft = [] {
    const char* e = std::getenv("BQ_LS_CUFFT");
    return e && e[0] == '1';
  }();
  if (force_cufft) return 1;
  return dtype == BQ_F32
             ? lsfft::dispatch<float>(n, B, op, khat, f, v, alpha, beta, addend, scratch, out, active, da, dotp, nblk, st)
             : lsfft::dispatch<double>(n, B, op, khat, f, v, alpha, beta, addend, scratch, out, active, da, dotp, nblk, st);
}

}  // namespace bq
