// wtv_fused_impl.cuh — the fast path of bq_wtv_prox: ONE persistent cooperative
// kernel in which every FGP iteration is ONE fused streaming pass plus ONE
// device-wide barrier.
//
// Reference algorithm (paths under /root/reference/pkg/src/tvqn/):
//   dual_tv_solver.py:161-250  FGP loop: P_next = Proj(P_bar + step D q), FISTA momentum,
//                              rel-change stop, final prox at P
//   dual_tv_solver.py:119-135  w(P) = v - reg W^-1 div(P), q = wpm_box(w(P))
//   tv_ops.py:107-180          stencils, divergence, dual-ball projection
//   wpm.py:92-106, 145-253     Woodbury inverse, structured WPM semi-smooth Newton
// with W = diag(d) + sign U U^T (d == NULL -> tau I, the reference metric).
//
// How one FGP iteration i maps onto the machine:
//  * P lives in a 3-slot ring (p_i, p_{i-1}, p_{i-2}); the momentum field
//    P_bar_{i-1} = p_{i-1} + m (p_{i-1} - p_{i-2}) is formed on the fly (the
//    reference's stored P_bar, same arithmetic).  `a` ping-pongs between two
//    buffers.  Nothing read in a pass is written in that pass, so halos can be
//    recomputed by any block without races.
//  * FUSED pass (z-march, 4 voxels per lane via 16-byte accesses, one warp per
//    x-row of K1 <= 128 voxels): q = clamp(a_{i-1} + s.gamma) evaluated on the
//    fly, p_i = Proj(P_bar_{i-1} + step D q), P_bar_i formed in registers,
//    a_i = v - reg D^-1 div(P_bar_i): the x-1 neighbour comes by shuffle, the
//    z-1 neighbour is carried in registers, the y-1 neighbour through shared
//    memory (one extra "halo" warp recomputes the row above the block tile).
//    The same pass accumulates ||p_i - p_{i-1}||^2, ||p_{i-1}||^2,
//    U^T D^-1 div (Woodbury right-hand side) and the Newton aggregates below.
//  * Semi-smooth Newton without passes: for a predicted box of the shift
//    gamma = gw - beta, each voxel is classified as always-inside,
//    always-clamped or "near" (clamp state may change in the box).  The pass
//    reduces K0 = sum_out u (a - bound) + sum_near u a, Cin = sum_in u s^T,
//    Cout = sum_out u s^T and compacts near-voxel indices per warp.  Then
//    phi(beta) = K0 + Cout gw + Cin beta + beta - sum_near u clamp(a + s.gamma)
//    and H = I + Cin + sum_near,inside u s^T are exact for every gamma in the
//    box, so every block evaluates the Newton steps redundantly over the short
//    near list: no full pass, no barrier.  If gamma leaves the box or the list
//    overflows, the step falls back to the full-pass Newton of the reference.
//  * Barriers: release/acquire atomics; the last block reduces the per-block
//    partials in block order (deterministic) and publishes them; every block
//    runs the controller on its own shared-memory copy of the state.
#pragma once
#include <stdlib.h>

#ifndef BQ_PROX_TRACE
#define BQ_PROX_TRACE 0  // device timeline hooks (bench/micro/trace_*.py); build with -DBQ_PROX_TRACE=1
#endif
// inter-pass timeline of block 0, thread 0 (BQ_PROX_TRACE_THREAD=-3): stamp i of iteration trace_pass
#if BQ_PROX_TRACE
#define TR3(i) do { if (blockIdx.x == 0 && threadIdx.x == 0 && tr3_on) A.trace[320 + (i)] = global_ns(); } while (0)
#else
#define TR3(i) do { } while (0)
#endif

#include <algorithm>
#include <type_traits>

#include <cooperative_groups.h>

#include "prox_common.cuh"

namespace bq {
namespace fused {
using namespace prox;

enum : int { F_SETUP = 0, F_DIV = 1, F_NEWTON = 2, F_FUSED = 3, F_FINAL = 4, F_DONE = 5, F_NLOCAL = 6, F_NDIST = 7 };

constexpr int CAPW = 64;   // minimum near-list capacity per warp per pass (FArgs::capw scales it with the grid)
constexpr unsigned FULLM = 0xffffffffu;

template <int R>
struct FV {
  static constexpr int S = R * (R + 1) / 2;
  static constexpr int RHS = 0;
  static constexpr int K0 = R;
  static constexpr int CIN = 2 * R;
  static constexpr int COUT = 2 * R + S;  // end of the accumulated classes (Cout itself is never reduced:
                                          // the controller forms it from the setup gram and Cin)
  static constexpr int NRM = COUT;
  static constexpr int OVF = NRM + 2;
  static constexpr int NCNT = OVF + 1;  // near-list entries (block total / grid total)
  static constexpr int PASS = NCNT + 1;
  static constexpr int NEWTON = R + S;
  static constexpr int ACC = PASS > NEWTON ? PASS : NEWTON;
};
static_assert(FV<8>::PASS <= kMaxVals, "kMaxVals too small");

struct FCtl {
  int phase, it, newton_it, newton_total;
  int converged, status, last_newton_it, last_newton_conv;
  int final_mode, div_p, have_hist, fallbacks;
  int slot_cur, slot_prev, a_cur, local_steps;
  int single, nl_ok, ndist, cl_on;  // ndist: long near list -> distributed Newton steps; cl_on: see compact_near
  double t, t_next, m_prev, m_cur, rel, best_res, last_res, grow;
  double beta[BQ_MAX_RANK], best_beta[BQ_MAX_RANK], gw[BQ_MAX_RANK];
  double gc[BQ_MAX_RANK], gwid[BQ_MAX_RANK], glast[BQ_MAX_RANK], dmax[BQ_MAX_RANK];
  double chol[BQ_MAX_RANK * BQ_MAX_RANK];
  double chol_rdiag[BQ_MAX_RANK];  // 1 / L_ii (the per-iteration solves multiply)
  double K0[BQ_MAX_RANK], Cin[36], Cout[36];
  double gram[36];  // setup U^T D^-1 U (raw partials): sum over all voxels of u s^T = sign * gsc(gram)
  double tau;       // the launch's tau (host or dev_metric[0])
  unsigned long long t_last;
  unsigned long long phase_ns[8], phase_work_ns[8];
  int phase_cnt[8];
};

// rank thresholds of the staged pass (A/B hooks): pair accumulators, shift / box
// constants in registers, 3-deep stage ring
#ifndef BQ_PAIR_R
#define BQ_PAIR_R 2
#endif
#ifndef BQ_REGC_R
#define BQ_REGC_R 2
#endif
#ifndef BQ_RING3_R
#define BQ_RING3_R 3  // (rank 3 at 128^3: 4.17 -> 4.05 ms with the 3-deep ring; rank 4 is faster 2-deep)
#endif
constexpr int kMaxTileTab = 96; // row tiles the per-tile block assignment can describe
constexpr int NSTAGE = 3;      // max depth of the bulk-copy pipeline (3 where the stages fit, else 2)

// per-slot use counters of the stage ring, kept in registers (runtime slot
// index -> selects, not a local-memory array)
struct Uses {
  unsigned u0, u1, u2;
  __device__ unsigned get(int b) const { return b == 0 ? u0 : (b == 1 ? u1 : u2); }
  __device__ void inc(int b) {
    u0 += b == 0, u1 += b == 1, u2 += b == 2;
  }
};
__device__ __forceinline__ int ring_next(int b, int ns) { return b + 1 == ns ? 0 : b + 1; }

struct StageGeo {
  int W, SRW, nstage;           // warps used, staged rows, pipeline depth (<= NSTAGE)
  long long slot_elems;         // SRW * K1
  long long stage_elems;        // fields * slot_elems
};

template <typename T>
struct FArgs {
  int ndim, mode, sign, accelerated, max_iter, newton_max_iter, wpm_only, vec;
  int K1, K2, K3, lpr, rpw, nty, lpr_log2;
  int wpr;  // warps per x-row: 1 (K1 <= 128, rpw rows per warp) or 2 (K1 == 256, a half row each)
  long long N, plane, tile_planes;
  double tau, reg, step, eps, newton_eps, lo, hi;
  const T* lo_arr;
  const T* hi_arr;
  const T* d;
  const T* U;
  const T* v;
  T* ring[3];  // ring[0] is the caller's P (in: warm start, out: P*)
  T* abuf[2];
  T* x;
  double* beta_io;
  bq_wtv_report* report;
  double* partials;
  double* red;
  unsigned* bar;
  void* near_data;  // [2][G * NW * capw * EW] entries (T), NW = warps per block; by pass parity
  int capw;         // near-list capacity per warp per pass (>= CAPW, ~1/20 of a warp's voxels per pass)
  T* ie;            // 1/d per voxel (written by the setup pass; staged instead of d)
  int* near_cnt;  // [2][G * NW]  (pass parity: a fast block's next pass never
                  //  overwrites lists a slow block is still gathering)
  StageGeo geo;   // staged FUSED pass geometry
  long long dyn_bytes;  // dynamic shared memory of the launch
  long long list_off;   // near-list region of the dynamic smem (bytes), after the stages
  long long list_bytes;
  unsigned long long* trace;  // optional: block-0 per-step timestamps of one FUSED pass
  int trace_pass;             // which FUSED pass (iteration) to trace
  int trace_thread;           // which thread of block 0 records
  int dbg;                    // debug switches (timing experiments only)
  double grow_min;            // minimum box growth factor of the near-list Newton
  double ndist_min;           // near lists longer than this take distributed (per-block + barrier) steps
  int pre_max;                // stages of the next FUSED pass prefetched across the barrier (<= nstage)
  double* dev_metric;         // optional device [tau, rank_eff, rank_prev] (bq_wtv_desc::dev_metric)
  int cluster;                // 1: the whole grid is ONE thread-block cluster (small grids): the
                              // inter-pass barrier is a cluster barrier and the partials are
                              // exchanged through distributed shared memory
  // Staged FUSED pass, per-tile block assignment: blocks [tile_blk0[t], tile_blk0[t+1])
  // split the K3 planes of row tile t evenly, so no block's z-segment crosses a
  // tile (a crossing costs a second pre-step + warm-up plane, and those blocks
  // were the last to arrive at every barrier).  ntile_tab == 0: one contiguous
  // split of the tile-plane sequence over the grid.
  int ntile_tab;
  short tile_blk0[kMaxTileTab + 1];
  T* cl_data;        // [2][CL][EW] compact near list by pass parity (compact_near), or null
  unsigned* cl_key;  // [2][CL]
  unsigned* cl_ctr;  // monotonic slot counter (zeroed at launch)
};

// tau and the dual step of this launch: host values, or from the device
// scalars of a GPU-resident outer loop (step as dual_tv_solver.py:155-158 with
// omega = 1/tau, same operation order)
template <typename T>
__device__ __forceinline__ double eff_tau(const FArgs<T>& A) {
  return A.dev_metric ? __ldcg(A.dev_metric) : A.tau;
}
template <typename T>
__device__ __forceinline__ double eff_step(const FArgs<T>& A) {
  if (!A.dev_metric) return A.step;
  return A.reg > 0.0 ? 1.0 / (((4.0 * A.ndim) * (1.0 / __ldcg(A.dev_metric))) * A.reg) : 0.0;
}

// shared, per-block copy of what the passes read
template <typename T>
struct FShared {
  T gz[BQ_MAX_RANK];   // gamma = gw - beta (shift of the clamp argument)
  T gw[BQ_MAX_RANK];
  T gc[BQ_MAX_RANK];   // box centre / half width for the aggregates
  T gwid[BQ_MAX_RANK];
  T m_prev, m_cur;
  int phase, slot_cur, slot_prev, slot_new, a_cur, div_p, single, iter;
  int tr7;  // trace builds: stamp the first stage of this pass
  int cl_on;  // the pass also fills the grid-wide compact near list (compact_near)
};

// ---------------------------------------------------------------------------
// per-voxel helpers
// ---------------------------------------------------------------------------
template <typename T, int R>
struct Fields {
  const T* __restrict__ d;
  const T* __restrict__ U;
  const T* __restrict__ lo_arr;
  const T* __restrict__ hi_arr;
  long long N;
  T tau, lo, hi, sg;

  // q = clamp(a + s.gamma), s_c = sign u_c / e; also returns 1/e and u (4 voxels)
  __device__ __forceinline__ void q4x(const T* __restrict__ a, long long j, const T* gz, T (&q)[4], T (&ie)[4],
                                      T (&u)[R > 0 ? R : 1][4]) const {
    Vec4<T>::rw(a + j, q);
    if (R > 0) {
      T e[4];
      if (d) Vec4<T>::ro(d + j, e);
      else e[0] = e[1] = e[2] = e[3] = tau;
#pragma unroll
      for (int k = 0; k < 4; ++k) ie[k] = rcp(e[k]);
#pragma unroll
      for (int c = 0; c < R; ++c) Vec4<T>::ro(U + (long long)c * N + j, u[c]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        T z = q[k];
#pragma unroll
        for (int c = 0; c < R; ++c) z += (sg * u[c][k] * ie[k]) * gz[c];
        q[k] = z;
      }
    } else {
      T e[4];
      if (d) Vec4<T>::ro(d + j, e);
      else e[0] = e[1] = e[2] = e[3] = tau;
#pragma unroll
      for (int k = 0; k < 4; ++k) ie[k] = rcp(e[k]);
    }
    T l[4], h[4];
    bounds4(j, l, h);
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = clampv(q[k], l[k], h[k]);
  }
  __device__ __forceinline__ void q4(const T* __restrict__ a, long long j, const T* gz, T (&q)[4]) const {
    Vec4<T>::rw(a + j, q);
    if (R > 0) {
      T e[4];
      if (d) Vec4<T>::ro(d + j, e);
      else e[0] = e[1] = e[2] = e[3] = tau;
      T u[R > 0 ? R : 1][4];
#pragma unroll
      for (int c = 0; c < R; ++c) Vec4<T>::ro(U + (long long)c * N + j, u[c]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const T ie = rcp(e[k]);
        T z = q[k];
#pragma unroll
        for (int c = 0; c < R; ++c) z += (sg * u[c][k] * ie) * gz[c];
        q[k] = z;
      }
    }
    T l[4], h[4];
    bounds4(j, l, h);
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = clampv(q[k], l[k], h[k]);
  }
  // 1/e and u only (standalone DIV pass)
  __device__ __forceinline__ void ieu4(long long j, T (&ie)[4], T (&u)[R > 0 ? R : 1][4]) const {
    T e[4];
    if (d) Vec4<T>::ro(d + j, e);
    else e[0] = e[1] = e[2] = e[3] = tau;
#pragma unroll
    for (int k = 0; k < 4; ++k) ie[k] = rcp(e[k]);
#pragma unroll
    for (int c = 0; c < R; ++c) Vec4<T>::ro(U + (long long)c * N + j, u[c]);
  }
  __device__ __forceinline__ void bounds4(long long j, T (&l)[4], T (&h)[4]) const {
    if (lo_arr) Vec4<T>::ro(lo_arr + j, l);
    else l[0] = l[1] = l[2] = l[3] = lo;
    if (hi_arr) Vec4<T>::ro(hi_arr + j, h);
    else h[0] = h[1] = h[2] = h[3] = hi;
  }
  // scalar versions (near list, full Newton, final)
  __device__ __forceinline__ void voxel(const T* __restrict__ a, long long j, T& av, T (&s)[R > 0 ? R : 1],
                                        T (&u)[R > 0 ? R : 1], T& l, T& h) const {
    av = a[j];
    const T e = d ? __ldg(d + j) : tau;
    const T ie = rcp(e);
#pragma unroll
    for (int c = 0; c < R; ++c) {
      u[c] = __ldg(U + (long long)c * N + j);
      s[c] = sg * u[c] * ie;
    }
    l = lo_arr ? __ldg(lo_arr + j) : lo;
    h = hi_arr ? __ldg(hi_arr + j) : hi;
  }
};

// Classify voxel (a, s, u) for the Newton aggregates of box (gc, gwid) and
// accumulate; returns true for a "near" voxel (must go to the list).
// Only Cin is accumulated: Cout = sum_all u s^T - Cin = sign * gram - Cin is
// formed by the controller from the setup gram (one accumulator class fewer).
// HINF: the upper bound is +inf (no "high" class).
template <typename T, int R, int NACC, typename AccT, bool HINF = false>
__device__ __forceinline__ bool aggregate(T av, const T (&s)[R > 0 ? R : 1], const T (&u)[R > 0 ? R : 1], T l, T h,
                                          const T* gc, const T* gwid, AccT (&acc)[NACC]) {
  using V = FV<R>;
  T zc = av, rho = 0;
#pragma unroll
  for (int c = 0; c < R; ++c) {
    zc += s[c] * gc[c];
    rho += fabs(s[c]) * gwid[c];
  }
  // safety margin for rounding of a + s.gamma anywhere in the box
  const T eps = (sizeof(T) == 4) ? (T)1e-5 : (T)1e-13;
  rho = rho * ((T)1 + eps) + (fabs(zc) + fabs(av)) * eps;
  const bool inside = (zc - rho > l) && (HINF || zc + rho < h);
  const bool low = !inside && (zc + rho <= l);
  const bool high = HINF ? false : (!inside && !low && (zc - rho >= h));
  const bool near = !inside && !low && !high;
  // branch-free accumulation (selects, never arithmetic on an unused +-inf bound)
  const T k0 = low ? av - l : (HINF ? (near ? av : (T)0) : (high ? av - h : (near ? av : (T)0)));
  // Cin += [inside] u s^T as one select per column and fused multiply-adds
  int k = 0;
#pragma unroll
  for (int c = 0; c < R; ++c) {
    const AccT ui = inside ? (AccT)u[c] : (AccT)0;
#pragma unroll
    for (int c2 = 0; c2 <= c; ++c2, ++k) acc[V::CIN + k] = fma(ui, (AccT)s[c2], acc[V::CIN + k]);
    acc[V::K0 + c] = fma((AccT)u[c], (AccT)k0, acc[V::K0 + c]);
  }
  return near;
}

// aggregate() for a voxel pair (packed f32x2 where the arithmetic allows):
// the same classification and sums, element by element; u is the lane's
// [RR][2] pair array, p selects the pair.
template <typename T, int R, int NACC, bool HINF, typename AccT>
__device__ __forceinline__ void aggregate2(pair_t<T> av, const pair_t<T> (&s)[R > 0 ? R : 1],
                                           const pair_t<T> (&u)[R > 0 ? R : 1][2], int p, pair_t<T> l,
                                           pair_t<T> h, const T* gc, const T* gwid,
                                           AccT (&acc)[NACC], bool& n0, bool& n1) {
  using V = FV<R>;
  using P = pair_t<T>;
  P zc = av, rho = bc2((T)0);
#pragma unroll
  for (int c = 0; c < R; ++c) {
    zc = fma2(s[c], bc2(gc[c]), zc);
    rho = fma2(abs2(s[c]), bc2(gwid[c]), rho);
  }
  const T eps = (sizeof(T) == 4) ? (T)1e-5 : (T)1e-13;
  rho = fma2(rho, bc2((T)1 + eps), mul2(add2(abs2(zc), abs2(av)), bc2(eps)));
  const P lo_side = sub2(zc, rho), hi_side = add2(zc, rho);
  const P avl = sub2(av, l);
  bool in[2], nr[2];
  P k0;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const T ls = e ? lo_side.y : lo_side.x, hs = e ? hi_side.y : hi_side.x;
    const T le = e ? l.y : l.x, he = e ? h.y : h.x, a = e ? av.y : av.x;
    const bool inside = (ls > le) && (HINF || hs < he);
    const bool low = !inside && (hs <= le);
    const bool high = HINF ? false : (!inside && !low && (ls >= he));
    const bool near = !inside && !low && !high;
    const T kl = e ? avl.y : avl.x;
    const T kv = low ? kl : (HINF ? (near ? a : (T)0) : (high ? a - he : (near ? a : (T)0)));
    if (e) k0.y = kv;
    else k0.x = kv;
    in[e] = inside, nr[e] = near;
  }
  int k = 0;
#pragma unroll
  for (int c = 0; c < R; ++c) {
    const P uu = u[c][p];
    const P ui = mk2(in[0] ? uu.x : (T)0, in[1] ? uu.y : (T)0);
#pragma unroll
    for (int c2 = 0; c2 <= c; ++c2, ++k) accf(acc[V::CIN + k], ui, s[c2]);
    accf(acc[V::K0 + c], uu, k0);
  }
  n0 = nr[0], n1 = nr[1];
}

// Warp-deterministic compaction of near voxels into this warp's segment; the
// entry carries the voxel's data (a, lo, hi, u[R], s[R]) so the on-chip Newton
// never has to chase indices.
template <typename T, int R>
__device__ __forceinline__ void near_push(bool flag, T av, T l, T h, const T (&u)[R > 0 ? R : 1],
                                          const T (&s)[R > 0 ? R : 1], int lane, T* seg, int& cnt, bool& ovf,
                                          int cap) {
  constexpr int EW = 3 + 2 * (R > 0 ? R : 1);
  const unsigned m = __ballot_sync(FULLM, flag);
  if (m == 0) return;
  const int n = __popc(m);
  if (cnt + n > cap) {
    ovf = true;
    cnt = cap;
    return;
  }
  if (flag) {
    T* d = seg + (long long)(cnt + __popc(m & ((1u << lane) - 1u))) * EW;
    d[0] = av, d[1] = l, d[2] = h;
#pragma unroll
    for (int c = 0; c < R; ++c) d[3 + c] = u[c], d[3 + R + c] = s[c];
  }
  cnt += n;
}

// Grid-wide compact copy of SHORT near lists (steady state: 0-3 entries in
// the whole grid).  After a pass, a warp that listed voxels reserves slots in
// one small global array with an atomic on a monotonic counter (slot = old -
// base, base = the counter after the previous pass, the same in every block)
// and copies its entries there, each with its position in segment order as
// key.  After the barrier every block already holds those CL slots (loaded
// with the partials, no further round trip: no count scan, no gather) and
// sorts them by key, so the evaluation order is the segment order whatever
// order the atomics ran in.  Done outside the march loop (inlined into it, the
// reservation cost the loop 0.05 ms per 128^3 solve).
constexpr int CL = 32;
template <typename T, int EW>
__device__ __forceinline__ void compact_near(const T* seg, int cnt, unsigned key0, unsigned* ctr, unsigned base,
                                             T* data, unsigned* key, int lane) {
  __syncwarp();  // the segment was written lane by lane
  unsigned slot0 = 0;
  if (lane == 0) slot0 = atomicAdd(ctr, (unsigned)cnt) - base;
  slot0 = __shfl_sync(FULLM, slot0, 0);
  for (int e = lane; e < cnt; e += 32) {
    const unsigned slot = slot0 + (unsigned)e;
    if (slot < (unsigned)CL) {
#pragma unroll
      for (int f = 0; f < EW; ++f) data[(long long)slot * EW + f] = __ldcg(seg + (long long)e * EW + f);
      key[slot] = key0 + (unsigned)e;
    }
  }
}

// ---------------------------------------------------------------------------
// controller (thread 0 of every block, on the block's own shared state)
// ---------------------------------------------------------------------------
template <typename T, int R>
struct Ctl {
  using V = FV<R>;
  const FArgs<T>& A;
  FCtl& c;
  bool writer;

  __device__ bool diag() const { return A.d != nullptr; }
  // gram-like reduced entry -> metric units (scalar metric divides by tau)
  __device__ double gsc(double g) const { return diag() ? g : g / c.tau; }

  __device__ void timeline(int phase, const double* red, bool passed_barrier) {
    const unsigned long long now = global_ns();
    if (phase == F_SETUP) {
      for (int i = 0; i < 8; ++i) c.phase_ns[i] = 0, c.phase_work_ns[i] = 0, c.phase_cnt[i] = 0;
    } else {
      c.phase_ns[phase] += now - c.t_last;
      const unsigned long long arrive = passed_barrier ? __double_as_longlong(red[kMaxVals - 1]) : now;
      if (arrive > c.t_last && arrive <= now) c.phase_work_ns[phase] += arrive - c.t_last;
      c.phase_cnt[phase] += 1;
    }
    c.t_last = now;
  }

  __device__ void next_box_and_continue(bool used_fallback) {
    // predict the next gamma box from the last two Newton solutions
    double g[BQ_MAX_RANK > 0 ? BQ_MAX_RANK : 1];
    for (int i = 0; i < R; ++i) g[i] = c.gw[i] - c.beta[i];
    if (used_fallback) c.grow = fmin(c.grow * 4.0, 1e12);
    else c.grow = fmax(A.grow_min, c.grow * 0.5);
    double scale = 0.0;
    for (int i = 0; i < R; ++i) scale = fmax(scale, fabs(g[i]));
    for (int i = 0; i < R; ++i) {
      const double dg = c.have_hist ? g[i] - c.glast[i] : 0.0;
      // decaying envelope of recent steps: the trajectory of gamma is not smooth
      c.dmax[i] = c.have_hist ? fmax(0.75 * c.dmax[i], fabs(dg)) : 0.0;
      c.gc[i] = g[i] + dg;
      c.gwid[i] = c.grow * (fabs(dg) + c.dmax[i]) + 1e-7 * c.grow * (fabs(g[i]) + scale) + 1e-300;
      c.glast[i] = g[i];
    }
    c.have_hist = 1;
  }

  __device__ void finish_newton(int converged) {
    for (int i = 0; i < R; ++i) c.beta[i] = c.best_beta[i];
    c.newton_total += c.newton_it;
    c.last_newton_it = c.newton_it;
    c.last_newton_conv = converged;
    c.last_res = (R == 0) ? 0.0 : c.best_res;
    next_box_and_continue(c.fallbacks > 0);
    c.phase = c.final_mode ? F_FINAL : F_FUSED;
  }

  // one Newton evaluation result (phi without beta, H without I) -> decision
  // wpm.py:207-224.  Returns the next phase.
  __device__ void newton_step(const double* phi_part, const double* h_part) {
    double phi[BQ_MAX_RANK > 0 ? BQ_MAX_RANK : 1];
    double ss = 0.0;
    for (int i = 0; i < R; ++i) {
      phi[i] = phi_part[i] + c.beta[i];
      ss += phi[i] * phi[i];
    }
    const double res = R == 1 ? fabs(phi[0]) : sqrt(ss);
    if (res < c.best_res) {
      c.best_res = res;
      for (int i = 0; i < R; ++i) c.best_beta[i] = c.beta[i];
    }
    if (res <= A.newton_eps) return finish_newton(1);
    if (c.newton_it == A.newton_max_iter) return finish_newton(0);
    double h[R > 0 ? R * R : 1], hs[R > 0 ? R * R : 1], st[R > 0 ? R : 1];
    int k = 0;
    for (int i = 0; i < R; ++i)
      for (int j = 0; j <= i; ++j, ++k) {
        const double val = (i == j ? 1.0 : 0.0) + h_part[k];
        h[i * R + j] = val;
        h[j * R + i] = val;
      }
    for (int i = 0; i < R * R; ++i) hs[i] = h[i];
    for (int i = 0; i < R; ++i) st[i] = phi[i];
    if (!lu<R>(hs, st)) {
      double ninf = 0.0;  // Levenberg fallback, wpm.py:219-223
      for (int i = 0; i < R; ++i) {
        double rs = 0.0;
        for (int j = 0; j < R; ++j) rs += fabs(h[i * R + j]);
        ninf = fmax(ninf, rs);
      }
      for (int i = 0; i < R * R; ++i) hs[i] = h[i];
      for (int i = 0; i < R; ++i) hs[i * R + i] += 1e-8 * ninf, st[i] = phi[i];
      lu<R>(hs, st);
    }
    for (int i = 0; i < R; ++i) c.beta[i] -= st[i];
    c.newton_it += 1;
    choose_newton_mode();
  }

  // local (near-list) evaluation is exact while gamma stays in the box
  __device__ void choose_newton_mode() {
    bool in_box = c.nl_ok != 0;
    for (int i = 0; i < R; ++i) {
      const double g = c.gw[i] - c.beta[i];
      if (!(fabs(g - c.gc[i]) <= c.gwid[i])) in_box = false;
    }
    if (in_box) {
      c.phase = c.ndist ? F_NDIST : F_NLOCAL;
    } else {
      if (c.phase != F_NEWTON) c.fallbacks += 1;
      c.phase = F_NEWTON;
    }
  }

  // after a DIV or FUSED pass: Woodbury coefficient and Newton start
  __device__ void after_div(const double* red) {
    double coef[R > 0 ? R : 1];
    for (int i = 0; i < R; ++i) coef[i] = gsc(red[V::RHS + i]);
    if (R > 0) chol_solve_rd<R>(c.chol, c.chol_rdiag, coef);
    for (int i = 0; i < R; ++i) c.gw[i] = c.single ? 0.0 : A.reg * coef[i];
    for (int i = 0; i < R; ++i) c.K0[i] = red[V::K0 + i];
    for (int k = 0; k < V::S; ++k) c.Cin[k] = red[V::CIN + k], c.Cout[k] = A.sign * gsc(c.gram[k]) - c.Cin[k];
    c.nl_ok = red[V::OVF] == 0.0;
    c.ndist = red[V::NCNT] > A.ndist_min ? 1 : 0;
    c.cl_on = (!A.cluster && A.cl_data && red[V::NCNT] <= 2.0 * CL) ? 1 : 0;  // lists shrink slowly: worth filling
    c.fallbacks = 0;
    c.newton_it = 0;
    c.best_res = INFINITY;
    for (int i = 0; i < R; ++i) c.best_beta[i] = c.beta[i];
    if (R == 0) {
      c.best_res = 0.0;
      finish_newton(1);
      return;
    }
    c.phase = F_DIV;  // sentinel so a first out-of-box start is not counted twice
    choose_newton_mode();
  }

  // phi(beta) = K0 + Cout gw + Cin beta - sum_near u clamp(a + s.gamma) (+ beta in newton_step),
  // H = Cin + sum_near,inside u s^T (+ I): exact while gamma stays in the aggregates' box
  __device__ void local_eval(const double* nacc, double* phi, double* hp) const {
    for (int i = 0; i < R; ++i) {
      double cw = 0.0, cb = 0.0;
      for (int k2 = 0; k2 < R; ++k2) {
        const int kk = i >= k2 ? i * (i + 1) / 2 + k2 : k2 * (k2 + 1) / 2 + i;
        cw += c.Cout[kk] * c.gw[k2];
        cb += c.Cin[kk] * c.beta[k2];
      }
      phi[i] = c.K0[i] + cw + cb - nacc[i];
    }
    for (int k = 0; k < V::S; ++k) hp[k] = c.Cin[k] + nacc[R + k];
  }

  __device__ void run(int phase, const double* red) {
    switch (phase) {
      case F_SETUP: {
        c.tau = eff_tau(A);
        double cap[R > 0 ? R * R : 1];
        int k = 0;
        for (int i = 0; i < R; ++i)
          for (int j = 0; j <= i; ++j, ++k) {
            const double val = (i == j ? 1.0 : 0.0) + A.sign * gsc(red[k]);
            cap[i * R + j] = val;
            cap[j * R + i] = val;
          }
        for (int q = 0; q < V::S; ++q) c.gram[q] = red[q];
        c.status = 0;
        if (R > 0 && !chol<R>(cap)) {
          c.status = BQ_ENOTPD;
          c.phase = F_DONE;
          if (writer) A.report->status = BQ_ENOTPD;
          return;
        }
        for (int i = 0; i < R * R; ++i) c.chol[i] = cap[i];
        for (int i = 0; i < R; ++i) c.chol_rdiag[i] = 1.0 / cap[i * R + i];
        // GPU-resident loop: the warm start is dropped when the effective rank changed
        const bool keep = !A.dev_metric || __ldcg(A.dev_metric + 1) == __ldcg(A.dev_metric + 2);
        for (int i = 0; i < R; ++i) {
          c.beta[i] = (A.beta_io && keep) ? A.beta_io[i] : 0.0;
          c.gw[i] = 0.0;
          c.gc[i] = -c.beta[i];  // gw == 0 when the warm start is zero
          c.gwid[i] = 0.0;       // forces one full Newton evaluation first
          c.glast[i] = 0.0;
        }
        c.have_hist = 0;
        c.grow = A.grow_min;
        for (int i = 0; i < R; ++i) c.dmax[i] = 0.0;
        c.t = 1.0;
        c.it = 1;
        c.newton_total = 0;
        c.converged = 0;
        c.rel = INFINITY;
        c.last_newton_it = 0;
        c.last_newton_conv = 1;
        c.last_res = 0.0;
        c.single = (A.wpm_only || A.reg == 0.0) ? 1 : 0;
        c.final_mode = c.single;
        c.slot_cur = 0;
        c.slot_prev = 0;
        c.a_cur = 1;    // the DIV pass writes abuf[1 - a_cur] = abuf[0]
        c.m_prev = 0.0; // P_bar_0 = P_0
        c.div_p = 1;    // DIV source: P_0 (== P_bar_0)
        c.cl_on = 0;
        c.phase = F_DIV;
        return;
      }
      case F_DIV:
        c.a_cur ^= 1;
        after_div(red);
        return;
      case F_NEWTON: {
        // full-pass evaluation of phi and H at beta (wpm.py:150-167)
        double hp[V::S > 0 ? V::S : 1];
        for (int k = 0; k < V::S; ++k) hp[k] = red[R + k];
        newton_step(red, hp);
        return;
      }
      case F_NDIST: {
        // box-exact evaluation, near terms summed block by block (red = sum_near u clamp, H near part)
        double phi[R > 0 ? R : 1], hp[V::S > 0 ? V::S : 1];
        local_eval(red, phi, hp);
        newton_step(phi, hp);
        return;
      }
      case F_FUSED: {
        // dual_tv_solver.py:226-239 on the ring
        const double num = sqrt(red[V::NRM]), den = sqrt(red[V::NRM + 1]);
        const double rel = (num == 0.0) ? 0.0 : (den > 0.0 ? num / den : INFINITY);
        c.rel = rel;
        const int slot_new = (c.slot_cur == c.slot_prev) ? (c.slot_cur + 1) % 3 : 3 - c.slot_cur - c.slot_prev;
        c.slot_prev = c.slot_cur;
        c.slot_cur = slot_new;
        c.a_cur ^= 1;
        if (rel < A.eps) {
          c.converged = 1;
          c.final_mode = 1;
          if (!c.div_p) {
            // a was built from P_bar_i; the final prox needs div(p_i)
            c.div_p = 1;
            c.m_prev = 0.0;
            c.slot_prev = c.slot_cur;
            c.phase = F_DIV;
            return;
          }
        } else {
          c.t = c.t_next;  // 0.5 (1 + sqrt(1 + 4 t^2)), computed by prepare_fused
          if (c.div_p) c.final_mode = 1;  // that was the last iteration
          else c.it += 1;
        }
        c.m_prev = c.m_cur;
        after_div(red);
        return;
      }
      case F_FINAL: {
        if (writer) {
          bq_wtv_report* rp = A.report;
          rp->iterations = c.single ? 1 : c.it;
          rp->converged = c.single ? 1 : c.converged;
          rp->rel_change = c.single ? 0.0 : c.rel;
          rp->newton_iterations = c.newton_total;
          rp->status = 0;
          rp->newton_residual = c.last_res;
          rp->last_newton_iterations = c.last_newton_it;
          rp->last_newton_converged = c.last_newton_conv;
          if (A.beta_io)
            for (int i = 0; i < R; ++i) A.beta_io[i] = c.beta[i];
          if (A.dev_metric) A.dev_metric[2] = A.dev_metric[1];
          for (int i = 0; i < 6; ++i) {
            // [setup, div, newton (full pass), fused, final, newton (on-chip + distributed near list)]
            const int src = (i == 5) ? F_NLOCAL : i;
            rp->phase_ns[i] = (double)c.phase_ns[src] + (i == 5 ? (double)c.phase_ns[F_NDIST] : 0.0);
            rp->phase_work_ns[i] = (double)c.phase_work_ns[src] + (i == 5 ? (double)c.phase_work_ns[F_NDIST] : 0.0);
            rp->phase_count[i] = c.phase_cnt[src] + (i == 5 ? c.phase_cnt[F_NDIST] : 0);
          }
        }
        c.phase = F_DONE;
        return;
      }
      default:
        c.phase = F_DONE;
    }
  }

  // before a FUSED pass: momentum coefficients and the div source
  __device__ void prepare_fused() {
    const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * c.t * c.t));
    c.t_next = tn;
    c.m_cur = A.accelerated ? (c.t - 1.0) / tn : 0.0;
    c.div_p = (c.it >= A.max_iter) ? 1 : 0;
  }
};

// ---------------------------------------------------------------------------
// FUSED pass with bulk-async staging (TMA engine): per plane-step one thread
// copies the block's contiguous row ranges of every input field into a
// double-buffered shared-memory stage (mbarrier completion); all warps compute
// from shared memory.  Stage of step k: q-inputs (a, d, U, bounds) of plane
// k+1 and P_{i-1}, P_{i-2}, v of plane k.  Staged rows y_base .. y_base+W*rpw:
// warp 0 owns the halo rows above the tile, the last staged row is the row
// below it (its q is computed by warp 0 too).
// ---------------------------------------------------------------------------

struct StepIter {
  int pos, seg_end, tile;
  int z0, z1, zs, k, K3, nd;
  bool valid;
  __device__ void init(long long b, long long e, int K3_, int nd_) {
    pos = (int)b, seg_end = (int)e, K3 = K3_, nd = nd_;
    next_segment();
  }
  __device__ void next_segment() {
    valid = pos < seg_end;
    if (!valid) return;
    tile = pos / K3;
    z0 = pos - tile * K3;
    z1 = min(K3, z0 + (seg_end - pos));
    pos += z1 - z0;
    zs = (z0 > 0 && nd >= 3) ? z0 - 1 : z0;
    k = zs - 1;  // pre-step: q-inputs of plane zs only
  }
  __device__ void advance() {
    if (++k > z1 - 1) next_segment();
  }
  __device__ bool has_qin() const { return k + 1 < K3; }
  __device__ bool has_pin() const { return k >= zs; }
};

template <int R>
struct StageMap {
  int A, D, U0, LO, HI, V, PC0, PP0, nfield;  // field slots (-1: absent)
  __host__ __device__ void make(bool diag, bool lo_arr, bool hi_arr, int nd, bool need_pp) {
    int f = 0;
    A = f++;
    D = diag ? f++ : -1;
    U0 = f;
    f += R;
    LO = lo_arr ? f++ : -1;
    HI = hi_arr ? f++ : -1;
    V = f++;
    PC0 = f;
    f += nd;
    PP0 = need_pp ? f : -1;
    if (need_pp) f += nd;
    nfield = f;
  }
};

// Issue the bulk copies of one step.  Called by all 32 lanes of the producer
// warp: copy i is issued by lane i (descriptor math in parallel), lane 0 arms
// the mbarrier with the total byte count.
template <typename T, int R>
__device__ __forceinline__ void issue_step(const FArgs<T>& A, const StepIter& it, const StageMap<R>& M,
                                           const StageGeo& g, T* stage, unsigned long long* bar, const T* Pc,
                                           const T* Pp, const T* Ain, int lane) {
  const int K1 = A.K1, K2 = A.K2, rpw = A.rpw;
  const long long N = A.N, plane = A.plane;
  const int GW = g.W / A.wpr;  // row groups (the first is the halo group)
  const int TYe = (GW - 1) * rpw;
  const int y0 = (int)it.tile * TYe;
  const int y_base = y0 - rpw;
  // enumerate copies: index -> (slot, base, plane, row range)
  int slot = -1, ya = 0, yb = 0;
  const T* base = nullptr;
  long long zp = 0;
  int idx = 0;
  auto pick = [&](int sl, const T* bs, long long z, int a, int b) {
    if (sl < 0) return;
    if (idx == lane) slot = sl, base = bs, zp = z, ya = a, yb = b;
    ++idx;
  };
  if (it.has_qin()) {
    const long long zq = it.k + 1;
    pick(M.A, Ain, zq, y_base, y_base + g.SRW);
    pick(M.D, A.ie, zq, y_base, y_base + g.SRW);
    for (int c = 0; c < R; ++c) pick(M.U0 + c, A.U + (long long)c * N, zq, y_base, y_base + g.SRW);
    pick(M.LO, A.lo_arr, zq, y_base, y_base + g.SRW);
    pick(M.HI, A.hi_arr, zq, y_base, y_base + g.SRW);
  }
  if (it.has_pin()) {
    const long long zk = it.k;
    pick(M.V, A.v, zk, y0, y0 + TYe);
    for (int n = 0; n < A.ndim; ++n) {
      pick(M.PC0 + n, Pc + n * N, zk, y_base, y_base + GW * rpw);
      if (M.PP0 >= 0) pick(M.PP0 + n, Pp + n * N, zk, y_base, y_base + GW * rpw);
    }
  }
  unsigned bytes = 0;
  if (slot >= 0) {
    ya = max(ya, 0);
    yb = min(yb, K2);
    if (yb > ya) bytes = (unsigned)((long long)(yb - ya) * K1 * (long long)sizeof(T));
  }
  unsigned total = bytes;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(FULLM, total, o);
  if (lane == 0) {
    fence_proxy_async_smem();
    mbar_expect_tx(bar, total);
  }
  __syncwarp();
  if (bytes)
    bulk_g2s(stage + slot * g.slot_elems + (long long)(ya - y_base) * K1, base + zp * plane + (long long)ya * K1,
             bytes, bar);
}

// MODE 0: generic (optional bound arrays); 1: scalar bounds (the bounds are
// pass constants, no bound fields in the stage).  Per-voxel d or scalar tau is
// a runtime choice in both.
// KX > 0: the row length K1 == KX is a compile-time constant (lane -> voxel
// mapping, row offsets and every per-row branch fold; K1 == 128 is the
// common 128^3 case), KX == 0: runtime K1.
template <typename T, int R, int NACC, int MODE, int KX>
__device__ __forceinline__ void fused_staged(const FArgs<T>& A, const FShared<T>& sh, const StageGeo& g,
                                             long long seg_begin, long long seg_end, T* dyn,
                                             unsigned long long* full, unsigned long long* empty,
                                             Uses& uses, double (&acc)[NACC], T* near_seg,
                                             int& ncnt, bool& ovf, int pre) {
  using V = FV<R>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long N = A.N;
  constexpr int nd = 3;  // the fused path serves 3-D grids (others use wtv_prox.cu)
  const int K1 = KX > 0 ? KX : A.K1, K2 = A.K2, K3 = A.K3;
  // x-split (K1 == 256): warps 2g and 2g+1 hold the left / right half of row group g
  constexpr int wpr = KX > 128 ? 2 : 1;  // the x-split has its own instantiation (KX == 256)
  const int rpw = KX > 0 ? (KX >= 128 ? 1 : 128 / KX) : A.rpw;
  const int xr = KX > 0 ? (KX >= 128 ? lane : lane % (KX / 4)) : lane & (A.lpr - 1);
  const int yr = KX > 0 ? (KX >= 128 ? 0 : lane / (KX / 4)) : lane >> A.lpr_log2;
  const int xh = wpr == 2 ? (warp & 1) : 0;
  const int wg = wpr == 2 ? (warp >> 1) : warp;
  const int xb = 4 * xr + 128 * xh;
  const bool first_in_row = xr == 0 && xh == 0, last_in_row = xb + 4 >= K1;
  const bool edge_src = wpr == 2 && xh == 0 && lane == 31;  // publishes its x+1 / x-1 halves' values
  const bool edge_dst = wpr == 2 && xh == 1 && lane == 0;
  const int W = g.W;
  const int GW = W / wpr;
  const int TYe = (GW - 1) * rpw;
  const bool used = warp < W;
  const bool halo = wg == 0;
  const int sr = wg * rpw + yr;  // staged row of this thread
  __shared__ T s_edge[2][32];    // x-split: div source x = 127 of each staged row, by step parity
  const T* __restrict__ Pc = A.ring[sh.slot_cur];
  const T* __restrict__ Pp = A.ring[sh.slot_prev];
  T* __restrict__ Pn = A.ring[sh.slot_new];
  const T* __restrict__ Ain = A.abuf[sh.a_cur];
  T* __restrict__ Aout = A.abuf[sh.a_cur ^ 1];
  const T m_prev = sh.m_prev, m_cur = sh.m_cur;
  const bool div_p = sh.div_p;
  const T step = (T)eff_step(A), reg = (T)A.reg, sg = (T)A.sign;
  const bool diag = A.d != nullptr;
  const T itauT = diag ? (T)1 : rcp((T)eff_tau(A));
  const bool iso = A.mode == BQ_TV_ISO;
  StageMap<R> M;
  // p_{i-2} is always staged (unused while m_prev == 0) so that the layout does
  // not depend on the controller: the first stages are prefetched before it runs
  M.make(diag, MODE == 0 && A.lo_arr != nullptr, MODE == 0 && A.hi_arr != nullptr, nd, true);
  // measured at 128^3 (A/B in one call): rank 4 4.86 -> 4.69 ms, rank 5 6.27 -> 6.17 ms;
  // ranks 3, 6 and 8 are 1-2% slower with it
  constexpr bool ULATE = sizeof(T) == 4 && (R == 4 || R == 5);
  const int NS = g.nstage;
  T* const qbuf = dyn + NS * g.stage_elems;   // [2][SRW][K1]
  T* const srcbuf = qbuf + 2 * g.slot_elems;  // [2][SRW][K1]
  const T lo_s = (T)A.lo, hi_s = (T)A.hi;
  const bool hinf = !(MODE == 0 && A.hi_arr != nullptr) && isinf(A.hi) && A.hi > 0;  // box [lo, +inf)

  // ---- producer warp (warp W): issues the bulk copies, 2 stages ahead ----
  if (warp == W) {
    fence_proxy_async_global();  // this pass reads data written before the grid barrier
    StepIter prod;
    prod.init(seg_begin, seg_end, K3, nd);
    Uses pu = uses;  // includes the fills of the prefetched steps
    int ps = 0, b = 0;
    for (; ps < pre && prod.valid; ++ps) prod.advance(), b = ring_next(b, NS);
    while (prod.valid) {
      if (ps >= NS) mbar_wait(&empty[b], (pu.get(b) - 1) & 1u);  // consumers released it
      issue_step<T, R>(A, prod, M, g, dyn + b * g.stage_elems, &full[b], Pc, Pp, Ain, lane);
      pu.inc(b);
      prod.advance();
      ++ps;
      b = ring_next(b, NS);
    }
    uses = pu;  // in step with the consumers
    return;
  }
  if (warp > W) {
    StepIter cnt;
    cnt.init(seg_begin, seg_end, K3, nd);
    int b = 0;
    while (cnt.valid) {
      uses.inc(b);
      cnt.advance();
      b = ring_next(b, NS);
    }
    return;
  }
#if BQ_PROX_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0 && sh.tr7) A.trace[320 + 11] = global_ns();
#endif
  StepIter cons;
  cons.init(seg_begin, seg_end, K3, nd);
  // Partial sums of the pass: the accumulated classes (RHS, K0, Cin, norms) are
  // summed per thread in the field type across steps, as voxel pairs (packed
  // f32x2 in f32); in fp32 they are flushed every FLUSH steps through a
  // fixed-order warp reduction into per-warp f64 accumulators in shared memory
  // (so the f64 partials hold no registers during the march), and into acc at
  // the end of the pass.
  using P = pair_t<T>;
  constexpr int RR = R > 0 ? R : 1;
  constexpr int NSUM = V::COUT + 2;  // [0, COUT) and the two norms
  constexpr int FLUSH = sizeof(T) == 4 ? 32 : (1 << 30);
  __shared__ double s_wacc[16][sizeof(T) == 4 ? NSUM : 1];
  // pair accumulators at ranks <= 2; higher ranks fold each pair into a scalar
  // accumulator at once (their 2R + R(R+1)/2 classes would not fit as pairs)
  using AccT = typename std::conditional<(sizeof(T) == 4 && R <= BQ_PAIR_R), P, T>::type;
  AccT fa[NACC];
#pragma unroll
  for (int q = 0; q < NACC; ++q) acc_zero(fa[q]);
  if (sizeof(T) == 4)
    for (int q = lane; q < NSUM; q += 32) s_wacc[warp][q] = 0.0;
  P qc[2] = {bc2((T)0), bc2((T)0)}, iec[2] = {bc2((T)1), bc2((T)1)}, uc[RR][2];
  P f3p[2] = {bc2((T)0), bc2((T)0)};
#pragma unroll
  for (int c = 0; c < RR; ++c) uc[c][0] = uc[c][1] = bc2((T)0);
  // branch-free forms of the pass constants: src = w + m_src (w - p_{i-1})
  // (m_src = 0 on the last iteration, the div source is p_i itself); sgz =
  // sign * gamma so that q = clamp(a + (u / d) sgz) (the sign is exact)
  const P m_src2 = bc2(div_p ? (T)0 : m_cur), m_prev2 = bc2(m_prev), step2 = bc2(step);
  const P nreg2 = bc2(sh.single ? (T)0 : -reg);
  // ranks <= 2 keep the shift and box in registers, higher ranks read them
  // from shared memory at use (register budget)
  constexpr int RH = R <= BQ_REGC_R ? RR : 1;
  T sgz[RH], gcv[RH], gwv[RH];
#pragma unroll
  for (int c = 0; c < RH; ++c) sgz[c] = R > 0 ? sg * sh.gz[c] : (T)0, gcv[c] = sh.gc[c], gwv[c] = sh.gwid[c];
  const T* const gcp = R <= BQ_REGC_R ? gcv : sh.gc;
  const T* const gwp = R <= BQ_REGC_R ? gwv : sh.gwid;
  int s = 0, b = 0;
#if BQ_PROX_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0 && sh.tr7) A.trace[320 + 12] = global_ns();
#endif
  while (cons.valid) {
    T* const stg = dyn + b * g.stage_elems;
    unsigned long long t_a = 0, t_b = 0;
#if BQ_PROX_TRACE
    const bool tr = A.trace && blockIdx.x == 0 && threadIdx.x == A.trace_thread && sh.iter == A.trace_pass && s < 60;
#else
    constexpr bool tr = false;
#endif
    if (tr) t_a = global_ns();
    mbar_wait(&full[b], uses.get(b) & 1u);
#if BQ_PROX_TRACE
    if (s == 0 && blockIdx.x == 0 && threadIdx.x == 0 && sh.tr7) A.trace[320 + 7] = global_ns();
#endif
    if (tr) t_b = global_ns();
    uses.inc(b);
    const int k = cons.k;
    const int y0 = (int)cons.tile * TYe;
    const int y = y0 - rpw + sr;
    const bool act = used && y >= 0 && y < K2;
    const bool real = act && !halo;
    const bool warm = k < cons.z0;
    const bool pin = cons.has_pin();
    if (k == cons.zs - 1) f3p[0] = f3p[1] = bc2((T)0);
    const int rowoff = sr * K1 + xb;

    // ---- q(k+1) of this row (+ the row below the tile, by warp 0) -------
    P qn[2] = {bc2((T)0), bc2((T)0)}, ien[2] = {bc2((T)1), bc2((T)1)}, un[RR][2];
#pragma unroll
    for (int c = 0; c < RR; ++c) un[c][0] = un[c][1] = bc2((T)0);
    if (cons.has_qin()) {
      auto qrow = [&](long long off, P (&q)[2], P (&ie)[2], P (&u)[RR][2]) {
        P l[2], h[2];
        ld2(stg + M.A * g.slot_elems + off, q);
        if (diag) ld2(stg + M.D * g.slot_elems + off, ie);  // 1/d, precomputed
        else ie[0] = ie[1] = bc2(itauT);
#pragma unroll
        for (int c = 0; c < R; ++c) ld2(stg + (M.U0 + c) * g.slot_elems + off, u[c]);
        if (MODE == 0 && M.LO >= 0) ld2(stg + M.LO * g.slot_elems + off, l);
        else l[0] = l[1] = bc2(lo_s);
        if (MODE == 0 && M.HI >= 0) ld2(stg + M.HI * g.slot_elems + off, h);
        else h[0] = h[1] = bc2(hi_s);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          P z = q[p];
#pragma unroll
          for (int c = 0; c < R; ++c) z = fma2(mul2(u[c][p], ie[p]), bc2(R <= BQ_REGC_R ? sgz[c < RH ? c : 0] : sg * sh.gz[c]), z);
          q[p] = mk2(clampv(z.x, l[p].x, h[p].x), clampv(z.y, l[p].y, h[p].y));
        }
      };
      T* qdst = qbuf + (long long)((k + 1) & 1) * g.slot_elems;
      if (act) {
        if (ULATE) {
          // ranks > 2: u(k+1) is not kept across the dual update (the register
          // peak of the step); it is re-read from the stage before the release below
          P ut[RR][2];
          qrow(rowoff, qn, ien, ut);
        } else {
          qrow(rowoff, qn, ien, un);
        }
        st2(qdst + rowoff, qn);
      }
      if (halo && yr == 0 && y0 + TYe < K2) {
        const long long off = (long long)(GW * rpw) * K1 + xb;
        P qb[2], ib[2], ub[RR][2];
        qrow(off, qb, ib, ub);
        st2(qdst + off, qb);
      }
    }

    // ---- dual update at plane k (dual_tv_solver.py:225-235) -------------
    // x+1 of element 3; the row's last lane uses its own element 3 (zero gradient)
    const T qsh = __shfl_down_sync(FULLM, qc[0].x, 1);
    // x-split: q(x = 128) of this row comes from the q row published in the last step
    const T qright = last_in_row ? qc[1].y : (edge_src ? qbuf[(long long)(k & 1) * g.slot_elems + rowoff + 4] : qsh);
    P src[3][2];
    P vv[2] = {bc2((T)0), bc2((T)0)};
#pragma unroll
    for (int n = 0; n < 3; ++n) src[n][0] = src[n][1] = bc2((T)0);
    if (pin && act) {
      const bool has_y = y < K2 - 1;
      const bool has_up = k < K3 - 1;
      P qy[2];  // q of row y+1; at the last row q itself (zero gradient, no select)
      if (has_y) ld2(qbuf + (long long)(k & 1) * g.slot_elems + rowoff + K1, qy);
      else qy[0] = qc[0], qy[1] = qc[1];
      if (!has_up) qn[0] = qc[0], qn[1] = qc[1];  // last plane
      P pc[3][2], pp[3][2];
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        ld2(stg + (M.PC0 + n) * g.slot_elems + rowoff, pc[n]);
        ld2(stg + (M.PP0 + n) * g.slot_elems + rowoff, pp[n]);
      }
      const bool acc_n = real && !warm;
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        // x neighbours straddle the pairs: element 2p+1's right is 2p+2
        const T r0 = qc[p].y, r1 = p == 0 ? qc[1].x : qright;
        P w[3];
        w[0] = mk2(r0 - qc[p].x, r1 - qc[p].y);
        w[1] = sub2(qy[p], qc[p]);
        w[2] = sub2(qn[p], qc[p]);
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          // P_bar_{i-1} = p_{i-1} + m (p_{i-1} - p_{i-2})  (:235), then + step D q
          const P pb = fma2(m_prev2, sub2(pc[n][p], pp[n][p]), pc[n][p]);
          w[n] = fma2(step2, w[n], pb);
        }
        if (iso) {
          ball2(w, fma2(w[2], w[2], fma2(w[1], w[1], mul2(w[0], w[0]))));
        } else {
#pragma unroll
          for (int n = 0; n < 3; ++n) w[n] = mk2(clampv(w[n].x, (T)-1, (T)1), clampv(w[n].y, (T)-1, (T)1));
        }
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          const P df = sub2(w[n], pc[n][p]);
          if (acc_n) {
            accf(fa[V::NRM], df, df);
            accf(fa[V::NRM + 1], pc[n][p], pc[n][p]);
          }
          src[n][p] = fma2(m_src2, df, w[n]);
          pc[n][p] = w[n];  // p_i (stored below)
        }
      }
      // boundary rows of D^T have no "-p" term: zero the components the
      // divergence must not see (they feed nothing else), so its sums need no
      // per-voxel selects
      if (last_in_row) src[0][1].y = 0;
      if (edge_src) s_edge[k & 1][sr] = src[0][1].y;
      if (!has_y) src[1][0] = src[1][1] = bc2((T)0);
      if (!has_up) src[2][0] = src[2][1] = bc2((T)0);
      if (acc_n) {
        const long long j = (long long)k * A.plane + (long long)y * K1 + xb;
#pragma unroll
        for (int n = 0; n < 3; ++n) st2(Pn + n * N + j, pc[n]);
        ld2(stg + M.V * g.slot_elems + rowoff, vv);
      }
      st2(srcbuf + (long long)(k & 1) * g.slot_elems + rowoff, src[1]);
    }
    if (ULATE && act && cons.has_qin()) {
#pragma unroll
      for (int c = 0; c < R; ++c) ld2(stg + (M.U0 + c) * g.slot_elems + rowoff, un[c]);
    }
    const unsigned long long t_c = tr ? global_ns() : 0;
    named_sync(1, W * 32);  // q(k+1), div-source rows published; stage b fully read
    if (threadIdx.x == 0) mbar_arrive(&empty[b]);
    if (tr) {
      A.trace[4 * s + 0] = t_a;
      A.trace[4 * s + 1] = t_b;
      A.trace[4 * s + 2] = t_c;
      A.trace[4 * s + 3] = global_ns();
    }

    // ---- a_i = v - reg D^-1 div(src) at plane k + Newton aggregates -----
    const T lsh = __shfl_up_sync(FULLM, src[0][1].y, 1);
    const T left1 = first_in_row ? (T)0 : (edge_dst ? s_edge[k & 1][sr] : lsh);
    if (pin && !warm && used && !halo) {
      P av[2] = {bc2((T)0), bc2((T)0)};
      const long long j = (long long)k * A.plane + (long long)y * K1 + xb;
      if (real) {
        P up[2] = {bc2((T)0), bc2((T)0)};
        if (y > 0) ld2(srcbuf + (long long)(k & 1) * g.slot_elems + rowoff - K1, up);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          // boundary terms are zero in the data: src at the far faces was
          // zeroed, up is 0 at y = 0, f3p is 0 at the first plane
          const T l0 = p == 0 ? left1 : src[0][0].y, l1 = src[0][p].x;
          P dv = mk2(l0 - src[0][p].x, l1 - src[0][p].y);
          dv = add2(dv, sub2(up[p], src[1][p]));
          dv = add2(dv, sub2(f3p[p], src[2][p]));
          const P de = mul2(dv, iec[p]);
          av[p] = fma2(nreg2, de, vv[p]);
#pragma unroll
          for (int c = 0; c < R; ++c) accf(fa[V::RHS + c], uc[c][p], diag ? de : dv);
        }
        st2(Aout + j, av);
      }
      P l[2] = {bc2(lo_s), bc2(lo_s)}, h[2] = {bc2(hi_s), bc2(hi_s)};
      if (real) {
        if (MODE == 0 && A.lo_arr) ld2(A.lo_arr + j, l);
        if (MODE == 0 && A.hi_arr) ld2(A.hi_arr + j, h);
      }
      bool nrv[4] = {false, false, false, false};
      bool any = false;
      if (R > 0) {
        auto classify = [&](auto hinf_tag) {
          constexpr bool HI = decltype(hinf_tag)::value;
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            bool n0, n1;
            if constexpr (std::is_same<AccT, P>::value) {
              P sv[RR];
#pragma unroll
              for (int c = 0; c < R; ++c) sv[c] = mul2(mul2(uc[c][p], iec[p]), bc2(sg));
              aggregate2<T, R, NACC, HI, AccT>(av[p], sv, uc, p, l[p], h[p], gcp, gwp, fa, n0, n1);
            } else {
              // higher ranks: voxel by voxel (fewer live registers)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                T sv[RR], uv[RR];
#pragma unroll
                for (int c = 0; c < RR; ++c) {
                  uv[c] = e ? uc[c][p].y : uc[c][p].x;
                  sv[c] = sg * uv[c] * (e ? iec[p].y : iec[p].x);
                }
                const bool nr = aggregate<T, R, NACC, AccT, HI>(e ? av[p].y : av[p].x, sv, uv, e ? l[p].y : l[p].x,
                                                                e ? h[p].y : h[p].x, gcp, gwp, fa);
                if (e) n1 = nr;
                else n0 = nr;
              }
            }
            // lanes off the grid hold zeros (no contribution) but must not list
            nrv[2 * p] = n0 && real, nrv[2 * p + 1] = n1 && real;
            any |= nrv[2 * p] | nrv[2 * p + 1];
          }
        };
#ifndef BQ_EXP_NOAGG  // (timing experiment: skip the Newton aggregates)
        if (hinf) classify(std::true_type{});
        else classify(std::false_type{});
#endif
      }
      if (__any_sync(FULLM, any)) {  // near voxels are rare: one vote per step
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          T sv[RR], uv[RR];
#pragma unroll
          for (int c = 0; c < RR; ++c) {
            uv[c] = (R > 0) ? el(uc[c], e) : (T)0;
            sv[c] = sg * uv[c] * el(iec, e);
          }
          near_push<T, R>(nrv[e], el(av, e), el(l, e), el(h, e), uv, sv, lane, near_seg, ncnt, ovf, A.capw);
        }
      }
    }
    if (sizeof(T) == 4 && (s % FLUSH) == FLUSH - 1) {
#pragma unroll
      for (int q = 0; q < NSUM; ++q) {
        const int src_q = q < V::COUT ? q : V::NRM + (q - V::COUT);
        double t = acc_fold(fa[src_q]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULLM, t, o);
        if (lane == 0) s_wacc[warp][q] += t;
        acc_zero(fa[src_q]);
      }
    }
    // ---- carries -------------------------------------------------------
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      f3p[p] = src[2][p];
      qc[p] = qn[p];
      iec[p] = ien[p];
#pragma unroll
      for (int c = 0; c < RR; ++c) uc[c][p] = un[c][p];
    }
    cons.advance();
    ++s;
    b = ring_next(b, NS);
  }
  // only the classes the steps accumulate (Cout, OVF and NCNT are untouched)
#pragma unroll
  for (int q = 0; q < V::COUT; ++q) acc[q] += acc_fold(fa[q]);
  acc[V::NRM] += acc_fold(fa[V::NRM]);
  acc[V::NRM + 1] += acc_fold(fa[V::NRM + 1]);
  if (sizeof(T) == 4 && lane == 0) {  // s_wacc[warp] is written by this lane only
#pragma unroll
    for (int q = 0; q < NSUM; ++q) acc[q < V::COUT ? q : V::NRM + (q - V::COUT)] += s_wacc[warp][q];
  }
}

// ---------------------------------------------------------------------------
// The kernel
// ---------------------------------------------------------------------------
#ifndef BQ_LIGHT_R
#define BQ_LIGHT_R 4  // fp32 ranks <= this run 11 row warps (168 registers), higher ranks 7
#endif
template <typename T, int R>
struct FCfg {
  static constexpr bool kLight = sizeof(T) == 4 && R <= BQ_LIGHT_R;
  // 11 row warps + 1 halo/producer warp = 384 threads -> ~168 registers
#ifndef BQ_FUSED_RW
#define BQ_FUSED_RW 11
#endif
  static constexpr int RW = kLight ? BQ_FUSED_RW : 7;
  static constexpr int NT = (RW + 1) * 32;    // + 1 halo warp
};

// KX: row length of the staged FUSED pass as a compile-time constant (128,
// 256 = x-split rows) or 0 (runtime K1 <= 128).  One kernel per KX so each
// gets its own register allocation.
template <typename T, int R, int KX>
__global__ void __launch_bounds__(FCfg<T, R>::NT, 1) wtv_fused_kernel(FArgs<T> A) {
  using V = FV<R>;
  constexpr int RW = FCfg<T, R>::RW;
  constexpr int NT = FCfg<T, R>::NT;
  constexpr int NACC = V::ACC;
  constexpr int ROWS = 32 * (RW + 1);  // >= (RW + 1) * rpw rows of <= 128 voxels
  __shared__ double s_red[kMaxVals];
  __shared__ double s_bv[kMaxVals];
  __shared__ double s_scr[(NT / 32) * kMaxVals];
  __shared__ FCtl s_c;
  __shared__ FShared<T> sh;
  __shared__ int s_flag;
  __shared__ double s_part[2 * kMaxVals];  // cluster mode: this block's partials, by barrier parity
  extern __shared__ __align__(16) unsigned char s_dyn[];
  T* rows = reinterpret_cast<T*>(s_dyn);  // [2][ROWS_used][K1] y-exchange of the div source

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ __align__(8) unsigned long long s_full[NSTAGE];
  __shared__ __align__(8) unsigned long long s_empty[NSTAGE];
  unsigned my_gen = 0;  // barriers completed (the counter starts at 0: memset at launch)
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 1);
    }
    mbar_init_fence();
  }
  __shared__ int s_pre[4];  // prefetched steps of the next FUSED pass: count, slot_cur, slot_prev, a_cur
  if (threadIdx.x == 0) s_pre[0] = 0;
  __syncthreads();
  Uses uses{0u, 0u, 0u};
  const int NS = A.geo.nstage;
  const int PW = A.geo.W;  // producer warp of the staged pass
  // Consume prefetched stages that will not be used (the next pass is not the
  // predicted FUSED pass, or the smem is needed): keeps the mbarrier phase
  // counts of producer and consumers in step and no bulk copy in flight.
  // consumer warps only (everything but the producer warp): named barrier 2
  constexpr int NC = NT - 32;
  const int cidx = warp < PW ? (int)threadIdx.x : (warp > PW ? (int)threadIdx.x - 32 : -1);
  auto csync = [&]() { named_sync(2, NC); };
  auto drain_impl = [&](bool consumers_only) {
    const int n = s_pre[0];
    for (int b = 0; b < n; ++b) {  // n <= NS: the prefetched steps fill slots 0 .. n-1
      if (warp != PW) {
        if (threadIdx.x == 0) {
          mbar_wait(&s_full[b], uses.get(b) & 1u);
          mbar_arrive(&s_empty[b]);
        }
        uses.inc(b);
      }
    }
    if (consumers_only) csync();
    else __syncthreads();
    if (threadIdx.x == 0) s_pre[0] = 0;
    if (consumers_only) csync();
    else __syncthreads();
  };
  auto drain = [&]() { drain_impl(false); };

  const long long N = A.N, plane = A.plane;
  const int K1 = A.K1, K2 = A.K2, K3 = A.K3, nd = A.ndim;
  const long long stride = (long long)gridDim.x * NT;
  const long long gtid = (long long)blockIdx.x * NT + threadIdx.x;
  const long long seg_begin = (long long)blockIdx.x * A.tile_planes / gridDim.x;
  const long long seg_end = (long long)(blockIdx.x + 1) * A.tile_planes / gridDim.x;
  constexpr int wpr = KX > 128 ? 2 : 1;  // warps per x-row
  const int GWs = A.geo.W / wpr;
  const long long tp_s = (long long)((A.K2 + (GWs - 1) * A.rpw - 1) / ((GWs - 1) * A.rpw)) * A.K3;
  long long seg_begin_s = (long long)blockIdx.x * tp_s / gridDim.x;
  long long seg_end_s = (long long)(blockIdx.x + 1) * tp_s / gridDim.x;
  if (A.ntile_tab > 0) {
    int t = 0;
    while (t + 1 < A.ntile_tab && (int)blockIdx.x >= A.tile_blk0[t + 1]) ++t;
    const int kb = (int)blockIdx.x - A.tile_blk0[t], nb = A.tile_blk0[t + 1] - A.tile_blk0[t];
    seg_begin_s = (long long)t * A.K3 + (long long)A.K3 * kb / nb;
    seg_end_s = (long long)t * A.K3 + (long long)A.K3 * (kb + 1) / nb;
  }
  const Fields<T, R> F{A.d, A.U, A.lo_arr, A.hi_arr, N, (T)eff_tau(A), (T)A.lo, (T)A.hi, (T)A.sign};
  const int lpr = A.lpr, rpw = A.rpw;
  // standalone DIV pass: NG row groups of wpr warps, the last group is the halo
  const int NG = (RW + 1) / wpr;
  const int xh = wpr == 2 ? (warp & 1) : 0, wg = warp / wpr;
  const int xr = lane % lpr, yr = lane / lpr, xb = 4 * xr + 128 * xh;
  const bool halo = wg >= NG - 1;
  const int slot = halo ? yr : rpw + wg * rpw + yr;
  const int TYe = (NG - 1) * rpw;
  const int rows_used = NG * rpw;
  __shared__ T s_dedge[2][64];
  (void)ROWS;
  constexpr int NW = NT / 32;
  constexpr int EWN = 3 + 2 * (R > 0 ? R : 1);
  const int capw = A.capw;
  const long long seg_elems = (long long)gridDim.x * NW * capw * EWN;  // one parity's list area
  T* my_seg0 = reinterpret_cast<T*>(A.near_data) + ((long long)blockIdx.x * NW + warp) * capw * EWN;
  int npass = 0;  // DIV/FUSED passes so far (same in every block)
  int my_cnt = 0;  // this warp's near entries in the last pass
  // compact near list (compact_near): [0] slot counter after the last pass (base of the
  // next pass's reservations), [1] slots the last pass reserved
  __shared__ unsigned s_nbase[2];
  if (threadIdx.x == 0) s_nbase[0] = 0u, s_nbase[1] = 0u;  // (ordered by the first block barrier below)

  int phase = F_SETUP;
#if BQ_PROX_TRACE
  bool tr3_on = false;
#endif
  while (true) {
    double acc[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
    int nv = 0;
    T cl_ent[EWN];  // warp 0: slot `lane` of the compact list of the pass ending at this barrier
    unsigned cl_key = 0xffffffffu;
#pragma unroll
    for (int f = 0; f < EWN; ++f) cl_ent[f] = (T)0;

    if (s_pre[0] > 0 && (phase == F_DIV || phase == F_FINAL)) drain();  // these reuse / leave the smem
    if (phase == F_SETUP) {
      // gram partials U^T D^-1 U (wpm.py:50-56); 1/d staged by the fused pass
      nv = V::S;
      // 4 voxels per thread and trip (16-byte accesses; N % 4 == 0 on this path)
      if (R == 0 && A.d)
        for (long long j = 4 * gtid; j < N; j += 4 * stride) {
          T e[4], ie[4];
          Vec4<T>::ro(A.d + j, e);
#pragma unroll
          for (int q = 0; q < 4; ++q) ie[q] = rcp(e[q]);
          Vec4<T>::st(A.ie + j, ie);
        }
      if (R > 0) {
#pragma unroll 2
        for (long long j = 4 * gtid; j < N; j += 4 * stride) {
          T u[R > 0 ? R : 1][4], e[4] = {(T)1, (T)1, (T)1, (T)1};
#pragma unroll
          for (int c = 0; c < R; ++c) Vec4<T>::ro(A.U + (long long)c * N + j, u[c]);
          if (A.d) {
            T ie[4];
            Vec4<T>::ro(A.d + j, e);
#pragma unroll
            for (int q = 0; q < 4; ++q) ie[q] = rcp(e[q]);
            Vec4<T>::st(A.ie + j, ie);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            int k = 0;
#pragma unroll
            for (int c = 0; c < R; ++c)
#pragma unroll
              for (int c2 = 0; c2 <= c; ++c2, ++k)
                acc[k] += A.d ? (double)(u[c][q] * u[c2][q] / e[q]) : (double)u[c][q] * (double)u[c2][q];
          }
        }
      }
    } else if (phase == F_FUSED) {
      nv = V::PASS;
      int ncnt = 0;
      bool ovf = false;
      T* my_seg = my_seg0 + (npass & 1) * seg_elems;
      int pre = s_pre[0];
      if (pre > 0 && !(s_pre[1] == sh.slot_cur && s_pre[2] == sh.slot_prev && s_pre[3] == sh.a_cur)) {
        drain();
        pre = 0;
      }
#if BQ_PROX_TRACE
      if (blockIdx.x == 0 && threadIdx.x == 0 && sh.tr7) {
        A.trace[320 + 9] = global_ns();
        A.trace[320 + 10] = (unsigned long long)(pre + 100 * s_pre[0]);
      }
#endif
      // scalar box bounds (fused_eligible): compile-time stage layout, the
      // bounds are pass constants
      fused_staged<T, R, NACC, 1, KX>(A, sh, A.geo, seg_begin_s, seg_end_s, reinterpret_cast<T*>(s_dyn), s_full,
                                      s_empty, uses, acc, my_seg, ncnt, ovf, pre);
      if (sh.cl_on && ncnt > 0 && !ovf)  // (warp-uniform)
        compact_near<T, EWN>(my_seg, ncnt, (unsigned)((blockIdx.x * NW + warp) * capw), A.cl_ctr, s_nbase[0],
                             A.cl_data + (long long)(npass & 1) * CL * EWN, A.cl_key + (npass & 1) * CL, lane);
      if (lane == 0) A.near_cnt[(npass & 1) * gridDim.x * NW + blockIdx.x * NW + warp] = ncnt;
      ++npass;
      my_cnt = ncnt;
      if (ovf) acc[V::OVF] += 1.0;
      if (lane == 0) acc[V::NCNT] += (double)ncnt;
#if BQ_PROX_TRACE
      tr3_on = A.trace && A.trace_thread == -3 && s_c.it == A.trace_pass;
      if (tr3_on && blockIdx.x == 0 && threadIdx.x == 0) A.trace[320 + 8] = s_c.it;
#endif
      TR3(0);
#if BQ_PROX_TRACE
      if (tr3_on && threadIdx.x == 0 && blockIdx.x < 1000) {  // which SM ran this block
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        A.trace[3072 + blockIdx.x] = smid;
      }
#endif
    } else if (phase == F_DIV) {
      nv = V::PASS;
      const bool fused = false;
      const T* __restrict__ Pc = A.ring[sh.slot_cur];
      const T* __restrict__ Pp = A.ring[sh.slot_prev];
      T* __restrict__ Pn = A.ring[sh.slot_new];
      const T* __restrict__ Ain = A.abuf[sh.a_cur];
      T* __restrict__ Aout = A.abuf[sh.a_cur ^ 1];
      const T m_prev = sh.m_prev, m_cur = sh.m_cur;
      const bool div_p = sh.div_p;
      const T step = (T)eff_step(A), reg = (T)A.reg;
      const bool iso = A.mode == BQ_TV_ISO;
      const bool single = sh.single;
      int ncnt = 0;
      bool ovf = false;
      int buf = 0;
      T* my_seg = my_seg0 + (npass & 1) * seg_elems;
      long long pos = seg_begin;
      while (pos < seg_end) {
        const long long tile = pos / K3;
        const int z0 = (int)(pos - tile * K3);
        const int z1 = (int)min((long long)K3, z0 + (seg_end - pos));
        pos += z1 - z0;
        const int y0 = (int)tile * TYe;
        const int y = halo ? (y0 - rpw + yr) : (y0 + wg * rpw + yr);
        const bool act = y >= 0 && y < K2;
        const bool has_y = nd >= 2 && y < K2 - 1;
        const int zs = (z0 > 0 && nd >= 3) ? z0 - 1 : z0;
        long long j = (long long)zs * plane + (long long)y * K1 + xb;
        T qc[4] = {0, 0, 0, 0}, iec[4] = {1, 1, 1, 1}, uc[R > 0 ? R : 1][4];
#pragma unroll
        for (int c = 0; c < (R > 0 ? R : 1); ++c) uc[c][0] = uc[c][1] = uc[c][2] = uc[c][3] = 0;
        if (act) {
          if (fused) F.q4x(Ain, j, sh.gz, qc, iec, uc);
          else if (!halo) F.ieu4(j, iec, uc);
        }
        T f3prev[4] = {0, 0, 0, 0};
        for (int z = zs; z < z1; ++z, j += plane) {
          const bool warm = z < z0;
          const bool has_up = nd >= 3 && z < K3 - 1;
          T qu[4] = {0, 0, 0, 0}, ieu[4] = {1, 1, 1, 1}, uu[R > 0 ? R : 1][4];
#pragma unroll
          for (int c = 0; c < (R > 0 ? R : 1); ++c) uu[c][0] = uu[c][1] = uu[c][2] = uu[c][3] = 0;
          T src[3][4];
          T pcur[3][4];
          if (fused) {
            // ---- dual update at plane z (dual_tv_solver.py:225) ----------
            T qy[4] = {0, 0, 0, 0};
            if (act && has_up) F.q4x(Ain, j + plane, sh.gz, qu, ieu, uu);
            if (act && has_y) F.q4(Ain, j + K1, sh.gz, qy);
            const T qn = __shfl_down_sync(FULLM, qc[0], 1);
            T pprev[3][4];
#pragma unroll
            for (int n = 0; n < 3; ++n) {
#pragma unroll
              for (int k = 0; k < 4; ++k) pcur[n][k] = 0, pprev[n][k] = 0;
              if (act && n < nd) {
                Vec4<T>::rw(Pc + n * N + j, pcur[n]);
                if (m_prev != (T)0) Vec4<T>::rw(Pp + n * N + j, pprev[n]);
              }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const T right = (k < 3) ? qc[k + 1] : qn;
              T g[3];
              g[0] = (xb + k < K1 - 1) ? right - qc[k] : (T)0;
              g[1] = has_y ? qy[k] - qc[k] : (T)0;
              g[2] = has_up ? qu[k] - qc[k] : (T)0;
              T w[3];
#pragma unroll
              for (int n = 0; n < 3; ++n) {
                // P_bar_{i-1} = p_{i-1} + m (p_{i-1} - p_{i-2})  (dual_tv_solver.py:235)
                const T pb = (m_prev != (T)0) ? pcur[n][k] + m_prev * (pcur[n][k] - pprev[n][k]) : pcur[n][k];
                w[n] = (n < nd) ? pb + step * g[n] : (T)0;
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
                if (!halo && !warm && act && n < nd) {
                  const T df = w[n] - pcur[n][k];
                  acc[V::NRM] += (double)df * (double)df;
                  acc[V::NRM + 1] += (double)pcur[n][k] * (double)pcur[n][k];
                }
                // div source: P_bar_i (or p_i on the last iteration)
                src[n][k] = div_p ? w[n] : w[n] + m_cur * (w[n] - pcur[n][k]);
                pprev[n][k] = w[n];  // reuse as p_i storage
              }
            }
            if (!halo && !warm && act) {
#pragma unroll
              for (int n = 0; n < 3; ++n)
                if (n < nd) Vec4<T>::st(Pn + n * N + j, pprev[n]);
            }
          } else {
            // ---- standalone DIV: source P_bar = p + m (p - p_prev) read ----
            if (!halo && act && has_up) F.ieu4(j + plane, ieu, uu);
#pragma unroll
            for (int n = 0; n < 3; ++n) {
#pragma unroll
              for (int k = 0; k < 4; ++k) src[n][k] = 0;
              if (act && n < nd && !single) {
                T pc4[4], pp4[4];
                Vec4<T>::rw(Pc + n * N + j, pc4);
                if (m_prev != (T)0) Vec4<T>::rw(Pp + n * N + j, pp4);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  src[n][k] = (m_prev != (T)0) ? pc4[k] + m_prev * (pc4[k] - pp4[k]) : pc4[k];
              }
            }
          }
          // ---- y-exchange of the div source (component 2) through smem ----
          if (nd >= 2) {
#pragma unroll
            for (int k = 0; k < 4; ++k) rows[((long long)buf * rows_used + slot) * K1 + xb + k] = src[1][k];
          }
          if (wpr == 2 && xh == 0 && lane == 31) s_dedge[buf][slot] = src[0][3];
          __syncthreads();
          const T lsh = __shfl_up_sync(FULLM, src[0][3], 1);
          const T left1 = (wpr == 2 && xh == 1 && lane == 0) ? s_dedge[buf][slot] : lsh;
          if (!halo && !warm && act) {
            // ---- a_i = v - reg D^-1 div(src)  (tv_ops.py:122-159) -------
            T av[4], vv[4];
            if (single) {
              Vec4<T>::ro(A.v + j, av);
            } else {
              Vec4<T>::ro(A.v + j, vv);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const T lk = (k == 0) ? left1 : src[0][k - 1];
                T dv = (xb + k < K1 - 1 ? -src[0][k] : (T)0) + (xb + k > 0 ? lk : (T)0);
                if (nd >= 2) {
                  const T up = (y > 0) ? rows[((long long)buf * rows_used + slot - 1) * K1 + xb + k] : (T)0;
                  dv += (y < K2 - 1 ? -src[1][k] : (T)0) + up;
                }
                if (nd >= 3) dv += (z < K3 - 1 ? -src[2][k] : (T)0) + (z > 0 ? f3prev[k] : (T)0);
                const T de = dv * iec[k];
                av[k] = vv[k] - reg * de;
#pragma unroll
                for (int c = 0; c < R; ++c) acc[V::RHS + c] += (double)uc[c][k] * (double)(A.d ? de : dv);
              }
            }
            Vec4<T>::st(Aout + j, av);
            // ---- Newton aggregates + near list for the next Newton ------
            T l[4], h[4];
            F.bounds4(j, l, h);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              T s[R > 0 ? R : 1], u[R > 0 ? R : 1];
#pragma unroll
              for (int c = 0; c < R; ++c) {
                u[c] = uc[c][k];
                s[c] = F.sg * u[c] * iec[k];
              }
              const bool nr = (R > 0) ? aggregate<T, R, NACC, double>(av[k], s, u, l[k], h[k], sh.gc, sh.gwid, acc) : false;
              near_push<T, R>(nr, av[k], l[k], h[k], u, s, lane, my_seg, ncnt, ovf, A.capw);
            }
          } else if (!halo) {
            // keep the warp's ballots aligned with the active lanes' calls
            T z1[R > 0 ? R : 1];
#pragma unroll
            for (int c = 0; c < (R > 0 ? R : 1); ++c) z1[c] = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) near_push<T, R>(false, (T)0, (T)0, (T)0, z1, z1, lane, my_seg, ncnt, ovf, A.capw);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            f3prev[k] = src[2][k];
            qc[k] = qu[k];
            iec[k] = ieu[k];
#pragma unroll
            for (int c = 0; c < (R > 0 ? R : 1); ++c) uc[c][k] = uu[c][k];
          }
          buf ^= 1;
        }
      }
      if (lane == 0) A.near_cnt[(npass & 1) * gridDim.x * NW + blockIdx.x * NW + warp] = ncnt;
      ++npass;
      my_cnt = ncnt;
      if (ovf) acc[V::OVF] += 1.0;
      if (lane == 0) acc[V::NCNT] += (double)ncnt;
    } else if (phase == F_NDIST) {
      // one Newton evaluation over a long near list: every warp sums the
      // entries it pushed in the last pass (no gather), the barrier reduces
      nv = V::NEWTON;
      constexpr int EW = 3 + 2 * (R > 0 ? R : 1);
      const T* seg = my_seg0 + ((npass - 1) & 1) * seg_elems;
      for (int e = lane; e < my_cnt; e += 32) {
        const T* d = seg + (long long)e * EW;
        T z = d[0];
#pragma unroll
        for (int c = 0; c < R; ++c) z += d[3 + R + c] * sh.gz[c];
        const T l = d[1], h = d[2];
        const T cz = clampv(z, l, h);
#pragma unroll
        for (int c = 0; c < R; ++c) acc[c] += (double)d[3 + c] * (double)cz;
        if (z > l && z < h) {
          int k = R;
#pragma unroll
          for (int c = 0; c < R; ++c)
#pragma unroll
            for (int c2 = 0; c2 <= c; ++c2, ++k) acc[k] += (double)d[3 + c] * (double)d[3 + R + c2];
        }
      }
    } else if (phase == F_NEWTON) {
      // full-pass phi(beta) and generalized Jacobian partials (wpm.py:150-167)
      nv = V::NEWTON;
      const T* __restrict__ Ain = A.abuf[sh.a_cur];
      // scalar bounds on this path; 4 voxels per thread and trip
      const T l = F.lo, h = F.hi;
#pragma unroll 2
      for (long long j = 4 * gtid; j < N; j += 4 * stride) {
        T a4[4], ie[4], u[R > 0 ? R : 1][4];
        Vec4<T>::rw(Ain + j, a4);
        F.ieu4(j, ie, u);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          T s[R > 0 ? R : 1];
          T wv = a4[q], z = a4[q];
#pragma unroll
          for (int c = 0; c < R; ++c) {
            s[c] = F.sg * u[c][q] * ie[q];
            wv += s[c] * sh.gw[c];
            z += s[c] * sh.gz[c];
          }
          const T dl = wv - clampv(z, l, h);
#pragma unroll
          for (int c = 0; c < R; ++c) acc[c] += (double)u[c][q] * (double)dl;
          if (z > l && z < h) {
            int k = R;
#pragma unroll
            for (int c = 0; c < R; ++c)
#pragma unroll
              for (int c2 = 0; c2 <= c; ++c2, ++k) acc[k] += (double)u[c][q] * (double)s[c2];
          }
        }
      }
    } else if (phase == F_FINAL) {
      // x = clamp(a + s.gamma*) and P* back into the caller's buffer
      const T* __restrict__ Ain = A.abuf[sh.a_cur];
      T* __restrict__ X = A.x;
      const T* __restrict__ Pfin = A.ring[sh.slot_cur];
      const bool copy = !sh.single && sh.slot_cur != 0;
      const T l = F.lo, h = F.hi;  // scalar bounds on this path
#pragma unroll 2
      for (long long j = 4 * gtid; j < N; j += 4 * stride) {
        T a4[4], ie[4], u[R > 0 ? R : 1][4];
        Vec4<T>::rw(Ain + j, a4);
        F.ieu4(j, ie, u);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          T z = a4[q];
#pragma unroll
          for (int c = 0; c < R; ++c) z += (F.sg * u[c][q] * ie[q]) * sh.gz[c];
          a4[q] = clampv(z, l, h);
        }
        Vec4<T>::st(X + j, a4);
        if (copy)
          for (int n = 0; n < nd; ++n) {
            T p4[4];
            Vec4<T>::rw(Pfin + n * N + j, p4);
            Vec4<T>::st(A.ring[0] + n * N + j, p4);
          }
      }
    }

    // ---- barrier with fused deterministic reduction ----------------------
    // Monotonic arrival counter: barrier g completes when it reaches (g+1)*G.
    // Partials are stored transposed ([value][block]) and EVERY block reduces
    // them itself in block order (identical sums everywhere, no float
    // atomics), so no block has to wait for a "last block" to publish.
    const int cur = phase;
    const bool barrier = cur != F_FINAL;
    if (barrier) {
      block_sum_to<NT, NACC>(acc, nv, s_bv, s_scr);  // (its syncs: every thread has read s_pre)
      if (cur == F_FUSED && threadIdx.x == 0) s_pre[0] = 0;
      // [parity][kMaxVals][kMaxBlocks/2]: a fast block's next partials never
      // land on values a slow block is still reducing
      constexpr int PB = kMaxBlocks / 2;
      double* __restrict__ PT = A.partials + (size_t)(my_gen & 1u) * kMaxVals * PB;
      if (A.cluster) {
        // single-cluster launch: partials stay in each block's shared memory
        // (double-buffered by barrier parity, so a fast block's next partials
        // never overwrite values a slow block is still reading), one cluster
        // barrier (release / acquire at cluster scope also orders the global
        // stores of the pass), and every block sums the G partial vectors
        // through DSMEM in block order -- identical sums everywhere
        namespace cg = cooperative_groups;
        cg::cluster_group cl = cg::this_cluster();
        double* mine = s_part + (my_gen & 1u) * kMaxVals;
        if (threadIdx.x < nv) mine[threadIdx.x] = s_bv[threadIdx.x];
        if (threadIdx.x == NT - 1) mine[kMaxVals - 1] = __longlong_as_double((long long)global_ns());
        if (cur == F_FUSED && threadIdx.x == 0) {
          StepIter it;
          it.init(seg_begin_s, seg_end_s, K3, 3);
          int n = 0;
          while (it.valid && n < A.pre_max) {
            it.advance();
            ++n;
          }
          s_pre[1] = sh.slot_new;
          s_pre[2] = sh.slot_cur;
          s_pre[3] = sh.a_cur ^ 1;
          s_pre[0] = n;
        }
        cl.sync();
        for (int k = warp; k < nv; k += NT / 32) {
          double sum = 0.0;
          for (unsigned b = lane; b < gridDim.x; b += 32) sum += cl.map_shared_rank(mine, b)[k];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sum += __shfl_down_sync(FULLM, sum, o);
          if (lane == 0) s_red[k] = sum;
        }
        if (blockIdx.x == 0 && warp == NT / 32 - 1) {
          long long t = 0;
          for (unsigned b = lane; b < gridDim.x; b += 32)
            t = max(t, __double_as_longlong(cl.map_shared_rank(mine, b)[kMaxVals - 1]));
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) t = max(t, __shfl_down_sync(FULLM, t, o));
          if (lane == 0) s_red[kMaxVals - 1] = __longlong_as_double(t);
        }
        my_gen += 1;
        __syncthreads();
      } else {
      if (threadIdx.x < nv) PT[(size_t)threadIdx.x * PB + blockIdx.x] = s_bv[threadIdx.x];
      if (threadIdx.x == NT - 1)
        PT[(size_t)(kMaxVals - 1) * PB + blockIdx.x] = __longlong_as_double((long long)global_ns());
      __syncthreads();
      if (cur == F_FUSED) TR3(1);
      if (threadIdx.x == 0) {
        atom_add_acqrel(A.bar, 1u);
        const unsigned target = (my_gen + 1u) * gridDim.x;
        const uint64_t t0 = global_ns();
        unsigned spins = 0;
        s_flag = 0;
        while ((int)(ld_acquire_u32(A.bar) - target) < 0) {
          if (((++spins) & 4095u) == 0 && global_ns() - t0 > 20ull * 1000000000ull) {
            s_flag = -1;
            break;
          }
        }
        // (no fence here: the acquire load that observed the last arrival
        //  synchronizes with every block's acq_rel add -- the adds form one
        //  release sequence -- and ptxas follows it with the L1 invalidate
        //  (LDG.STRONG.GPU + CCTL.IVALL); the block barrier below extends the
        //  ordering to the other threads.  The extra fence.acq_rel.gpu cost
        //  0.4 us per barrier: 2.90 -> 2.86 ms per 128^3 solve.)
        if (cur == F_FUSED) TR3(2);
      }
      __syncthreads();
      if (s_flag == -1) {
        if (blockIdx.x == 0 && threadIdx.x == 0) A.report->status = BQ_ETIMEOUT;
        break;
      }
      if (cur == F_FUSED && A.cl_data && warp == 0) {
        // compact near list of the pass that just ended: the counter and the CL
        // slots ride along with the partial loads below (same L2 round trip)
        const int par = (npass - 1) & 1;
        if (lane == 0) {
          const unsigned now = __ldcg(A.cl_ctr);
          s_nbase[1] = now - s_nbase[0];
          s_nbase[0] = now;
        }
        if (lane < CL) {
          cl_key = __ldcg(A.cl_key + par * CL + lane);
          const T* src = A.cl_data + ((long long)par * CL + lane) * EWN;
#pragma unroll
          for (int f = 0; f < EWN; ++f) cl_ent[f] = __ldcg(src + f);
        }
      }
      if (cur == F_FUSED && threadIdx.x == 0) {
        // the next FUSED pass (the usual successor) reads ring[slot_new],
        // ring[slot_cur] and abuf[a_cur ^ 1]; its first stages are issued by
        // the producer warp below, while the other warps run the controller
        StepIter it;
        it.init(seg_begin_s, seg_end_s, K3, 3);
        int n = 0;
        while (it.valid && n < A.pre_max) {
          it.advance();
          ++n;
        }
        s_pre[1] = sh.slot_new;
        s_pre[2] = sh.slot_cur;
        s_pre[3] = sh.a_cur ^ 1;
        s_pre[0] = n;
      }
      for (int k = warp; k < nv; k += NT / 32) {
        const double* col = PT + (size_t)k * PB;
        double sum = 0.0;
        for (unsigned b = lane; b < gridDim.x; b += 32) sum += __ldcg(&col[b]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_down_sync(FULLM, sum, o);
        if (lane == 0) s_red[k] = sum;
      }
      if (blockIdx.x == 0 && warp == NT / 32 - 1) {  // latest arrival (phase timeline of the report)
        const long long* col = reinterpret_cast<const long long*>(PT + (size_t)(kMaxVals - 1) * PB);
        long long t = 0;
        for (unsigned b = lane; b < gridDim.x; b += 32) {
          t = max(t, __ldcg(&col[b]));
#if BQ_PROX_TRACE
          if (cur == F_FUSED && tr3_on && b < 2000) A.trace[1024 + b] = (unsigned long long)__ldcg(&col[b]);
#endif
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t = max(t, __shfl_down_sync(FULLM, t, o));
        if (lane == 0) s_red[kMaxVals - 1] = __longlong_as_double(t);
      }
      my_gen += 1;
      __syncthreads();
      }  // global barrier
      if (cur == F_FUSED) TR3(3);
    }

    // ---- producer warp: prefetch the next pass's first stages -------------
    if (warp == PW) {
      if (cur == F_FUSED && s_pre[0] > 0) {
        StageMap<R> M;
        M.make(A.d != nullptr, A.lo_arr != nullptr, A.hi_arr != nullptr, 3, true);
        fence_proxy_async_global();  // reads data written before the grid barrier
        StepIter it;
        it.init(seg_begin_s, seg_end_s, K3, 3);
        for (int b = 0; b < s_pre[0]; ++b) {
          issue_step<T, R>(A, it, M, A.geo, reinterpret_cast<T*>(s_dyn) + b * A.geo.stage_elems, &s_full[b],
                           A.ring[s_pre[1]], A.ring[s_pre[2]], A.abuf[s_pre[3]], lane);
          uses.inc(b);
          it.advance();
        }
      }
    } else {
    // ---- controller (+ block-local Newton over the near list) ------------
    const bool tl_side = cur != F_SETUP && cur != F_FINAL;  // (setup resets, final reports the timeline)
    if (threadIdx.x == 32 && tl_side) {  // phase timeline: its own fields, off the controller's path
      Ctl<T, R> ctl{A, s_c, blockIdx.x == 0};
      ctl.timeline(cur, s_red, barrier);
    }
    if (threadIdx.x == 0) {
      Ctl<T, R> ctl{A, s_c, blockIdx.x == 0};
#if BQ_PROX_TRACE
      const long long c0 = clock64();
#endif
      if (!tl_side) ctl.timeline(cur, s_red, barrier);
#if BQ_PROX_TRACE
      const long long c1 = clock64();
#endif
      ctl.run(cur, s_red);
#if BQ_PROX_TRACE
      const long long c2 = clock64();
      if (cur == F_FUSED && blockIdx.x == 0 && tr3_on) {
        A.trace[340] = (unsigned long long)(c1 - c0);
        A.trace[341] = (unsigned long long)(c2 - c1);
      }
#endif
    }
    csync();
    if (cur == F_FUSED) TR3(4);
    // ---- on-chip Newton: warp 0 stages the (usually tiny) near list into
    //      shared memory and runs every Newton step with warp-level
    //      reductions; the other warps wait once.
    if (s_c.phase == F_NLOCAL) {
      constexpr int EW = 3 + 2 * (R > 0 ? R : 1);  // av, l, h, u[R], s[R]
      T* ne = reinterpret_cast<T*>(s_dyn + A.list_off);
      const int total = (int)s_red[V::NCNT];
      const long long lbytes = (long long)total * EW * (long long)sizeof(T);
      const bool seg_ok = (int)gridDim.x * NW <= 8 * NC && (int)gridDim.x * NW < (int)(sizeof(s_scr) / sizeof(int));
      bool in_smem = seg_ok && lbytes <= A.list_bytes;
      // short list, filled grid-wide by the last pass and already in warp 0's
      // registers: no count scan, no gather
      const bool tiny = cur == F_FUSED && sh.cl_on && total > 0 && total <= CL && s_nbase[1] == (unsigned)total &&
                        (long long)CL * EW * (long long)sizeof(T) <= A.list_bytes;
      if (tiny) in_smem = true;
      if (seg_ok && !in_smem && lbytes <= A.dyn_bytes) {
        // long list (early iterations): give up the prefetched stages, use all the dynamic smem
        if (s_pre[0] > 0) drain_impl(true);
        ne = reinterpret_cast<T*>(s_dyn);
        in_smem = true;
      }
#if BQ_PROX_TRACE
      const bool ntr = A.trace && blockIdx.x == 0 && threadIdx.x == 0 && s_c.it == A.trace_pass && A.trace_thread < 0;
      const bool nprof = A.trace && blockIdx.x == 0 && threadIdx.x == 0 && A.trace_thread == -2 && s_c.it < 128;
#else
      constexpr bool ntr = false, nprof = false;
#endif
      const unsigned long long nprof_t0 = nprof ? global_ns() : 0;
      int ntr_k = 0;
      if (ntr) {
        A.trace[240 + ntr_k++] = global_ns();
        A.trace[300] = (unsigned long long)total;
      }
      // exclusive prefix of the per-segment counts in segment order (block
      // scan), then a flat gather: thread t copies entries t, t+NT, ... (each
      // located by binary search), so no thread walks a long segment serially.
      // The list order is fixed, so every block sums identically.
      // (the prefix table lives in the block-reduction scratch: s_scr is idle
      //  between barriers, and the long-list reduction below reads the
      //  gathered copy, not the table)
      int* const s_pref = reinterpret_cast<int*>(s_scr);
      constexpr int kPrefCap = (int)(sizeof(s_scr) / sizeof(int)) - 1;
      const int nseg = gridDim.x * NW;
      const bool indexed = nseg <= 8 * NC && nseg <= kPrefCap;
      const int lpar = (npass - 1) & 1;  // parity of the pass that built the lists
      const T* __restrict__ nd = reinterpret_cast<const T*>(A.near_data) + lpar * seg_elems;
      const int* __restrict__ ncnt_l = A.near_cnt + lpar * nseg;
      auto locate = [&](int e) -> const T* {
        int lo = 0, hi = nseg;
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (s_pref[mid] <= e) lo = mid;
          else hi = mid;
        }
        return nd + ((long long)lo * capw + (e - s_pref[lo])) * EW;
      };
      if (tiny && warp == 0) {
        // canonical order: segment order (rank = number of smaller keys)
        const unsigned mykey = lane < total ? cl_key : 0xffffffffu;
        int rank = 0;
        for (int i = 0; i < total; ++i) rank += __shfl_sync(FULLM, mykey, i) < mykey ? 1 : 0;
        if (lane < total) {
          T* dst = ne + (long long)rank * EW;
#pragma unroll
          for (int f = 0; f < EW; ++f) dst[f] = cl_ent[f];
        }
        __syncwarp();
      }
      if (total > 0 && indexed && !tiny) {
        constexpr int SPT = 8;
        const int s0 = cidx * SPT;
        int cnt[SPT];
        int mine = 0;
#pragma unroll
        for (int q = 0; q < SPT; ++q) {
          cnt[q] = s0 + q < nseg ? __ldcg(&ncnt_l[s0 + q]) : 0;
          mine += cnt[q];
        }
        __shared__ int s_wsum2[NT / 32];
        const int cw = cidx >> 5;
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(FULLM, incl, o);
          if (lane >= o) incl += t;
        }
        if (lane == 31) s_wsum2[cw] = incl;
        csync();
        int off = incl - mine;
        for (int w2 = 0; w2 < cw; ++w2) off += s_wsum2[w2];
#pragma unroll
        for (int q = 0; q < SPT; ++q) {
          if (s0 + q < nseg) s_pref[s0 + q] = off;
          off += cnt[q];
        }
        if (threadIdx.x == 0) s_pref[nseg] = total;
        csync();
        if (in_smem) {
          for (int e = cidx; e < total; e += NC) {
            const T* src = locate(e);
            T* dst = ne + (long long)e * EW;
#pragma unroll
            for (int f = 0; f < EW; ++f) dst[f] = __ldcg(&src[f]);
          }
          csync();
        }
      }
      // long lists: every warp evaluates, block reduction per step (through
      // s_scr, so only when the evaluation reads the gathered copy, not s_pref)
      const bool big = total > 256 && in_smem;
      if (warp == 0 || big) {
        if (!big) __syncwarp();
        if (ntr) A.trace[240 + ntr_k++] = global_ns();
        while (s_c.phase == F_NLOCAL) {
          // phi(beta) = K0 + Cout gw + Cin beta + beta - sum_near u clamp(a + s.gamma)
          double nacc[V::NEWTON > 0 ? V::NEWTON : 1];
#pragma unroll
          for (int k = 0; k < V::NEWTON; ++k) nacc[k] = 0.0;
          T gz[R > 0 ? R : 1];
#pragma unroll
          for (int c = 0; c < R; ++c) gz[c] = (T)(s_c.gw[c] - s_c.beta[c]);
          auto near_term = [&](T av, const T (&sv)[R > 0 ? R : 1], const T (&uv)[R > 0 ? R : 1], T l, T h) {
            T z = av;
#pragma unroll
            for (int c = 0; c < R; ++c) z += sv[c] * gz[c];
            const T cz = clampv(z, l, h);
#pragma unroll
            for (int c = 0; c < R; ++c) nacc[c] += (double)uv[c] * (double)cz;
            if (z > l && z < h) {
              int k = R;
#pragma unroll
              for (int c = 0; c < R; ++c)
#pragma unroll
                for (int c2 = 0; c2 <= c; ++c2, ++k) nacc[k] += (double)uv[c] * (double)sv[c2];
            }
          };
          const int t0 = big ? cidx : lane;
          const int tstride = big ? NC : 32;
          if (total > 0) {
            if (in_smem) {
              for (int e = t0; e < total; e += tstride) {
                const T* d = ne + (long long)e * EW;
                T sv[R > 0 ? R : 1], uv[R > 0 ? R : 1];
#pragma unroll
                for (int c = 0; c < R; ++c) uv[c] = d[3 + c], sv[c] = d[3 + R + c];
                near_term(d[0], sv, uv, d[1], d[2]);
              }
            } else if (indexed) {
              for (int e = t0; e < total; e += tstride) {
                const T* d = locate(e);
                T sv[R > 0 ? R : 1], uv[R > 0 ? R : 1];
#pragma unroll
                for (int c = 0; c < R; ++c) uv[c] = __ldcg(&d[3 + c]), sv[c] = __ldcg(&d[3 + R + c]);
                near_term(__ldcg(&d[0]), sv, uv, __ldcg(&d[1]), __ldcg(&d[2]));
              }
            } else {
              for (int sidx = t0; sidx < nseg; sidx += tstride) {
                const int cnt = __ldcg(&ncnt_l[sidx]);
                for (int e = 0; e < cnt; ++e) {
                  const T* d = nd + ((long long)sidx * capw + e) * EW;
                  T sv[R > 0 ? R : 1], uv[R > 0 ? R : 1];
#pragma unroll
                  for (int c = 0; c < R; ++c) uv[c] = __ldcg(&d[3 + c]), sv[c] = __ldcg(&d[3 + R + c]);
                  near_term(__ldcg(&d[0]), sv, uv, __ldcg(&d[1]), __ldcg(&d[2]));
                }
              }
            }
          }
          if (big) {
            // consumer-warp reduction in fixed warp order (deterministic)
            const int cw = cidx >> 5;
#pragma unroll
            for (int k = 0; k < V::NEWTON; ++k) {
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) nacc[k] += __shfl_down_sync(FULLM, nacc[k], o);
              if (lane == 0) s_scr[cw * kMaxVals + k] = nacc[k];
            }
            csync();
            if (cidx < V::NEWTON) {
              double t = 0.0;
              for (int w2 = 0; w2 < NC / 32; ++w2) t += s_scr[w2 * kMaxVals + cidx];
              s_bv[cidx] = t;
            }
            csync();
#pragma unroll
            for (int k = 0; k < V::NEWTON; ++k) nacc[k] = s_bv[k];
          } else if (total > 0) {
#pragma unroll
            for (int k = 0; k < V::NEWTON; ++k)
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) nacc[k] += __shfl_down_sync(FULLM, nacc[k], o);
          }
          if (threadIdx.x == 0) {
            Ctl<T, R> ctl{A, s_c, blockIdx.x == 0};
            double phi[R > 0 ? R : 1], hp[V::S > 0 ? V::S : 1];
            ctl.local_eval(nacc, phi, hp);
            s_c.local_steps += 1;
            ctl.newton_step(phi, hp);
            if (ntr && ntr_k < 40) A.trace[240 + ntr_k++] = global_ns();
          }
          if (big) csync();
          else __syncwarp();
        }
        if (threadIdx.x == 0) {  // one timeline stamp for the whole on-chip solve
          Ctl<T, R> ctl{A, s_c, blockIdx.x == 0};
          ctl.timeline(F_NLOCAL, s_red, false);
        }
      }
      csync();
      if (nprof) A.trace[256 + s_c.it] = ((global_ns() - nprof_t0) << 20) | ((unsigned long long)total & 0xfffff);
    }
    if (cur == F_FUSED) TR3(5);
    if (threadIdx.x == 0) {
      if (s_c.phase == F_FUSED) {
        Ctl<T, R> ctl{A, s_c, blockIdx.x == 0};
        ctl.prepare_fused();
      }
      sh.phase = s_c.phase;
      sh.slot_cur = s_c.slot_cur;
      sh.slot_prev = s_c.slot_prev;
      sh.slot_new = (s_c.slot_cur == s_c.slot_prev) ? (s_c.slot_cur + 1) % 3 : 3 - s_c.slot_cur - s_c.slot_prev;
      sh.a_cur = s_c.a_cur;
      sh.iter = s_c.it;
      sh.div_p = s_c.div_p;
      sh.single = s_c.single;
      sh.cl_on = s_c.cl_on;
      sh.m_prev = (T)s_c.m_prev;
      sh.m_cur = (T)s_c.m_cur;
#if BQ_PROX_TRACE
      sh.tr7 = (cur == F_FUSED && tr3_on) ? 1 : 0;
#else
      sh.tr7 = 0;
#endif
      for (int i = 0; i < R; ++i) {
        sh.gw[i] = (T)s_c.gw[i];
        sh.gz[i] = (T)(s_c.gw[i] - s_c.beta[i]);
        sh.gc[i] = (T)s_c.gc[i];
        sh.gwid[i] = (T)s_c.gwid[i];
      }
    }
    }  // consumer warps
    __syncthreads();
    if (cur == F_FUSED) TR3(6);
    phase = sh.phase;
    if (phase == F_DONE) {
      if (s_pre[0] > 0) drain();
      break;
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
inline bool al16(const void* p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; }

template <typename T, int R>
int fused_launch(bq_ctx* ctx, const bq_wtv_desc& D, int wpm_only, cudaStream_t st) {
  constexpr int RW = FCfg<T, R>::RW;
  constexpr int NT = FCfg<T, R>::NT;
  FArgs<T> A{};
  A.ndim = D.ndim;
  A.mode = D.mode;
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
  A.dev_metric = D.dev_metric;
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
  A.ring[0] = (T*)D.p;
  A.ring[1] = (T*)D.pb;
  A.ring[2] = (T*)D.p2;
  A.abuf[0] = (T*)D.a;
  A.abuf[1] = (T*)D.a2;
  A.x = (T*)D.x;
  A.beta_io = D.beta;
  A.report = (bq_wtv_report*)D.report;
  BQ_STREAM_WS(sw, ctx, st);
  A.partials = sw->ws.partials;
  A.red = (double*)sw->ws.ctl;
  A.bar = sw->ws.barrier;
  A.lpr = std::min(A.K1 / 4, 32);
  A.rpw = 32 / A.lpr;
  A.wpr = A.K1 > 128 ? A.K1 / 128 : 1;
  A.lpr_log2 = 0;
  while ((1 << A.lpr_log2) < A.lpr) ++A.lpr_log2;
  if (D.d) {
    const size_t ib = (size_t)A.N * sizeof(T);
    if (sw->aux_bytes < ib) {
      cudaFree(sw->aux_buf);
      sw->aux_buf = nullptr;
      sw->aux_bytes = 0;
      BQ_CUDA(cudaMalloc(&sw->aux_buf, ib));
      sw->aux_bytes = ib;
    }
    A.ie = (T*)sw->aux_buf;
  }
  const int TYe = ((RW + 1) / A.wpr - 1) * A.rpw;  // standalone DIV pass tile
  A.nty = (A.K2 + TYe - 1) / TYe;
  A.tile_planes = (long long)A.nty * A.K3;

  auto kern = A.K1 == 128 ? wtv_fused_kernel<T, R, 128> : (A.K1 == 256 ? wtv_fused_kernel<T, R, 256> : wtv_fused_kernel<T, R, 0>);
  // staged FUSED pass: widest tile whose double-buffered stage fits in smem
  StageMap<R> M;
  M.make(D.d != nullptr, D.lo_arr != nullptr, D.hi_arr != nullptr, D.ndim, true);
  int optin = 0, static_b = 0;
  BQ_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  {
    cudaFuncAttributes fa{};
    BQ_CUDA(cudaFuncGetAttributes(&fa, (const void*)kern));
    static_b = (int)fa.sharedSizeBytes;
  }
  const size_t cap_kb = getenv("BQ_PROX_SMEMCAP_KB") ? (size_t)atoi(getenv("BQ_PROX_SMEMCAP_KB")) : 212;
  const size_t smem_cap = std::min<size_t>(cap_kb * 1024, (size_t)std::max(0, optin - static_b - 3072));
  int W = NT / 32 - 1;  // + 1 producer warp
  W -= W % A.wpr;       // whole row groups
  const char* ns_env = getenv("BQ_PROX_STAGES");
  int nst = ns_env ? std::max(2, std::min(NSTAGE, atoi(ns_env))) : NSTAGE;
  auto staged_bytes = [&](int w) {
    const long long srw = (long long)(w / A.wpr) * A.rpw + 1;
    return (size_t)(nst * M.nfield + 4) * srw * A.K1 * sizeof(T);
  };
  const char* w_env = getenv("BQ_PROX_WARPS");
  if (w_env) W = std::max(2, std::min(W, atoi(w_env)));
  W -= W % A.wpr;
  // a 3-deep ring for ranks <= 2 where it costs at most one warp of tile width
  // (rows <= 128 voxels) or none (x-split rows); measured: 128^3 rank 1
  // 3.29 -> 3.14 ms, 256^3 rank 1 scalar tau 19.6 -> 18.2 ms; the config-2
  // law at 256^3 (one field more, narrower tile) and rank 4 are faster 2-deep
  if (!ns_env) {
    int w3 = W;
    while (w3 > 2 * A.wpr && staged_bytes(w3) > smem_cap) w3 -= A.wpr;
    if (!(R <= BQ_RING3_R && w3 >= W - (A.K1 <= 128 ? 1 : 0))) nst = 2;
  }
  while (W > 2 * A.wpr && staged_bytes(W) > smem_cap) W -= A.wpr;
  BQ_CHECK(staged_bytes(W) <= smem_cap, BQ_EINVAL, "wtv_fused: stage does not fit in shared memory");
  A.geo.W = W;
  A.geo.nstage = nst;
  A.pre_max = getenv("BQ_PROX_PRE") ? std::max(0, std::min(nst, atoi(getenv("BQ_PROX_PRE")))) : nst;
  A.geo.SRW = (W / A.wpr) * A.rpw + 1;
  A.geo.slot_elems = (long long)A.geo.SRW * A.K1;
  A.geo.stage_elems = (long long)M.nfield * A.geo.slot_elems;
  const size_t base_dyn = std::max<size_t>(2ull * ((RW + 1) / A.wpr) * A.rpw * A.K1 * sizeof(T), staged_bytes(W));
  // near-list region after the stages (so the next pass's prefetched stages survive the on-chip Newton)
  const long long room = (long long)optin - static_b - (long long)base_dyn - 2048;
  const size_t list_bytes = room > 0 ? (size_t)(room / 16 * 16) : 0;
  const size_t dyn = base_dyn + list_bytes;
  BQ_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn + 1024));
  int per_sm = 0;
  BQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, dyn));
  BQ_CHECK(per_sm > 0, BQ_ECUDA, "wtv_fused: kernel does not fit on an SM");
  // one block per SM; small problems use fewer (cheaper barriers, enough work)
  long long G = std::min<long long>(ctx->num_sms, A.tile_planes);
  {
    // small grids: at least ~min_vox voxels per block (the z-march depth per block
    // sets the pass latency there, the barrier cost grows only slowly with G)
    const char* mv = getenv("BQ_PROX_MINVOX");
    const long long min_vox = mv ? std::max(64, atoi(mv)) : 512;
    G = std::max<long long>(1, std::min<long long>(G, (A.N + min_vox - 1) / min_vox));
  }
  {
    const int GW = W / A.wpr;
    const long long tp_s = (long long)((A.K2 + (GW - 1) * A.rpw - 1) / ((GW - 1) * A.rpw)) * A.K3;
    G = std::min<long long>(G, tp_s);
  }
  G = std::min<long long>(G, kMaxBlocks / 2);  // partials are double-buffered
  // opt-in (BQ_PROX_CLUSTER=1): small grids as ONE thread-block cluster of up
  // to 16 blocks (cluster barrier + DSMEM partials instead of the device-wide
  // barrier) when the grid has at most `cluster_vox` voxels per block and the
  // cluster can be scheduled (one GPC).  Measured at 32^3 (100 iterations):
  // fp64 rank 1 2.31 ms against 1.42 ms for the 64-block cooperative launch,
  // fp32 1.08 vs 1.03 ms -- the march of 4x more voxels per block costs more
  // than the cheaper barrier saves, so it is off by default
  A.cluster = 0;
  cudaLaunchConfig_t ccfg = {};
  cudaLaunchAttribute cat[1];
  {
    const char* ce = getenv("BQ_PROX_CLUSTER");
    const long long cvox = getenv("BQ_PROX_CLUSTER_VOX") ? atoll(getenv("BQ_PROX_CLUSTER_VOX")) : 2048;
    const int cmax = 16;
    long long Gc = std::min<long long>(cmax, (A.N + cvox - 1) / cvox);
    {
      const int GW = W / A.wpr;
      const long long tp_s = (long long)((A.K2 + (GW - 1) * A.rpw - 1) / ((GW - 1) * A.rpw)) * A.K3;
      Gc = std::min<long long>(Gc, tp_s);
    }
    if (ce && atoi(ce) == 1 && A.N <= cmax * cvox && Gc >= 2) {
      ccfg.gridDim = dim3((unsigned)Gc);
      ccfg.blockDim = dim3(NT);
      ccfg.dynamicSmemBytes = dyn;
      ccfg.stream = st;
      cat[0].id = cudaLaunchAttributeClusterDimension;
      cat[0].val.clusterDim.x = (unsigned)Gc;
      cat[0].val.clusterDim.y = 1;
      cat[0].val.clusterDim.z = 1;
      ccfg.attrs = cat;
      ccfg.numAttrs = 1;
      int ncl = 0;
      bool ok = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                cudaSuccess;
      ok = ok && cudaOccupancyMaxActiveClusters(&ncl, (void*)kern, &ccfg) == cudaSuccess && ncl >= 1;
      if (ok) {
        A.cluster = 1;
        G = Gc;
      } else {
        (void)cudaGetLastError();  // not schedulable as one cluster: the cooperative launch
      }
    }
  }
  // per-tile block assignment of the staged pass (see FArgs::tile_blk0): greedy,
  // one more block to the tile whose blocks would otherwise finish last.  A
  // step's cost grows with the tile's real rows (the last tile may be partial).
  A.ntile_tab = 0;
  {
    const int GW = W / A.wpr, TYs = (GW - 1) * A.rpw;
    const int ntile = (A.K2 + TYs - 1) / TYs;
    const char* te = getenv("BQ_PROX_TILEBLK");
    if ((!te || atoi(te) != 0) && !A.cluster && ntile <= kMaxTileTab && G >= ntile && G < 32768) {
      const double alpha = getenv("BQ_PROX_TILEALPHA") ? atof(getenv("BQ_PROX_TILEALPHA")) : 0.8;
      int nb[kMaxTileTab];
      auto cost = [&](int t) {
        const int rows = std::min(TYs, A.K2 - t * TYs);
        const int planes = (A.K3 + nb[t] - 1) / nb[t];
        return (planes + (nb[t] > 1 ? 2 : 0)) * (alpha + (1.0 - alpha) * rows / TYs);
      };
      for (int t = 0; t < ntile; ++t) nb[t] = 1;
      for (long long left = G - ntile; left > 0; --left) {
        int best = -1;
        double bc = 0.0;
        for (int t = 0; t < ntile; ++t)
          if (nb[t] < A.K3 && cost(t) > bc) bc = cost(t), best = t;
        if (best < 0) break;
        nb[best] += 1;
      }
      int acc = 0;
      double worst = 0.0;
      for (int t = 0; t < ntile; ++t) A.tile_blk0[t] = (short)acc, acc += nb[t], worst = std::max(worst, cost(t));
      A.tile_blk0[ntile] = (short)acc;
      // the contiguous split's slowest blocks cross a tile: ceil(planes) + 2 x (pre-step + warm-up);
      // few blocks per tile (large grids) split unevenly by tile and stay contiguous
      const double contiguous = (double)((long long)ntile * A.K3 + G - 1) / G + 4.0;
      if (acc == G && (worst < contiguous - 0.5 || (te && atoi(te) == 2))) A.ntile_tab = ntile;
    }
  }
  // near-list workspace
  constexpr int EWN = 3 + 2 * (R > 0 ? R : 1);
  {
    // near-list capacity: ~1/20 of the voxels a warp sees per pass (64 at 128^3, 512 at 256^3)
    const long long per_warp = A.N / (G * (NT / 32));
    int cap = CAPW;
    while (cap < 1024 && cap < per_warp / 20) cap *= 2;
    A.capw = cap;
  }
  const size_t data_bytes = 2 * (size_t)G * (NT / 32) * A.capw * EWN * sizeof(T);
  const size_t cnt_bytes = (2 * (size_t)G * (NT / 32) * sizeof(int) + 15) / 16 * 16;
  const size_t cl_bytes = 2 * (size_t)CL * EWN * sizeof(T);
  const size_t need = data_bytes + cnt_bytes + cl_bytes + 2 * CL * sizeof(unsigned);
  if (sw->near_bytes < need) {
    cudaFree(sw->near_buf);
    sw->near_buf = nullptr;
    sw->near_bytes = 0;
    BQ_CUDA(cudaMalloc(&sw->near_buf, need));
    sw->near_bytes = need;
  }
  A.near_data = sw->near_buf;
  A.near_cnt = (int*)((char*)sw->near_buf + data_bytes);
  const bool cl_use = !getenv("BQ_PROX_NOCL") || atoi(getenv("BQ_PROX_NOCL")) == 0;
  A.cl_data = cl_use ? (T*)((char*)sw->near_buf + data_bytes + cnt_bytes) : nullptr;
  A.cl_key = (unsigned*)((char*)sw->near_buf + data_bytes + cnt_bytes + cl_bytes);
  A.cl_ctr = sw->ws.barrier + 12;  // (+4: helper reductions, +8: bq_metric_check)

  A.dyn_bytes = (long long)dyn;
  A.list_off = (long long)base_dyn;
  A.list_bytes = (long long)list_bytes;
  A.trace = getenv("BQ_PROX_TRACE") ? (unsigned long long*)sw->ws.scratch : nullptr;
  A.trace_pass = getenv("BQ_PROX_TRACE") ? atoi(getenv("BQ_PROX_TRACE")) : 0;
  A.trace_thread = getenv("BQ_PROX_TRACE_THREAD") ? atoi(getenv("BQ_PROX_TRACE_THREAD")) : 0;
  A.dbg = getenv("BQ_PROX_DBG") ? atoi(getenv("BQ_PROX_DBG")) : 0;
  // minimum growth of the predicted gamma box: ranks <= 2 take the tighter box (fewer near voxels; measured at
  // 128^3: rank 1 2.854 -> 2.821 ms, rank 2 3.046 -> 3.020 ms, full-pass fallbacks unchanged); at rank 4 it costs
  // fallbacks on large grids (256^3: 25.5 -> 26.6 ms)
  A.grow_min = getenv("BQ_PROX_GROW") ? atof(getenv("BQ_PROX_GROW")) : (R <= 2 ? 4.0 : 8.0);
  A.ndist_min = getenv("BQ_PROX_NDIST") ? atof(getenv("BQ_PROX_NDIST")) : 1024.0;
  BQ_CUDA(cudaMemsetAsync(sw->ws.barrier, 0, 2 * sizeof(unsigned), st));
  BQ_CUDA(cudaMemsetAsync(sw->ws.barrier + 12, 0, sizeof(unsigned), st));
  if (A.cluster) {
    BQ_CUDA(cudaLaunchKernelEx(&ccfg, kern, A));
    return BQ_OK;
  }
  void* args[] = {&A};
  BQ_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3((unsigned)G), dim3(NT), args, dyn, st));
  return BQ_OK;
}

}  // namespace fused
}  // namespace bq
