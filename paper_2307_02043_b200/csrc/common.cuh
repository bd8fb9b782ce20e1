// common.cuh — shared plumbing of libbq.so: error text, context, device-wide
// barrier with fused deterministic reduction, block reductions.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <cmath>
#include <string>

#include "../../include/bq.h"

namespace bq {

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* where);

#define BQ_CUDA(call)                                          \
  do {                                                         \
    cudaError_t e_ = (call);                                   \
    if (e_ != cudaSuccess) return bq::cuda_fail(e_, #call);    \
  } while (0)

#define BQ_CHECK(cond, code, ...)        \
  do {                                   \
    if (!(cond)) {                       \
      bq::set_error(__VA_ARGS__);        \
      return code;                       \
    }                                    \
  } while (0)

// Max doubles one block contributes to one barrier-reduction:
// r (phi) + r(r+1)/2 (Newton matrix) for r = 8.
constexpr int kMaxVals = 96;
// Upper bound on resident blocks of any persistent kernel (148 SMs x 8).
constexpr int kMaxBlocks = 2048;

struct Workspace {
  double* partials = nullptr;     // kMaxBlocks * kMaxVals
  unsigned* barrier = nullptr;    // [0] arrival count, [1] generation
  void* ctl = nullptr;            // control block of the running persistent kernel
  size_t ctl_bytes = 0;
  double* scratch = nullptr;      // small device scratch (reductions of helpers)
};

}  // namespace bq

struct bq_ctx;
namespace bq {
// ls_fft.cu: padded-Green convolution as pruned line passes; returns 1 when the
// size has no instantiation (the caller then uses the cuFFT path).
// Optional: active[b] == 0 skips view b; dotp != NULL writes per-block partials
// (sum conj(da) out, sum |out|^2) as [B][*nblk][3] doubles.
int ls_conv_pruned(bq_ctx* ctx, int dtype, int n, int B, int op, const void* khat, const void* f, const void* v,
                   double alpha, double beta, const void* addend, void* scratch, void* out, cudaStream_t st,
                   const int* active = nullptr, const void* da = nullptr, double* dotp = nullptr, int* nblk = nullptr);
}  // namespace bq

namespace bq {
// Per-stream workspace: every buffer a launch writes outside the caller's
// tensors (barrier counters, block partials, controller block, near lists,
// 1/d, pinned BiCGSTAB flags).  One set per stream the context is used on, so
// calls on different streams of one context never share scratch (two
// concurrently running reductions would otherwise race on the partials and the
// arrival counter).  Calls on ONE stream are ordered, so they can share.
struct StreamWs {
  cudaStream_t stream = nullptr;
  Workspace ws;
  void* near_buf = nullptr;       // near-voxel lists of the fused prox kernel
  size_t near_bytes = 0;
  void* aux_buf = nullptr;        // per-voxel 1/d of the fused prox kernel
  size_t aux_bytes = 0;
  int* host_flags = nullptr;      // pinned: active-view counts of the device BiCGSTAB
  cudaEvent_t flag_ev[2] = {nullptr, nullptr};
};
// The workspace of `st` (created on first use); nullptr (error text set) when
// the allocation fails.
StreamWs* stream_ws(bq_ctx* ctx, cudaStream_t st);
}  // namespace bq

struct bq_ctx {
  int device = 0;
  int num_sms = 0;
  void* fft_cache = nullptr;      // owned by views code
  bq::StreamWs* streams[16] = {}; // per-stream workspaces (see StreamWs)
  int n_streams = 0;
};

#define BQ_STREAM_WS(var, ctx, st)                                   \
  bq::StreamWs* var = bq::stream_ws((ctx), (st));                    \
  if (!var) return BQ_ECUDA

namespace bq {

// ---------------------------------------------------------------------------
// Memory-model helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Block-wide sum of `nv` (<= NACC) per-thread doubles.  Deterministic: fixed
// shuffle tree inside each warp, then warps combined in index order.  Result
// written to out[0..nv) (shared memory).
template <int NT, int NACC>
__device__ __forceinline__ void block_sum_to(const double (&vals)[NACC], int nv, double* out,
                                            double* smem /* >= NT/32 * kMaxVals */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
#pragma unroll
  for (int k = 0; k < NACC; ++k) {
    if (k < nv) {
      double s = vals[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) smem[warp * kMaxVals + k] = s;
    }
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += smem[w * kMaxVals + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// Device-wide barrier whose last arriving block reduces every block's
// partial vector (in block-index order: deterministic, no float atomics) and
// then runs `controller`.  All blocks must be co-resident (cooperative launch).
// Returns false when the barrier timed out (abort).
struct GridSync {
  unsigned* count;
  unsigned* gen;
  unsigned nblocks;
  unsigned my_gen;
};

template <int NT, typename Controller>
__device__ bool grid_reduce_sync(GridSync& gs, const double* block_vals, int nv, double* partials,
                                 double* red /* smem kMaxVals */, double* smem_scratch,
                                 Controller&& controller) {
  __shared__ int s_last;
  // 1. publish this block's partials
  if (threadIdx.x < nv) partials[(size_t)blockIdx.x * kMaxVals + threadIdx.x] = block_vals[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned old = atomicAdd(gs.count, 1u);
    s_last = (old == gs.nblocks - 1);
    if (s_last) __threadfence();
  }
  __syncthreads();
  bool ok = true;
  if (s_last) {
    // 2. last block: fixed-order reduction over blocks.  Warp w owns values
    // w, w+NW, ...; lane l sums blocks l, l+32, ... then a fixed shuffle tree.
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = NT / 32;
    for (int k = warp; k < nv; k += NW) {
      double s = 0.0;
      for (unsigned b = lane; b < gs.nblocks; b += 32) s += __ldcg(&partials[(size_t)b * kMaxVals + k]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) red[k] = s;
    }
    __syncthreads();
    controller(red);  // every thread calls; controller decides who works
    __syncthreads();
    if (threadIdx.x == 0) {
      *gs.count = 0;
      __threadfence();
      atomicAdd(gs.gen, 1u);
    }
  } else {
    if (threadIdx.x == 0) {
      const uint64_t t0 = global_ns();
      unsigned spins = 0;
      while (ld_acquire_u32(gs.gen) == gs.my_gen) {
        __nanosleep(64);
        if (((++spins) & 1023u) == 0 && global_ns() - t0 > 20ull * 1000000000ull) {
          s_last = -1;  // timeout
          break;
        }
      }
      __threadfence();
    }
    __syncthreads();
    ok = (s_last != -1);
  }
  gs.my_gen += 1;
  return ok;
}

}  // namespace bq
