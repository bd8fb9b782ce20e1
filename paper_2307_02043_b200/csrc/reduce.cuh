// reduce.cuh — "last block done" deterministic reductions for ordinary
// (non-cooperative) launches: every block writes its partial vector, the last
// block to arrive sums them in block-index order (no float atomics, no
// co-residency requirement) and may run a scalar epilogue.
#pragma once

#include "common.cuh"

namespace bq {

struct RedWs {
  double* partials;  // MAXB * kMaxVals
  unsigned* count;
};

// Returns true in the last block; red[0..nv) then holds the totals (smem).
template <int NT, int NACC>
__device__ bool last_block_reduce(const double (&acc)[NACC], int nv, RedWs ws, double* red,
                                  double* scr) {
  __shared__ double s_bv[kMaxVals];
  __shared__ int s_last;
  block_sum_to<NT, NACC>(acc, nv, s_bv, scr);
  if (threadIdx.x < nv) ws.partials[(size_t)blockIdx.x * kMaxVals + threadIdx.x] = s_bv[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned old = atomicAdd(ws.count, 1u);
    s_last = (old == gridDim.x - 1);
    if (s_last) __threadfence();
  }
  __syncthreads();
  if (!s_last) return false;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = warp; k < nv; k += NT / 32) {
    double s = 0.0;
    for (unsigned b = lane; b < gridDim.x; b += 32) s += __ldcg(&ws.partials[(size_t)b * kMaxVals + k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) red[k] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) *ws.count = 0;  // ready for the next launch
  return true;
}

inline RedWs red_ws(StreamWs* sw) { return RedWs{sw->ws.partials, sw->ws.barrier + 4}; }

}  // namespace bq
