// Microbenchmarks that size the prox kernel's design choices on B200
// (not product code; built and run by bench/micro/run_micro.sh under gpurun):
//   1. stream:  read 6 fp32 fields + write 1 at N = 128^3 (the DIV-phase byte
//               pattern), float4 grid-stride, as a normal launch; L2-warm and
//               L2-flushed.
//   2. barrier: a persistent kernel that does nothing but the prox kernel's
//               last-block-reduces grid barrier, G = 148 x k blocks.
//   3. stencil: the DIV z-march (x-vectorised) as a normal launch.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);      \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

__global__ void stream6(const float4* __restrict__ a, const float4* __restrict__ b, const float4* __restrict__ c,
                        const float4* __restrict__ d, const float4* __restrict__ e, const float4* __restrict__ f,
                        float4* __restrict__ o, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 x = __ldg(a + i), y = __ldg(b + i), z = __ldg(c + i), w = __ldg(d + i), u = __ldg(e + i), v = __ldg(f + i);
    o[i] = make_float4(x.x + y.x + z.x + w.x + u.x + v.x, x.y + y.y + z.y + w.y + u.y + v.y,
                       x.z + y.z + z.z + w.z + u.z + v.z, x.w + y.w + z.w + w.w + u.w + v.w);
  }
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void barrier_only(unsigned* bar, double* partials, double* red, int rounds, int nv, int sleep_ns) {
  __shared__ int s_flag;
  __shared__ double s_red[64];
  unsigned my_gen = 0;
  if (threadIdx.x == 0) my_gen = ld_acquire(bar + 1);
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x < nv) partials[blockIdx.x * 48 + threadIdx.x] = r + threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      unsigned old = atomicAdd(bar, 1u);
      s_flag = old == gridDim.x - 1;
      if (s_flag) __threadfence();
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (s_flag) {
      for (int k = warp; k < nv; k += blockDim.x / 32) {
        double s = 0;
        for (unsigned b = lane; b < gridDim.x; b += 32) s += __ldcg(&partials[b * 48 + k]);
        for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (lane == 0) __stcg(&red[k], s);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        bar[0] = 0;
        __threadfence();
        atomicAdd(bar + 1, 1u);
      }
    } else {
      if (threadIdx.x == 0) {
        while (ld_acquire(bar + 1) == my_gen) {
          if (sleep_ns) __nanosleep(sleep_ns);
        }
        __threadfence();
      }
      __syncthreads();
      if (threadIdx.x < nv) s_red[threadIdx.x] = __ldcg(&red[threadIdx.x]);
    }
    my_gen++;
    __syncthreads();
  }
}

// DIV-phase z-march, x-vectorised (4 voxels / lane), as a normal launch.
template <int TY>
__global__ void div_march(const float* __restrict__ F, const float* __restrict__ D, const float* __restrict__ V,
                          const float* __restrict__ U, float* __restrict__ Aout, int K, long long seg_len,
                          double* out) {
  const long long N = (long long)K * K * K, plane = (long long)K * K;
  const float* F1 = F + N;
  const float* F2 = F + 2 * N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long tiles = (long long)(K / TY) * K;
  const long long b0 = blockIdx.x * tiles / gridDim.x, b1 = (blockIdx.x + 1) * tiles / gridDim.x;
  double acc = 0;
  for (long long pos = b0; pos < b1;) {
    const long long tile = pos / K;
    const int z0 = pos - tile * K;
    const int z1 = min((long long)K, z0 + (b1 - pos));
    pos += z1 - z0;
    const int xb = 4 * lane, y = (int)tile * TY + warp;
    long long j = (long long)z0 * plane + (long long)y * K + xb;
    float4 p3 = z0 > 0 ? *(const float4*)(F2 + j - plane) : make_float4(0, 0, 0, 0);
#pragma unroll 2
    for (int z = z0; z < z1; ++z, j += plane) {
      float4 c1 = *(const float4*)(F + j);
      float left = __shfl_up_sync(0xffffffffu, c1.w, 1);
      if (lane == 0) left = 0;
      float4 c2 = *(const float4*)(F1 + j);
      float4 l2 = y > 0 ? *(const float4*)(F1 + j - K) : make_float4(0, 0, 0, 0);
      float4 c3 = *(const float4*)(F2 + j);
      float4 d = __ldg((const float4*)(D + j)), v = __ldg((const float4*)(V + j)), u = __ldg((const float4*)(U + j));
      float4 dv;
      dv.x = -c1.x + left - c2.x + l2.x - c3.x + p3.x;
      dv.y = -c1.y + c1.x - c2.y + l2.y - c3.y + p3.y;
      dv.z = -c1.z + c1.y - c2.z + l2.z - c3.z + p3.z;
      dv.w = -c1.w + c1.z - c2.w + l2.w - c3.w + p3.w;
      p3 = c3;
      float4 a;
      a.x = v.x - 0.05f * dv.x * __frcp_rn(d.x);
      a.y = v.y - 0.05f * dv.y * __frcp_rn(d.y);
      a.z = v.z - 0.05f * dv.z * __frcp_rn(d.z);
      a.w = v.w - 0.05f * dv.w * __frcp_rn(d.w);
      *(float4*)(Aout + j) = a;
      acc += (double)u.x * dv.x + (double)u.y * dv.y + (double)u.z * dv.z + (double)u.w * dv.w;
    }
  }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  const int K = 128;
  const long long N = (long long)K * K * K;
  int dev = 0, sms = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  float* buf;
  CK(cudaMalloc(&buf, sizeof(float) * N * 12));
  CK(cudaMemset(buf, 0, sizeof(float) * N * 12));
  float* flush;
  const size_t FL = 512ull << 20;
  CK(cudaMalloc(&flush, FL));
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  float ms;

  // 1. streaming
  for (int bpsm : {2, 4, 8}) {
    for (int flushit = 0; flushit < 2; ++flushit) {
      const int G = sms * bpsm;
      float tot = 0;
      const int reps = 20;
      for (int r = 0; r < reps + 2; ++r) {
        if (flushit) CK(cudaMemsetAsync(flush, r, FL));
        cudaEventRecord(t0);
        stream6<<<G, 256>>>((float4*)buf, (float4*)(buf + N), (float4*)(buf + 2 * N), (float4*)(buf + 3 * N),
                            (float4*)(buf + 4 * N), (float4*)(buf + 5 * N), (float4*)(buf + 6 * N), N / 4);
        cudaEventRecord(t1);
        CK(cudaEventSynchronize(t1));
        cudaEventElapsedTime(&ms, t0, t1);
        if (r >= 2) tot += ms;
      }
      const double us = 1e3 * tot / reps;
      printf("stream6+1 N=128^3 blocks/SM=%d flush=%d: %.2f us  %.0f GB/s\n", bpsm, flushit, us,
             7.0 * 4 * N / (us * 1e-6) / 1e9);
    }
  }

  // 2. barrier only
  unsigned* bar;
  double *partials, *red;
  CK(cudaMalloc(&bar, 64));
  CK(cudaMalloc(&partials, sizeof(double) * 4096 * 48));
  CK(cudaMalloc(&red, sizeof(double) * 64));
  for (int nt : {256, 512, 1024}) {
    for (int bpsm : {1, 2}) {
      if (nt * bpsm > 2048) continue;
      for (int sl : {0, 32}) {
        const int G = sms * bpsm, rounds = 2000, nv = 2;
        CK(cudaMemset(bar, 0, 64));
        void* args[] = {&bar, &partials, &red, (void*)&rounds, (void*)&nv, (void*)&sl};
        int rr = rounds;
        args[3] = &rr;
        int nvv = nv;
        args[4] = &nvv;
        int sll = sl;
        args[5] = &sll;
        cudaEventRecord(t0);
        CK(cudaLaunchCooperativeKernel((void*)barrier_only, G, nt, args, 0, 0));
        cudaEventRecord(t1);
        CK(cudaEventSynchronize(t1));
        cudaEventElapsedTime(&ms, t0, t1);
        printf("barrier G=%d (x%d/SM, %d thr) nanosleep=%d: %.3f us per barrier\n", G, bpsm, nt, sl,
               1e3 * ms / rounds);
      }
    }
  }

  // 3. DIV z-march as a plain launch
  for (int bpsm : {1, 2, 4}) {
    const int G = sms * bpsm;
    float tot = 0;
    const int reps = 20;
    for (int r = 0; r < reps + 2; ++r) {
      cudaEventRecord(t0);
      div_march<16><<<G, 512>>>(buf, buf + 3 * N, buf + 4 * N, buf + 5 * N, buf + 6 * N, K, 0, partials);
      cudaEventRecord(t1);
      CK(cudaEventSynchronize(t1));
      cudaEventElapsedTime(&ms, t0, t1);
      if (r >= 2) tot += ms;
    }
    const double us = 1e3 * tot / reps;
    printf("div_march TY=16 NT=512 blocks/SM=%d: %.2f us  (%.0f GB/s of 7 words/voxel)\n", bpsm, us,
           7.0 * 4 * N / (us * 1e-6) / 1e9);
  }
  for (int bpsm : {2, 4}) {
    const int G = sms * bpsm;
    float tot = 0;
    const int reps = 20;
    for (int r = 0; r < reps + 2; ++r) {
      cudaEventRecord(t0);
      div_march<8><<<G, 256>>>(buf, buf + 3 * N, buf + 4 * N, buf + 5 * N, buf + 6 * N, K, 0, partials);
      cudaEventRecord(t1);
      CK(cudaEventSynchronize(t1));
      cudaEventElapsedTime(&ms, t0, t1);
      if (r >= 2) tot += ms;
    }
    const double us = 1e3 * tot / reps;
    printf("div_march TY=8 NT=256 blocks/SM=%d: %.2f us  (%.0f GB/s of 7 words/voxel)\n", bpsm, us,
           7.0 * 4 * N / (us * 1e-6) / 1e9);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
