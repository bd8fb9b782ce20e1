// ctx.cu — context lifetime, thread-local error text, version string.
#include <stdarg.h>

#include <algorithm>

#include "common.cuh"

namespace bq {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* where) {
  set_error("CUDA error %s (%s) at %s", cudaGetErrorName(e), cudaGetErrorString(e), where);
  return BQ_ECUDA;
}

void fft_cache_destroy(void* cache);  // views code

static void stream_ws_free(StreamWs* w) {
  if (!w) return;
  cudaFree(w->near_buf);
  cudaFree(w->aux_buf);
  if (w->host_flags) cudaFreeHost(w->host_flags);
  if (w->flag_ev[0]) cudaEventDestroy(w->flag_ev[0]);
  if (w->flag_ev[1]) cudaEventDestroy(w->flag_ev[1]);
  cudaFree(w->ws.partials);
  cudaFree(w->ws.barrier);
  cudaFree(w->ws.ctl);
  cudaFree(w->ws.scratch);
  delete w;
}

StreamWs* stream_ws(bq_ctx* ctx, cudaStream_t st) {
  for (int i = 0; i < ctx->n_streams; ++i)
    if (ctx->streams[i]->stream == st) return ctx->streams[i];
  if (ctx->n_streams == (int)(sizeof(ctx->streams) / sizeof(ctx->streams[0]))) {
    set_error("bq_ctx: more than %d streams used on one context", ctx->n_streams);
    return nullptr;
  }
  StreamWs* w = new StreamWs();
  w->stream = st;
  w->ws.ctl_bytes = 4096;
  cudaError_t e;
  if ((e = cudaMalloc(&w->ws.partials, sizeof(double) * kMaxBlocks * kMaxVals)) != cudaSuccess ||
      (e = cudaMalloc(&w->ws.barrier, 64)) != cudaSuccess ||
      (e = cudaMalloc(&w->ws.ctl, w->ws.ctl_bytes)) != cudaSuccess ||
      (e = cudaMalloc(&w->ws.scratch, sizeof(double) * 4096)) != cudaSuccess ||
      // zeroed ON the stream that will use them: a plain cudaMemset would queue on
      // the legacy default stream, behind whatever runs there, and a kernel on a
      // non-blocking stream could read the counters before they are cleared
      (e = cudaMemsetAsync(w->ws.barrier, 0, 64, st)) != cudaSuccess ||
      (e = cudaMemsetAsync(w->ws.ctl, 0, w->ws.ctl_bytes, st)) != cudaSuccess) {
    stream_ws_free(w);
    cuda_fail(e, "bq stream workspace");
    return nullptr;
  }
  ctx->streams[ctx->n_streams++] = w;
  return w;
}

}  // namespace bq

extern "C" const char* bq_last_error(void) { return bq::g_err; }

extern "C" const char* bq_version(void) { return "bq 0.1 sm_100a"; }

extern "C" int bq_ctx_create(int device, bq_ctx** out) {
  using namespace bq;
  BQ_CHECK(out, BQ_EINVAL, "bq_ctx_create: null out");
  *out = nullptr;
  int ndev = 0;
  BQ_CUDA(cudaGetDeviceCount(&ndev));
  BQ_CHECK(device >= 0 && device < ndev, BQ_EINVAL, "device %d out of range (%d devices)", device, ndev);
  BQ_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  BQ_CUDA(cudaGetDeviceProperties(&prop, device));
  BQ_CHECK(prop.major == 10 && prop.minor == 0, BQ_EINVAL,
           "libbq is built for sm_100a (B200); device %d is sm_%d%d", device, prop.major, prop.minor);
  int coop = 0;
  BQ_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
  BQ_CHECK(coop, BQ_ECUDA, "device %d does not support cooperative launch", device);
  bq_ctx* c = new bq_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  *out = c;
  return BQ_OK;
}

extern "C" int bq_ctx_destroy(bq_ctx* c) {
  using namespace bq;
  if (!c) return BQ_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  fft_cache_destroy(c->fft_cache);
  for (int i = 0; i < c->n_streams; ++i) stream_ws_free(c->streams[i]);
  delete c;
  return BQ_OK;
}
