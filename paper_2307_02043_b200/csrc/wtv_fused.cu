// wtv_fused.cu — dispatch of the fused prox kernel (instantiations live in
// wtv_fused_inst_*.cu so they compile in parallel).
#include "wtv_fused_impl.cuh"

namespace bq {
namespace fused {
#define BQ_FUSED_DECL(T, R) extern template int fused_launch<T, R>(bq_ctx*, const bq_wtv_desc&, int, cudaStream_t);
BQ_FUSED_DECL(float, 0) BQ_FUSED_DECL(float, 1) BQ_FUSED_DECL(float, 2) BQ_FUSED_DECL(float, 3)
BQ_FUSED_DECL(float, 4) BQ_FUSED_DECL(float, 5) BQ_FUSED_DECL(float, 6) BQ_FUSED_DECL(float, 7)
BQ_FUSED_DECL(float, 8) BQ_FUSED_DECL(double, 0) BQ_FUSED_DECL(double, 1) BQ_FUSED_DECL(double, 2)
BQ_FUSED_DECL(double, 3) BQ_FUSED_DECL(double, 4) BQ_FUSED_DECL(double, 5) BQ_FUSED_DECL(double, 6)
BQ_FUSED_DECL(double, 7) BQ_FUSED_DECL(double, 8)
#undef BQ_FUSED_DECL
}  // namespace fused

using fused::al16;
using fused::fused_launch;

// Fast-path eligibility: 16-byte-aligned fields, K1 in {4, 8, ..., 128}
// dividing 128 or K1 == 256 (two warps per x-row), ring/ping-pong scratch supplied.
bool fused_eligible(const bq_wtv_desc& D) {
  const long long K1 = D.dims[0];
  if (D.ndim != 3) return false;
  if (!((K1 >= 4 && K1 <= 128 && K1 % 4 == 0 && 128 % K1 == 0) || K1 == 256)) return false;
  if (!D.p2 || !D.a2 || !D.pb || !D.p) return false;
  // scalar box bounds only (the stage layout and the bounds are pass
  // constants); per-voxel bound arrays take the general kernel
  if (D.lo_arr || D.hi_arr) return false;
  const void* ptrs[] = {D.p, D.pb, D.p2, D.a, D.a2, D.v, D.x, D.d, D.U, D.lo_arr, D.hi_arr};
  for (const void* q : ptrs)
    if (!al16(q)) return false;
  return true;
}

int fused_dispatch(bq_ctx* ctx, const bq_wtv_desc& D, int wpm_only, cudaStream_t st) {
  const bool f = D.dtype == BQ_F32;
  switch (D.rank) {
#define FCASE(r) \
  case r: return f ? fused_launch<float, r>(ctx, D, wpm_only, st) : fused_launch<double, r>(ctx, D, wpm_only, st);
    FCASE(0) FCASE(1) FCASE(2) FCASE(3) FCASE(4) FCASE(5) FCASE(6) FCASE(7) FCASE(8)
#undef FCASE
  }
  set_error("wtv_fused: rank %d outside [0, %d]", D.rank, BQ_MAX_RANK);
  return BQ_EINVAL;
}

}  // namespace bq
