// explicit instantiations of the fused prox kernel (parallel compilation)
#include "wtv_fused_impl.cuh"

namespace bq {
namespace fused {
template int fused_launch<float, 0>(bq_ctx*, const bq_wtv_desc&, int, cudaStream_t);
template int fused_launch<float, 1>(bq_ctx*, const bq_wtv_desc&, int, cudaStream_t);
template int fused_launch<float, 2>(bq_ctx*, const bq_wtv_desc&, int, cudaStream_t);
}  // namespace fused
}  // namespace bq
