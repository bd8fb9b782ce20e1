// explicit instantiations of the fused prox kernel (parallel compilation)
#include "wtv_fused_impl.cuh"

namespace bq {
namespace fused {
template int fused_launch<double, 6>(bq_ctx*, const bq_wtv_desc&, int, cudaStream_t);
template int fused_launch<double, 7>(bq_ctx*, const bq_wtv_desc&, int, cudaStream_t);
template int fused_launch<double, 8>(bq_ctx*, const bq_wtv_desc&, int, cudaStream_t);
}  // namespace fused
}  // namespace bq
