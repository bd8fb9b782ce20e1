// explicit instantiations of the fused prox kernel (parallel compilation)
#include "wtv_fused_impl.cuh"

namespace bq {
namespace fused {
template int fused_launch<double, 3>(bq_ctx*, const bq_wtv_desc&, int, cudaStream_t);
template int fused_launch<double, 4>(bq_ctx*, const bq_wtv_desc&, int, cudaStream_t);
template int fused_launch<double, 5>(bq_ctx*, const bq_wtv_desc&, int, cudaStream_t);
}  // namespace fused
}  // namespace bq
