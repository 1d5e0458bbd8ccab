// Prefill expert FFN (row a6).  Temporary: routes through the decode GEMV kernels (which loop
// over 8-token chunks) until the tcgen05 grouped GEMM lands.
#include "../dymoe_internal.cuh"

namespace dymoe {
cudaError_t launch_ffn_prefill(const FfnArgs& a, cudaStream_t s, void* const* ev) {
  return launch_ffn_decode(a, s, ev);
}
}  // namespace dymoe
