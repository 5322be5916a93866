// k_gemm_tc.cu — tcgen05 GEMM (placeholder until the TMA/UMMA kernel lands).
#include "k_common.cuh"

namespace bb {
namespace k {
bool gemm_tc_supported(const Gemm &) { return false; }
cudaError_t gemm_tc(const Gemm &, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace k
}  // namespace bb
