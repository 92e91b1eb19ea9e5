// gemm_tc.cu -- tcgen05 / TMEM / TMA model-batched GEMM (placeholder; the
// SIMT path serves every shape until this lands).
#include "gemm.cuh"

namespace hfta {
bool gemm_tc_supported(const GemmP&, hfta_dtype, bool) { return false; }
hfta_status gemm_tc(const GemmP&, hfta_dtype, bool, cudaStream_t) {
  return fail(HFTA_ERR_UNSUPPORTED, "gemm_tc: not available");
}
}  // namespace hfta
