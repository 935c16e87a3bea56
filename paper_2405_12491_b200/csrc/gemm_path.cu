// GEMM-form lowering of steps a1..a4 (placeholder until the tcgen05 kernels land).
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "bridger_internal.h"

namespace bridger {

bool gemm_build(bridger_model* m, const bridger_model_desc*, const std::vector<int32_t>&, std::string* why) {
  m->gemm_ok = false;
  if (why) *why = "GEMM path not built";
  return false;
}
void gemm_free(bridger_model*) {}
cudaError_t gemm_run(const bridger_model*, const float*, int64_t, void*, int, int32_t, cudaStream_t) {
  return cudaErrorNotSupported;
}
cudaError_t gemm_step_decisions(const bridger_model*, const float*, int64_t, int32_t, int32_t, int8_t*, cudaStream_t,
                                std::string* why) {
  *why = "GEMM path not built";
  return cudaErrorNotSupported;
}
cudaError_t gemm_step_scores(const bridger_model*, int32_t, const int8_t*, int64_t, int32_t*, cudaStream_t,
                             std::string* why) {
  *why = "GEMM path not built";
  return cudaErrorNotSupported;
}

}  // namespace bridger
