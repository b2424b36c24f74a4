// ucg_gemm.cu — dense matmul device op (workload C5). tcgen05 kernel pending.
#include "ucg_common.cuh"

using namespace ucg;

extern "C" int ucg_gemm_tf32(const float* A, const float* B, float* C, uint64_t n, void* stream) {
  (void)A; (void)B; (void)C; (void)n; (void)stream;
  if (int rc = check_device()) return rc;
  return fail(UCG_ERR_ARG, "ucg_gemm_tf32: not built in this revision");
}
