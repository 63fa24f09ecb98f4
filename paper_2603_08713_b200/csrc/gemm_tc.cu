// gemm_tc.cu -- tcgen05 block-scaled GEMM (K7-K9).  Placeholder until the
// kernel lands; the C-ABI reports the path as unsupported.
#include <cuda_runtime.h>
#include "mxq_internal.h"

namespace mxq {
int launch_gemm_tc(const QDesc& a, const QDesc& b, void* c, int c_dtype, int64_t ldc, uint32_t* status,
                   cudaStream_t st) {
  (void)a; (void)b; (void)c; (void)c_dtype; (void)ldc; (void)status; (void)st;
  return set_error(ERR_UNSUPPORTED, "tcgen05 GEMM not built yet");
}
}  // namespace mxq
