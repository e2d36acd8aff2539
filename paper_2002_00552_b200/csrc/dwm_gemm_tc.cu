// dwm_gemm_tc.cu -- tcgen05/TMEM 3xTF32 transform-domain GEMM with the output
// transform fused in the epilogue.  (Round-1 placeholder: not yet eligible.)
#include "dwm_common.cuh"
#include "dwm_kernels.h"

namespace dwm {

bool tc_gemm_supported(const dwm_desc_t& d) { return false; }

int launch_gemm_tc(const dwm_desc_t& d, const void* V, const void* U, void* y, int32_t* flag,
                   cudaStream_t s) {
  return fail(DWM_EUNSUPPORTED, "tcgen05 GEMM not built in this revision");
}

}  // namespace dwm
