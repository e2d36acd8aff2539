// dwm_small_c_c3.cu -- small-C forward kernels for C_in = 3 (see dwm_small_c.cuh)
#include "dwm_small_c.cuh"

namespace dwm {
namespace smallc {
template int launch_cc<3>(const dwm_desc_t&, const float*, const float*, float*, int32_t*, cudaStream_t);
}  // namespace smallc
}  // namespace dwm
