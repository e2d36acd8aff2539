// dwm_kernels.h -- internal launcher declarations (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include "../../include/dwm_b200.h"

namespace dwm {

// strides: element strides (f, c, kh, kw) of the weight view; NULL = contiguous F,C,r_h,r_w
int launch_filter_transform(const dwm_desc_t& d, int dtype, const void* w, void* U, cudaStream_t s,
                            const int64_t* strides = nullptr);
// U for the tcgen05 path: TF32-valued RN split U_hi / U_lo, stacked per
// 64-filter block: [freq][ceil(F/64)][U_hi 64 rows; U_lo 64 rows][C] (zero rows
// past F), so one TMA box gives the GEMM its [U_hi; U_lo] N = 128 B operand.
int launch_filter_transform_tf32split(const dwm_desc_t& d, const void* w, void* U, cudaStream_t s,
                                      const int64_t* strides = nullptr);
int launch_input_transform(const dwm_desc_t& d, int dtype, const void* x, void* V, cudaStream_t s);
int launch_gemm_exact(const dwm_desc_t& d, int dtype, const void* V, const void* U, void* y,
                      int32_t* flag, cudaStream_t s);
int weight_grad_splits(const dwm_desc_t& d);
bool wgrad_tc_supported(const dwm_desc_t& d);
size_t wgrad_tc_workspace_bytes(const dwm_desc_t& d);
int launch_wgrad_tc(const dwm_desc_t& d, const void* x, const void* dy, void* gw, void* ws, size_t ws_bytes,
                    int32_t* flag, cudaStream_t s);
int launch_weight_grad(const dwm_desc_t& d, int dtype, const void* x, const void* dy, void* gw, void* ws,
                       size_t ws_bytes, int32_t* flag, cudaStream_t s);
bool small_c_supported(const dwm_desc_t& d);
int launch_small_c(const dwm_desc_t& d, const void* x, const void* U, void* y, int32_t* flag,
                   cudaStream_t s);
bool tc_gemm_supported(const dwm_desc_t& d);
size_t tc_filter_bytes(const dwm_desc_t& d);
int launch_gemm_tc(const dwm_desc_t& d, const void* V, const void* U, void* y, int32_t* flag,
                   cudaStream_t s);

}  // namespace dwm
