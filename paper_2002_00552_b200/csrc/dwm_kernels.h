// dwm_kernels.h -- internal launcher declarations (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include "../../include/dwm_b200.h"

namespace dwm {

// strides: element strides (f, c, kh, kw) of the weight view; NULL = contiguous F,C,r_h,r_w
int launch_filter_transform(const dwm_desc_t& d, int dtype, const void* w, void* U, cudaStream_t s,
                            const int64_t* strides = nullptr);
// U for the tcgen05 path: per-filter power-of-two scaled, fp16 split U'hi /
// U'lo, stacked per 64-filter block: [freq][ceil(F/64)][U'hi 64 rows; U'lo 64
// rows][C] fp16 (zero rows past F), so one TMA box gives the GEMM its
// [U'hi; U'lo] N = 128 B operand; then 1 / s_f per padded filter (fp32).
int launch_filter_transform_f16split(const dwm_desc_t& d, const void* w, void* U, cudaStream_t s,
                                     const int64_t* strides = nullptr);
// max|x| per image (float bits, one uint32 slot per image) that the float
// input transform fills when xmax != NULL (zeroed first, on the same stream):
// the tcgen05 GEMM's per-image V-scale bound, so an image's result never
// depends on the other images of the batch (chunking / sharding invariance)
inline size_t xmax_bytes(const dwm_desc_t& d) { return ((size_t)d.n * sizeof(uint32_t) + 15) & ~(size_t)15; }
int launch_input_transform(const dwm_desc_t& d, int dtype, const void* x, void* V, cudaStream_t s,
                           uint32_t* xmax = nullptr);
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
// xmax: the input transform's per-image max|x| slots; NULL = bound by the
// per-image max|V|, computed into scratch (>= xmax_bytes(d))
int launch_gemm_tc(const dwm_desc_t& d, const void* V, const void* U, void* y, int32_t* flag, const uint32_t* xmax,
                   void* scratch, size_t scratch_bytes, cudaStream_t s);

}  // namespace dwm
