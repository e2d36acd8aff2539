/*
 * dwm_b200.h -- C ABI of the B200-native Decomposable Winograd (DWM) conv2d.
 *
 * This is the drop-in boundary for the reference's hot path
 *   dwmconv.engines.dwm_conv2d(data, weights, spec, plan=None,
 *                              precision=None, counter=None)
 *   (reference: pkg/src/dwmconv/engines.py:219-255)
 * and the stages it runs.  The reference is pure Python/NumPy, so its
 * "FFI" is the Python call itself; the Python package
 * paper_2002_00552_b200 binds these symbols with ctypes
 * (paper_2002_00552_b200/_native.py) and re-exposes the reference's exact
 * signature.  INTEGRATION.md shows the ctypes stub a maintainer of the
 * reference package would add.
 *
 * Conventions
 *   - plain pointers and sizes only; every device pointer is CUDA global
 *     memory; `stream` is a cudaStream_t passed as void* (NULL = legacy
 *     default stream).  All compute entry points are stream-ordered and
 *     asynchronous; none synchronises the device.
 *   - tensors are row-major NCHW (data, output) and F,C,r_h,r_w (weights),
 *     exactly the reference's layouts.
 *   - no hidden global mutable state except the thread-local error message
 *     and the lazily-initialised per-device kernel attributes.
 *   - every function returns a dwm_status; on failure dwm_last_error()
 *     returns a human-readable message whose wording mirrors the
 *     reference's ValueError/TypeError/FloatingPointError texts.
 */
#ifndef DWM_B200_H
#define DWM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DWM_MAX_AXIS_PARTS 16

typedef enum dwm_status {
  DWM_OK = 0,
  DWM_EINVAL_SHAPE = 1,   /* -> ValueError   (engines.py:66-68,231-236; convspec.py:23-43) */
  DWM_EINVAL_DTYPE = 2,   /* -> TypeError    (tensor.py:18-23)                            */
  DWM_NONFINITE = 3,      /* -> FloatingPointError (tensor.py:27-30)                       */
  DWM_ECUDA = 4,          /* CUDA runtime failure                                          */
  DWM_EUNSUPPORTED = 5    /* geometry outside what the kernels implement                   */
} dwm_status;

typedef enum dwm_dtype { DWM_F32 = 0, DWM_F64 = 1 } dwm_dtype;

/* Transform-domain contraction engine.
 *   EXACT:   CUDA-core FMA chains in the reference's stage order (channel-
 *            ascending GEMM, At.m.A row then column stage, plan-order part
 *            sum) over a V workspace.  Bit-identical to the reference where
 *            its BLAS accumulates sequentially (small C); f32 and f64.
 *   TC:      tcgen05/TMEM GEMM (3 fp16 products of power-of-two scaled
 *            operands, FP32 accumulation) with the output transform, part sum and
 *            tile interleave fused in the epilogue (f32 only, C % 32 == 0;
 *            any F, in 64-filter blocks).
 *   SMALL_C: one fused kernel (input transform computed in shared memory,
 *            same arithmetic as EXACT, no V workspace); f32, C_in <= 4.
 *   AUTO:    SMALL_C for C_in <= 4, TC when eligible, C_in >= 64, F >= 32, else
 *            EXACT.  dwm_select_algo() reports the resolved engine. */
typedef enum dwm_algo {
  DWM_ALGO_AUTO = 0, DWM_ALGO_EXACT = 1, DWM_ALGO_TC = 2, DWM_ALGO_SMALL_C = 3
} dwm_algo;

/* One strided run of kernel taps along an axis: origin + step*i, i < count
 * (reference AxisPart, decompose.py:25-35). */
typedef struct dwm_axis_part {
  int32_t origin, step, count;
} dwm_axis_part_t;

/* Geometry + decomposition plan.  Filled by dwm_desc_init() from the
 * ConvSpec fields; the 2-D plan is the row-major cross product
 * row_parts x col_parts (decompose.py:103-114). */
typedef struct dwm_desc {
  int32_t n, c, h, w, f;                      /* data N,C,H,W; filters F    */
  int32_t r_h, r_w, s_h, s_w;                 /* kernel taps, stride        */
  int32_t pad_top, pad_bottom, pad_left, pad_right;
  /* derived */
  int32_t oh, ow;                             /* convspec.py:34-44          */
  int32_t th, tw;                             /* 2x2 output tiles per image */
  int32_t n_row_parts, n_col_parts;
  dwm_axis_part_t row_parts[DWM_MAX_AXIS_PARTS];
  dwm_axis_part_t col_parts[DWM_MAX_AXIS_PARTS];
  int32_t row_freqs, col_freqs;               /* sum of (count+1) per axis  */
  int32_t num_freqs;                          /* sum over parts a_r*a_c     */
  int64_t tiles;                              /* n * th * tw                */
} dwm_desc_t;

/* Plan a convolution: validates geometry exactly like ConvSpec/out_dims and
 * runs the C++ restatement of plan_decomposition (decompose.py:60-114). */
int dwm_desc_init(dwm_desc_t* desc, int n, int c, int h, int w, int f,
                  int r_h, int r_w, int s_h, int s_w,
                  int pad_top, int pad_bottom, int pad_left, int pad_right);

/* FlopCounter increment of one call: TH*TW*sum_parts a_r*a_c
 * (engines.py:190-191, == flops.flops_dwm, flops.py:107-119). */
int64_t dwm_elementwise_count(const dwm_desc_t* desc);

/* Bytes of caller-provided device workspace dwm_conv2d_forward needs. */
size_t dwm_workspace_bytes(const dwm_desc_t* desc, int dtype, int algo);

/* Resolve AUTO to the engine that will run (for reporting). */
int dwm_select_algo(const dwm_desc_t* desc, int dtype, int algo);

/* Stage kernels (exposed for the parity tests and the stage profiler).
 *   U layout: [num_freqs][F][C]      (frequency order: parts in plan order,
 *                                     row frequency, then column frequency)
 *   V layout: [num_freqs][tiles][C]  (tile = (n*TH + ty)*TW + tx)        */
int dwm_filter_transform(const dwm_desc_t* desc, int dtype, const void* w,
                         void* U, void* stream);
int dwm_input_transform(const dwm_desc_t* desc, int dtype, const void* x,
                        void* V, void* stream);
int dwm_gemm_output(const dwm_desc_t* desc, int dtype, int algo, const void* V,
                    const void* U, void* y, int32_t* nonfinite_flag,
                    void* workspace, size_t workspace_bytes, void* stream);

/* The tcgen05 engine's range-carrying stage pair (what dwm_conv2d_forward
 * runs internally): dwm_input_transform_ranged is dwm_input_transform (f32)
 * that also records each image's max|x| into `range` (dwm_range_bytes: one
 * uint32 per image, device, 16-byte aligned), from which dwm_gemm_output_tc
 * picks the per-image power-of-two V scale of its fp16 split; U from
 * dwm_prepare_filter(algo = DWM_ALGO_TC).  dwm_gemm_output with algo TC
 * derives the range from V itself instead (one more pass over V; workspace
 * >= dwm_range_bytes). */
size_t dwm_range_bytes(const dwm_desc_t* desc);
int dwm_input_transform_ranged(const dwm_desc_t* desc, const void* x, void* V, uint32_t* range,
                               void* stream);
int dwm_gemm_output_tc(const dwm_desc_t* desc, const void* V, const void* U, const uint32_t* range,
                       void* y, int32_t* nonfinite_flag, void* stream);

/* Fused small-C forward (DWM_ALGO_SMALL_C) from the filter-transform
 * output U ([num_freqs][F][C], f32): gathers and transforms x on chip. */
int dwm_conv2d_small_c(const dwm_desc_t* desc, const void* x, const void* U,
                       void* y, int32_t* nonfinite_flag, void* stream);

/* Cached-filter forward (the operator wrapper keeps U
 * per weight version; the reference recomputes G g G^T every call,
 * engines.py:246-248).  dwm_filter_bytes: bytes of U in the layout the
 * engine `algo` selects for this geometry (TC: scaled fp16 hi|lo planes and
 * per-filter scales).  U depends
 * only on (F, C, kernel, stride, algo), never on the batch or image size --
 * but the selected engine can, so prepare with the same desc as the forward.
 * dwm_conv2d_forward_prepared: the forward with U given; workspace holds V
 * only (dwm_workspace_bytes is an upper bound). */
size_t dwm_filter_bytes(const dwm_desc_t* desc, int dtype, int algo);
int dwm_prepare_filter(const dwm_desc_t* desc, int dtype, int algo, const void* w,
                       void* U, void* stream);
/* dwm_prepare_filter on a strided weight view: strides[4] are the element
 * strides of (f, c, kh, kw) (any sign; w points at element (0,0,0,0) of the
 * view).  The backward's data gradient uses it for the channel-transposed,
 * tap-reversed polyphase sub-kernels w[:, :, rho::s_h, sig::s_w] without
 * materialising them. */
int dwm_prepare_filter_strided(const dwm_desc_t* desc, int dtype, int algo, const void* w,
                               const int64_t* strides, void* U, void* stream);
int dwm_conv2d_forward_prepared(const dwm_desc_t* desc, int dtype, int algo, const void* x,
                                const void* U, void* y, void* workspace, size_t workspace_bytes,
                                int32_t* nonfinite_flag, void* stream);

/* Weight gradient of the forward (reference
 * dwm_backward / _winograd_grad_weight_impl, engines.py:258-330,342-399):
 * gw[F,C,r_h,r_w] from x[N,C,H,W] and dy[N,F,OH,OW].  Engines (`algo`):
 *   DWM_ALGO_TC    (AUTO's choice for float32, C % 32 == 0, C >= 64, F >= 64):
 *                  Winograd domain like the reference -- V = B^T x B (the
 *                  forward's input transform), DM = A dY A^T, per frequency
 *                  dU = V^T DM on tcgen05 (3xTF32, K = tiles, blocked FP32
 *                  sums), then G^T dU G placed at each part's taps;
 *   DWM_ALGO_EXACT (any shape, float64): implicit-im2col GEMM on CUDA cores,
 *                  geometry-fixed split-K, fixed-order partial sums.
 * Both deterministic.  workspace >= dwm_weight_grad_workspace_bytes (may be
 * 0 -> NULL allowed).  nonfinite_flag (device int32, may be NULL) is set to 1
 * when any gradient entry is NaN/Inf.  (The data gradient is computed by the forward engines
 * on the polyphase adjoint problems, see engines.py.) */
size_t dwm_weight_grad_workspace_bytes(const dwm_desc_t* desc, int dtype, int algo);
int dwm_weight_grad(const dwm_desc_t* desc, int dtype, int algo, const void* x, const void* dy,
                    void* gw, void* workspace, size_t workspace_bytes, int32_t* nonfinite_flag,
                    void* stream);

/* Whole forward: y[N,F,OH,OW] = dwm_conv2d(x[N,C,H,W], w[F,C,r_h,r_w]).
 * nonfinite_flag (device int32, may be NULL) is set to 1 when any output
 * is NaN/Inf; the caller raises FloatingPointError after syncing. */
int dwm_conv2d_forward(const dwm_desc_t* desc, int dtype, int algo,
                       const void* x, const void* w, void* y,
                       void* workspace, size_t workspace_bytes,
                       int32_t* nonfinite_flag, void* stream);

/* Thread-local message of the last failing call on this thread. */
const char* dwm_last_error(void);
const char* dwm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DWM_B200_H */
