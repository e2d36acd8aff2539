// dwm_capi.cu -- C ABI: planner, validation, workspace sizing and dispatch.
//
// The planner is a C++ restatement of the reference's decompose.py:60-114
// (stride-residue split, empty residues dropped, greedy blocks of 3 plus a
// remainder, low taps first; 2-D plan = row-major cross product).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "dwm_common.cuh"
#include "dwm_kernels.h"

namespace dwm {

static thread_local char g_err[512] = "";

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  return fail(DWM_ECUDA, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
              cudaGetErrorString(e), what, file, line);
}

namespace {
std::mutex g_launch_mu;
std::map<std::pair<const void*, int>, size_t> g_smem_set;           // (kernel, device) -> bytes set
std::map<std::tuple<const void*, int, int, size_t>, int> g_occupancy;  // (kernel, device, threads, smem)
int g_sms[64];
}  // namespace

int device_sm_count(int* sms) {
  int dev = 0;
  DWM_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_launch_mu);
  int& v = g_sms[dev & 63];
  if (!v) DWM_CUDA_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
  *sms = v;
  return DWM_OK;
}

int ensure_dynamic_smem(const void* kernel, size_t smem) {
  int dev = 0;
  DWM_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_launch_mu);
  size_t& have = g_smem_set[{kernel, dev}];
  if (smem > have || have == 0) {
    DWM_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    have = smem > have ? smem : have;
  }
  return DWM_OK;
}

int cached_occupancy(const void* kernel, int threads, size_t smem, int* per_sm) {
  int dev = 0;
  DWM_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_launch_mu);
  auto key = std::make_tuple(kernel, dev, threads, smem);
  auto it = g_occupancy.find(key);
  if (it == g_occupancy.end()) {
    int v = 0;
    DWM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel, threads, smem));
    it = g_occupancy.emplace(key, v).first;
  }
  *per_sm = it->second;
  return DWM_OK;
}

// decompose.py:73-100 -- stride split, then size split of each residue run.
static int plan_axis(int taps, int stride, dwm_axis_part_t* out, int* n_out) {
  int n = 0;
  for (int residue = 0; residue < stride; ++residue) {
    const int run = (taps - residue + stride - 1) / stride;  // ceil, <= 0 if empty
    if (run <= 0) continue;
    int first = 0;
    for (int left = run; left > 0;) {
      const int block = left >= 3 ? 3 : left;
      if (n >= DWM_MAX_AXIS_PARTS)
        return fail(DWM_EUNSUPPORTED,
                    "decomposition of %d taps at stride %d needs more than %d parts per axis",
                    taps, stride, DWM_MAX_AXIS_PARTS);
      out[n].origin = residue + stride * first;
      out[n].step = stride;
      out[n].count = block;
      ++n;
      first += block;
      left -= block;
    }
  }
  *n_out = n;
  return DWM_OK;
}

}  // namespace dwm

using namespace dwm;

extern "C" {

const char* dwm_last_error(void) { return g_err; }

const char* dwm_version(void) { return "dwm_b200 0.1.0 (sm_100a)"; }

int dwm_desc_init(dwm_desc_t* d, int n, int c, int h, int w, int f, int r_h, int r_w,
                  int s_h, int s_w, int pad_top, int pad_bottom, int pad_left, int pad_right) {
  if (!d) return fail(DWM_EINVAL_SHAPE, "descriptor pointer is NULL");
  std::memset(d, 0, sizeof(*d));
  // convspec.py:23-28
  if (r_h < 1 || r_w < 1)
    return fail(DWM_EINVAL_SHAPE, "kernel must be two positive integers, got (%d, %d)", r_h, r_w);
  if (s_h < 1 || s_w < 1)
    return fail(DWM_EINVAL_SHAPE, "stride must be two positive integers, got (%d, %d)", s_h, s_w);
  if (pad_top < 0 || pad_bottom < 0 || pad_left < 0 || pad_right < 0)
    return fail(DWM_EINVAL_SHAPE, "pad must be four non-negative integers, got (%d, %d, %d, %d)",
                pad_top, pad_bottom, pad_left, pad_right);
  if (n < 1 || c < 1 || h < 1 || w < 1 || f < 1)
    return fail(DWM_EINVAL_SHAPE, "empty tensor: data (%d, %d, %d, %d), filters %d", n, c, h, w, f);
  // convspec.py:34-44
  const int oh = (h + pad_top + pad_bottom - r_h) / s_h + 1;
  const int ow = (w + pad_left + pad_right - r_w) / s_w + 1;
  if (h + pad_top + pad_bottom < r_h || w + pad_left + pad_right < r_w || oh < 1 || ow < 1)
    return fail(DWM_EINVAL_SHAPE,
                "input %dx%d with pad (%d, %d, %d, %d) is too small for kernel (%d, %d) stride (%d, %d)",
                h, w, pad_top, pad_bottom, pad_left, pad_right, r_h, r_w, s_h, s_w);
  d->n = n; d->c = c; d->h = h; d->w = w; d->f = f;
  d->r_h = r_h; d->r_w = r_w; d->s_h = s_h; d->s_w = s_w;
  d->pad_top = pad_top; d->pad_bottom = pad_bottom; d->pad_left = pad_left; d->pad_right = pad_right;
  d->oh = oh; d->ow = ow;
  d->th = (oh + 1) / 2; d->tw = (ow + 1) / 2;
  int st = plan_axis(r_h, s_h, d->row_parts, &d->n_row_parts);
  if (st) return st;
  st = plan_axis(r_w, s_w, d->col_parts, &d->n_col_parts);
  if (st) return st;
  d->row_freqs = 0;
  for (int i = 0; i < d->n_row_parts; ++i) d->row_freqs += d->row_parts[i].count + 1;
  d->col_freqs = 0;
  for (int i = 0; i < d->n_col_parts; ++i) d->col_freqs += d->col_parts[i].count + 1;
  d->num_freqs = d->row_freqs * d->col_freqs;
  d->tiles = (int64_t)n * d->th * d->tw;
  return DWM_OK;
}

int64_t dwm_elementwise_count(const dwm_desc_t* d) {
  return d ? (int64_t)d->th * d->tw * d->num_freqs : 0;
}

int dwm_select_algo(const dwm_desc_t* d, int dtype, int algo) {
  if (!d) return -1;
  const bool tc_ok = dtype == DWM_F32 && tc_gemm_supported(*d);
  const bool sc_ok = dtype == DWM_F32 && small_c_supported(*d);
  switch (algo) {
    case DWM_ALGO_EXACT: return DWM_ALGO_EXACT;
    case DWM_ALGO_TC: return tc_ok ? DWM_ALGO_TC : -1;
    case DWM_ALGO_SMALL_C: return sc_ok ? DWM_ALGO_SMALL_C : -1;
    case DWM_ALGO_AUTO:
      if (sc_ok) return DWM_ALGO_SMALL_C;
      if (tc_ok && d->c >= 64 && d->f >= 32) return DWM_ALGO_TC;
      return DWM_ALGO_EXACT;
    default: return -1;
  }
}

static size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

static size_t v_bytes_of(const dwm_desc_t* d, size_t es) {
  return (size_t)d->num_freqs * (size_t)d->tiles * (size_t)d->c * es;
}

size_t dwm_workspace_bytes(const dwm_desc_t* d, int dtype, int algo) {
  if (!d) return 0;
  const size_t es = dtype == DWM_F64 ? 8 : 4;
  const int sel = dwm_select_algo(d, dtype, algo);
  size_t u = (size_t)d->num_freqs * (size_t)d->f * (size_t)d->c * es;
  if (sel == DWM_ALGO_TC) u = tc_filter_bytes(*d);  // stacked, scaled fp16 hi/lo split of U
  const size_t v = sel == DWM_ALGO_SMALL_C ? 0 : v_bytes_of(d, es);
  // TC: + the input transform's per-image max|x| slots (after V and U)
  return round_up(v, 256) + round_up(u, 256) + (sel == DWM_ALGO_TC ? xmax_bytes(*d) : 0);
}

// Workspace-type buffers (V, U, ws) are read with 16-byte vector loads and
// TMA, which need 16-byte aligned bases; x, w and y only need natural
// alignment (the kernels pick vector paths at run time when they can).
static int check_aligned(const void* p, const char* name) {
  if ((uintptr_t)p & 15u) return fail(DWM_EINVAL_SHAPE, "%s must be 16-byte aligned (got %p)", name, p);
  return DWM_OK;
}

static int check_common(const dwm_desc_t* d, int dtype) {
  if (!d) return fail(DWM_EINVAL_SHAPE, "descriptor pointer is NULL");
  if (dtype != DWM_F32 && dtype != DWM_F64)
    return fail(DWM_EINVAL_DTYPE, "dtype must be float32 or float64, got code %d", dtype);
  if (d->num_freqs <= 0 || d->tiles <= 0)
    return fail(DWM_EINVAL_SHAPE, "descriptor is not initialised (call dwm_desc_init)");
  return DWM_OK;
}

int dwm_filter_transform(const dwm_desc_t* d, int dtype, const void* w, void* U, void* stream) {
  if (int st = check_common(d, dtype)) return st;
  if (int st = check_aligned(U, "U")) return st;
  return launch_filter_transform(*d, dtype, w, U, (cudaStream_t)stream);
}

int dwm_input_transform(const dwm_desc_t* d, int dtype, const void* x, void* V, void* stream) {
  if (int st = check_common(d, dtype)) return st;
  if (int st = check_aligned(V, "V")) return st;
  return launch_input_transform(*d, dtype, x, V, (cudaStream_t)stream);
}

static int bad_algo(const dwm_desc_t* d, int algo) {
  return fail(DWM_EUNSUPPORTED,
              "engine %d not available for this geometry/dtype (tcgen05: float32, C %% 32 == 0; "
              "small-C: float32, C <= 4; got C=%d F=%d)", algo, d->c, d->f);
}

int dwm_gemm_output(const dwm_desc_t* d, int dtype, int algo, const void* V, const void* U,
                    void* y, int32_t* flag, void* ws, size_t ws_bytes, void* stream) {
  if (int st = check_common(d, dtype)) return st;
  if (int st = check_aligned(V, "V")) return st;
  if (int st = check_aligned(U, "U")) return st;
  int sel = dwm_select_algo(d, dtype, algo);
  if (sel == DWM_ALGO_SMALL_C) sel = algo == DWM_ALGO_AUTO ? DWM_ALGO_EXACT : -1;
  if (sel < 0) return bad_algo(d, algo);
  if (sel == DWM_ALGO_TC) {
    if (ws_bytes > 0)
      if (int st = check_aligned(ws, "workspace")) return st;
    return launch_gemm_tc(*d, V, U, y, flag, nullptr, ws, ws_bytes, (cudaStream_t)stream);
  }
  return launch_gemm_exact(*d, dtype, V, U, y, flag, (cudaStream_t)stream);
}

size_t dwm_range_bytes(const dwm_desc_t* d) { return d ? xmax_bytes(*d) : 0; }

int dwm_input_transform_ranged(const dwm_desc_t* d, const void* x, void* V, uint32_t* range, void* stream) {
  if (int st = check_common(d, DWM_F32)) return st;
  if (!range) return fail(DWM_EINVAL_SHAPE, "range pointer is NULL (dwm_range_bytes(desc) bytes of device memory)");
  if (int st = check_aligned(V, "V")) return st;
  if (int st = check_aligned(range, "range")) return st;
  return launch_input_transform(*d, DWM_F32, x, V, (cudaStream_t)stream, range);
}

int dwm_gemm_output_tc(const dwm_desc_t* d, const void* V, const void* U, const uint32_t* range, void* y,
                       int32_t* flag, void* stream) {
  if (int st = check_common(d, DWM_F32)) return st;
  if (!range) return fail(DWM_EINVAL_SHAPE, "range pointer is NULL (fill it with dwm_input_transform_ranged)");
  if (int st = check_aligned(V, "V")) return st;
  if (int st = check_aligned(U, "U")) return st;
  if (int st = check_aligned(range, "range")) return st;
  if (!tc_gemm_supported(*d)) return bad_algo(d, DWM_ALGO_TC);
  return launch_gemm_tc(*d, V, U, y, flag, range, nullptr, 0, (cudaStream_t)stream);
}

static int wgrad_select(const dwm_desc_t* d, int dtype, int algo) {
  const bool tc_ok = dtype == DWM_F32 && wgrad_tc_supported(*d);
  switch (algo) {
    case DWM_ALGO_AUTO: return tc_ok ? DWM_ALGO_TC : DWM_ALGO_EXACT;
    case DWM_ALGO_EXACT: return DWM_ALGO_EXACT;
    case DWM_ALGO_TC: return tc_ok ? DWM_ALGO_TC : -1;
    default: return -1;
  }
}

size_t dwm_weight_grad_workspace_bytes(const dwm_desc_t* d, int dtype, int algo) {
  if (!d || d->num_freqs <= 0) return 0;
  const int sel = wgrad_select(d, dtype, algo);
  if (sel == DWM_ALGO_TC) return wgrad_tc_workspace_bytes(*d);
  const int splits = weight_grad_splits(*d);
  if (splits <= 1) return 0;
  return (size_t)splits * d->f * d->c * d->r_h * d->r_w * (dtype == DWM_F64 ? 8 : 4);
}

int dwm_weight_grad(const dwm_desc_t* d, int dtype, int algo, const void* x, const void* dy, void* gw, void* ws,
                    size_t ws_bytes, int32_t* flag, void* stream) {
  if (int st = check_common(d, dtype)) return st;
  if (ws_bytes > 0)
    if (int st = check_aligned(ws, "workspace")) return st;
  const int sel = wgrad_select(d, dtype, algo);
  if (sel < 0)
    return fail(DWM_EUNSUPPORTED, "weight-gradient engine %d not available (tcgen05: float32, C %% 32 == 0, "
                "C >= 64, F >= 64; got C=%d F=%d)", algo, d->c, d->f);
  if (sel == DWM_ALGO_TC) return launch_wgrad_tc(*d, x, dy, gw, ws, ws_bytes, flag, (cudaStream_t)stream);
  return launch_weight_grad(*d, dtype, x, dy, gw, ws, ws_bytes, flag, (cudaStream_t)stream);
}

int dwm_conv2d_small_c(const dwm_desc_t* d, const void* x, const void* U, void* y, int32_t* flag,
                       void* stream) {
  if (int st = check_common(d, DWM_F32)) return st;
  if (int st = check_aligned(U, "U")) return st;
  if (!small_c_supported(*d)) return bad_algo(d, DWM_ALGO_SMALL_C);
  return launch_small_c(*d, x, U, y, flag, (cudaStream_t)stream);
}

int dwm_conv2d_forward(const dwm_desc_t* d, int dtype, int algo, const void* x, const void* w,
                       void* y, void* ws, size_t ws_bytes, int32_t* flag, void* stream) {
  if (int st = check_common(d, dtype)) return st;
  const int sel = dwm_select_algo(d, dtype, algo);
  if (sel < 0) return bad_algo(d, algo);
  const size_t need = dwm_workspace_bytes(d, dtype, sel);
  if (!ws || ws_bytes < need)
    return fail(DWM_EINVAL_SHAPE, "workspace too small: %zu bytes given, %zu needed", ws_bytes, need);
  if (int st2 = check_aligned(ws, "workspace")) return st2;
  const size_t es = dtype == DWM_F64 ? 8 : 4;
  char* base = (char*)ws;
  void* V = base;
  void* U = base + (sel == DWM_ALGO_SMALL_C ? 0 : round_up(v_bytes_of(d, es), 256));
  cudaStream_t s = (cudaStream_t)stream;
  int st;
  if (sel == DWM_ALGO_TC) {
    if ((st = launch_filter_transform_f16split(*d, w, U, s))) return st;
  } else {
    if ((st = launch_filter_transform(*d, dtype, w, U, s))) return st;
  }
  if (sel == DWM_ALGO_SMALL_C) return launch_small_c(*d, x, U, y, flag, s);
  if (sel == DWM_ALGO_TC) {
    uint32_t* xmax = (uint32_t*)(base + round_up(v_bytes_of(d, es), 256) + round_up(tc_filter_bytes(*d), 256));
    if ((st = launch_input_transform(*d, dtype, x, V, s, xmax))) return st;
    return launch_gemm_tc(*d, V, U, y, flag, xmax, nullptr, 0, s);
  }
  if ((st = launch_input_transform(*d, dtype, x, V, s))) return st;
  return launch_gemm_exact(*d, dtype, V, U, y, flag, s);
}

size_t dwm_filter_bytes(const dwm_desc_t* d, int dtype, int algo) {
  if (!d) return 0;
  const size_t es = dtype == DWM_F64 ? 8 : 4;
  size_t u = (size_t)d->num_freqs * (size_t)d->f * (size_t)d->c * es;
  if (dwm_select_algo(d, dtype, algo) == DWM_ALGO_TC) u = tc_filter_bytes(*d);
  return u;
}

int dwm_prepare_filter(const dwm_desc_t* d, int dtype, int algo, const void* w, void* U, void* stream) {
  if (int st = check_common(d, dtype)) return st;
  if (int st = check_aligned(U, "U")) return st;
  const int sel = dwm_select_algo(d, dtype, algo);
  if (sel < 0) return bad_algo(d, algo);
  if (sel == DWM_ALGO_TC) return launch_filter_transform_f16split(*d, w, U, (cudaStream_t)stream);
  return launch_filter_transform(*d, dtype, w, U, (cudaStream_t)stream);
}

int dwm_prepare_filter_strided(const dwm_desc_t* d, int dtype, int algo, const void* w, const int64_t* strides,
                               void* U, void* stream) {
  if (int st = check_common(d, dtype)) return st;
  if (!strides) return fail(DWM_EINVAL_SHAPE, "strides pointer is NULL");
  if (int st = check_aligned(U, "U")) return st;
  const int sel = dwm_select_algo(d, dtype, algo);
  if (sel < 0) return bad_algo(d, algo);
  if (sel == DWM_ALGO_TC) return launch_filter_transform_f16split(*d, w, U, (cudaStream_t)stream, strides);
  return launch_filter_transform(*d, dtype, w, U, (cudaStream_t)stream, strides);
}

int dwm_conv2d_forward_prepared(const dwm_desc_t* d, int dtype, int algo, const void* x, const void* U,
                                void* y, void* ws, size_t ws_bytes, int32_t* flag, void* stream) {
  if (int st = check_common(d, dtype)) return st;
  const int sel = dwm_select_algo(d, dtype, algo);
  if (sel < 0) return bad_algo(d, algo);
  cudaStream_t s = (cudaStream_t)stream;
  int st0;
  if (sel == DWM_ALGO_SMALL_C) {
    if ((st0 = check_aligned(U, "U"))) return st0;
    return launch_small_c(*d, x, U, y, flag, s);
  }
  const size_t vb = v_bytes_of(d, dtype == DWM_F64 ? 8 : 4);
  const size_t need = sel == DWM_ALGO_TC ? round_up(vb, 256) + xmax_bytes(*d) : vb;
  if (!ws || ws_bytes < need)
    return fail(DWM_EINVAL_SHAPE, "workspace too small: %zu bytes given, %zu needed", ws_bytes, need);
  if ((st0 = check_aligned(ws, "workspace")) || (st0 = check_aligned(U, "U"))) return st0;
  int st;
  if (sel == DWM_ALGO_TC) {
    uint32_t* xmax = (uint32_t*)((char*)ws + round_up(vb, 256));
    if ((st = launch_input_transform(*d, dtype, x, ws, s, xmax))) return st;
    return launch_gemm_tc(*d, ws, U, y, flag, xmax, nullptr, 0, s);
  }
  if ((st = launch_input_transform(*d, dtype, x, ws, s))) return st;
  return launch_gemm_exact(*d, dtype, ws, U, y, flag, s);
}

}  // extern "C"
