"""ctypes binding of ``include/dwm_b200.h`` (the C ABI in ``_lib/libdwm_b200.so``).

There is deliberately no fallback: if the library or a CUDA device is
missing, every compute entry point raises ``RuntimeError``.
"""

import ctypes
import os
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libdwm_b200.so"

DWM_MAX_AXIS_PARTS = 16

DWM_OK, DWM_EINVAL_SHAPE, DWM_EINVAL_DTYPE, DWM_NONFINITE, DWM_ECUDA, DWM_EUNSUPPORTED = range(6)
DWM_F32, DWM_F64 = 0, 1
DWM_ALGO_AUTO, DWM_ALGO_EXACT, DWM_ALGO_TC, DWM_ALGO_SMALL_C = 0, 1, 2, 3
ALGOS = {"auto": DWM_ALGO_AUTO, "exact": DWM_ALGO_EXACT, "tc": DWM_ALGO_TC, "small_c": DWM_ALGO_SMALL_C}
ALGO_NAMES = {v: k for k, v in ALGOS.items()}

# every symbol include/dwm_b200.h declares (checked by tests/test_native_abi.py)
EXPORTED_SYMBOLS = (
    "dwm_desc_init", "dwm_elementwise_count", "dwm_workspace_bytes", "dwm_select_algo",
    "dwm_filter_transform", "dwm_input_transform", "dwm_gemm_output", "dwm_input_transform_ranged",
    "dwm_gemm_output_tc", "dwm_range_bytes",
    "dwm_filter_bytes", "dwm_prepare_filter", "dwm_prepare_filter_strided", "dwm_conv2d_forward_prepared", "dwm_weight_grad_workspace_bytes", "dwm_weight_grad",
    "dwm_conv2d_small_c", "dwm_conv2d_forward", "dwm_last_error", "dwm_version",
)


class AxisPartC(ctypes.Structure):
    _fields_ = [("origin", ctypes.c_int32), ("step", ctypes.c_int32), ("count", ctypes.c_int32)]


class DescC(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32), ("c", ctypes.c_int32), ("h", ctypes.c_int32),
        ("w", ctypes.c_int32), ("f", ctypes.c_int32),
        ("r_h", ctypes.c_int32), ("r_w", ctypes.c_int32),
        ("s_h", ctypes.c_int32), ("s_w", ctypes.c_int32),
        ("pad_top", ctypes.c_int32), ("pad_bottom", ctypes.c_int32),
        ("pad_left", ctypes.c_int32), ("pad_right", ctypes.c_int32),
        ("oh", ctypes.c_int32), ("ow", ctypes.c_int32),
        ("th", ctypes.c_int32), ("tw", ctypes.c_int32),
        ("n_row_parts", ctypes.c_int32), ("n_col_parts", ctypes.c_int32),
        ("row_parts", AxisPartC * DWM_MAX_AXIS_PARTS),
        ("col_parts", AxisPartC * DWM_MAX_AXIS_PARTS),
        ("row_freqs", ctypes.c_int32), ("col_freqs", ctypes.c_int32),
        ("num_freqs", ctypes.c_int32),
        ("tiles", ctypes.c_int64),
    ]

    def axis(self, which: str) -> list:
        parts = self.row_parts if which == "row" else self.col_parts
        n = self.n_row_parts if which == "row" else self.n_col_parts
        return [(parts[i].origin, parts[i].step, parts[i].count) for i in range(n)]


_lib = None


class NativeError(RuntimeError):
    pass


def library_path() -> Path:
    return _LIB_PATH


def load(required: bool = True):
    """Load the native library (once).  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        if not required:
            return None
        raise NativeError(
            f"DWM native library not built: {_LIB_PATH} is missing "
            "(run `python -m paper_2002_00552_b200.build`); there is no CPU fallback")
    lib = ctypes.CDLL(str(_LIB_PATH))
    P, I, S = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    D = ctypes.POINTER(DescC)
    lib.dwm_desc_init.argtypes = [D] + [I] * 13
    lib.dwm_desc_init.restype = I
    lib.dwm_elementwise_count.argtypes = [D]
    lib.dwm_elementwise_count.restype = ctypes.c_int64
    lib.dwm_workspace_bytes.argtypes = [D, I, I]
    lib.dwm_workspace_bytes.restype = S
    lib.dwm_select_algo.argtypes = [D, I, I]
    lib.dwm_select_algo.restype = I
    lib.dwm_filter_transform.argtypes = [D, I, P, P, P]
    lib.dwm_filter_transform.restype = I
    lib.dwm_input_transform.argtypes = [D, I, P, P, P]
    lib.dwm_input_transform.restype = I
    lib.dwm_gemm_output.argtypes = [D, I, I, P, P, P, P, P, S, P]
    lib.dwm_gemm_output.restype = I
    lib.dwm_range_bytes.argtypes = [D]
    lib.dwm_range_bytes.restype = ctypes.c_size_t
    lib.dwm_input_transform_ranged.argtypes = [D, P, P, P, P]
    lib.dwm_input_transform_ranged.restype = I
    lib.dwm_gemm_output_tc.argtypes = [D, P, P, P, P, P, P]
    lib.dwm_gemm_output_tc.restype = I
    lib.dwm_filter_bytes.argtypes = [D, I, I]
    lib.dwm_filter_bytes.restype = ctypes.c_size_t
    lib.dwm_prepare_filter.argtypes = [D, I, I, P, P, P]
    lib.dwm_prepare_filter.restype = I
    lib.dwm_prepare_filter_strided.argtypes = [D, I, I, P, ctypes.POINTER(ctypes.c_int64), P, P]
    lib.dwm_prepare_filter_strided.restype = I
    lib.dwm_conv2d_forward_prepared.argtypes = [D, I, I, P, P, P, P, ctypes.c_size_t, P, P]
    lib.dwm_conv2d_forward_prepared.restype = I
    lib.dwm_weight_grad_workspace_bytes.argtypes = [D, I, I]
    lib.dwm_weight_grad_workspace_bytes.restype = S
    lib.dwm_weight_grad.argtypes = [D, I, I, P, P, P, P, S, P, P]
    lib.dwm_weight_grad.restype = I
    lib.dwm_conv2d_small_c.argtypes = [D, P, P, P, P, P]
    lib.dwm_conv2d_small_c.restype = I
    lib.dwm_conv2d_forward.argtypes = [D, I, I, P, P, P, P, S, P, P]
    lib.dwm_conv2d_forward.restype = I
    lib.dwm_last_error.argtypes = []
    lib.dwm_last_error.restype = ctypes.c_char_p
    lib.dwm_version.argtypes = []
    lib.dwm_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def last_error() -> str:
    return load().dwm_last_error().decode(errors="replace")


def check(status: int, what: str = "dwm"):
    """Map a dwm_status to the reference's exception types (engines/tensor.py)."""
    if status == DWM_OK:
        return
    msg = last_error()
    if status == DWM_EINVAL_SHAPE:
        raise ValueError(msg)
    if status == DWM_EINVAL_DTYPE:
        raise TypeError(msg)
    if status == DWM_NONFINITE:
        raise FloatingPointError(msg)
    if status == DWM_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise NativeError(f"{what}: {msg}")


def make_desc(n, c, h, w, f, kernel, stride, pad) -> DescC:
    d = DescC()
    check(load().dwm_desc_init(ctypes.byref(d), n, c, h, w, f, kernel[0], kernel[1],
                               stride[0], stride[1], *pad), "dwm_desc_init")
    return d
