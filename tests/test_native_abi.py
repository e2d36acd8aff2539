"""The C-ABI library loads here (no GPU needed for its host-side entry
points), exports every symbol include/dwm_b200.h declares, and its C++
planner agrees with the Python planner and the reference's plans."""

import ctypes
import json
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from paper_2002_00552_b200 import ConvSpec, flops_dwm, plan_decomposition, plan_to_json
from paper_2002_00552_b200 import _native


def _declared_symbols():
    text = (ROOT / "include" / "dwm_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\s*\*?\s*(dwm_[a-z0-9_]+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    declared = _declared_symbols()
    assert set(declared) == set(_native.EXPORTED_SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.dwm_version().startswith(b"dwm_b200")


def test_native_planner_matches_reference_golden_plans():
    golden = json.loads((GOLDEN / "plans.json").read_text())
    for g in golden:
        d = _native.make_desc(1, 1, 40, 40, 1, g["kernel"], g["stride"], (0, 0, 0, 0))
        rows = []
        cols = []
        for p in g["parts"]:
            r = (p["row"]["origin"], p["row"]["step"], p["row"]["count"])
            c = (p["col"]["origin"], p["col"]["step"], p["col"]["count"])
            rows.append(r) if r not in rows else None
            cols.append(c) if c not in cols else None
        assert d.axis("row") == rows and d.axis("col") == cols
        plan = plan_decomposition(ConvSpec(kernel=g["kernel"], stride=g["stride"]))
        assert d.num_freqs == plan.num_frequencies
        assert d.n_row_parts * d.n_col_parts == len(g["parts"])


@pytest.mark.parametrize("shape,kernel,stride,pad", [
    ((256, 3, 224, 224), (7, 7), (2, 2), (3, 3, 3, 3)),
    ((256, 3, 227, 227), (11, 11), (4, 4), (0, 0, 0, 0)),
    ((512, 256, 28, 28), (11, 11), (1, 1), (5, 5, 5, 5)),
    ((1, 2, 7, 9), (3, 3), (1, 1), (0, 0, 0, 0)),
    ((2, 3, 13, 11), (4, 6), (2, 1), (1, 2, 0, 3)),
])
def test_native_geometry_and_counter(shape, kernel, stride, pad):
    spec = ConvSpec(kernel=kernel, stride=stride, pad=pad)
    n, c, h, w = shape
    d = _native.make_desc(n, c, h, w, 8, kernel, stride, pad)
    oh, ow = spec.out_dims(h, w)
    assert (d.oh, d.ow) == (oh, ow)
    assert (d.th, d.tw) == (-(-oh // 2), -(-ow // 2))
    assert d.tiles == n * d.th * d.tw
    lib = _native.load()
    # FlopCounter semantics: engines.py:190-191 == flops.flops_dwm
    assert lib.dwm_elementwise_count(d) == flops_dwm(plan_decomposition(spec), (oh, ow))
    ws = lib.dwm_workspace_bytes(d, _native.DWM_F32, _native.DWM_ALGO_EXACT)
    assert ws >= 4 * d.num_freqs * d.tiles * c


def test_native_errors_mirror_reference_messages():
    with pytest.raises(ValueError, match="too small"):
        _native.make_desc(1, 1, 3, 3, 1, (5, 5), (1, 1), (0, 0, 0, 0))
    with pytest.raises(ValueError, match="kernel must be two positive integers"):
        _native.make_desc(1, 1, 8, 8, 1, (0, 3), (1, 1), (0, 0, 0, 0))
    with pytest.raises(ValueError, match="stride must be two positive integers"):
        _native.make_desc(1, 1, 8, 8, 1, (3, 3), (0, 1), (0, 0, 0, 0))
    with pytest.raises(ValueError, match="pad must be four non-negative"):
        _native.make_desc(1, 1, 8, 8, 1, (3, 3), (1, 1), (0, -1, 0, 0))
    with pytest.raises(NotImplementedError, match="more than 16 parts"):
        _native.make_desc(1, 1, 80, 80, 1, (60, 3), (1, 1), (0, 0, 0, 0))
    lib = _native.load()
    d = _native.DescC()
    st = lib.dwm_conv2d_forward(d, 7, 0, None, None, None, None, 0, None, None)
    assert st == _native.DWM_EINVAL_DTYPE
    st = lib.dwm_conv2d_forward(d, 0, 0, None, None, None, None, 0, None, None)
    assert st == _native.DWM_EINVAL_SHAPE and b"not initialised" in lib.dwm_last_error()


def test_workspace_pointers_must_be_16_byte_aligned():
    """V/U/workspace operands are read by 16-byte vectors and TMA: a
    misaligned pointer is rejected before any launch (no device needed)."""
    from paper_2002_00552_b200 import _native
    lib = _native.load()
    d = _native.make_desc(1, 32, 8, 8, 16, (3, 3), (1, 1), (1, 1, 1, 1))
    st = lib.dwm_filter_transform(d, _native.DWM_F32, 0x1000, 0x1004, None)
    assert st == _native.DWM_EINVAL_SHAPE and "16-byte aligned" in _native.last_error()
    st = lib.dwm_input_transform(d, _native.DWM_F32, 0x1000, 0x1008, None)
    assert st == _native.DWM_EINVAL_SHAPE


def test_range_stage_api_validation():
    """The tcgen05 range-carrying stage pair: one uint32 max|x| slot per image
    (16-byte rounded), a NULL or misaligned range is rejected before any
    launch (no device needed)."""
    from paper_2002_00552_b200 import _native
    lib = _native.load()
    d = _native.make_desc(5, 64, 8, 8, 64, (3, 3), (1, 1), (1, 1, 1, 1))
    assert lib.dwm_range_bytes(d) == 32  # 5 images x 4 bytes, rounded to 16
    st = lib.dwm_input_transform_ranged(d, 0x1000, 0x2000, None, None)
    assert st == _native.DWM_EINVAL_SHAPE and "range" in _native.last_error()
    st = lib.dwm_input_transform_ranged(d, 0x1000, 0x2000, 0x3004, None)
    assert st == _native.DWM_EINVAL_SHAPE and "16-byte aligned" in _native.last_error()
    st = lib.dwm_gemm_output_tc(d, 0x2000, 0x3000, None, 0x4000, None, None)
    assert st == _native.DWM_EINVAL_SHAPE and "range" in _native.last_error()
    # the forward's workspace holds V, U and the range slots
    ws = lib.dwm_workspace_bytes(d, _native.DWM_F32, _native.DWM_ALGO_TC)
    assert ws >= 4 * d.num_freqs * d.tiles * 64 + lib.dwm_filter_bytes(d, _native.DWM_F32, _native.DWM_ALGO_TC) + 32
