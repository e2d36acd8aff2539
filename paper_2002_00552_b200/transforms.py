"""Winograd F(2, r) transform constants for the DWM hot path (r <= 3).

The decomposition never produces a sub-kernel with more than three taps per
axis (``decompose.py:60-70`` of the reference), so the hot path only ever
needs F(2,1), F(2,2) and F(2,3).  The reference builds them by an exact
Cook-Toom construction (``pkg/src/dwmconv/transforms.py:129-208``) over the
node prefix (0, 1, -1) with "infinity" last and an identity pass-through for
r == 1 (``transforms.py:163-167``).  Those three triples are tabulated here as
exact rationals; every entry is in {0, +-1, +-1/2}, so they are exactly
representable in binary32 and the CUDA kernels hard-code them as add/sub and
exact halvings (see ``csrc/dwm_transforms.cuh``).

Layouts follow the reference: y = a_t @ ((g @ filt) * (b_t @ data)),
``g`` is alpha x r, ``b_t`` alpha x alpha, ``a_t`` 2 x alpha, alpha = r + 1.
"""

from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache

import numpy as np

_H = Fraction(1, 2)

# (points, g, b_t, a_t) per tap count; rows ordered node 0, 1, -1, then infinity.
_TABLE = {
    1: ((),
        ((1,), (1,)),
        ((1, 0), (0, 1)),
        ((1, 0), (0, 1))),
    2: ((0, 1),
        ((1, 0), (1, 1), (0, 1)),
        ((1, -1, 0), (0, 1, 0), (0, 1, -1)),
        ((1, 1, 0), (0, 1, -1))),
    3: ((0, 1, -1),
        ((1, 0, 0), (_H, _H, _H), (_H, -_H, _H), (0, 0, 1)),
        ((1, 0, -1, 0), (0, 1, 1, 0), (0, -1, 1, 0), (0, 1, 0, -1)),
        ((1, 1, 1, 0), (0, 1, -1, -1))),
}

_DTYPE_ALIASES = {
    "binary32": np.float32, "f32": np.float32, "float32": np.float32,
    "binary64": np.float64, "f64": np.float64, "float64": np.float64,
}


def precision_dtype(precision) -> np.dtype:
    """Map binary32/binary64/f32/f64 names or dtypes to a numpy dtype
    (reference ``transforms.py:52-62``)."""
    if isinstance(precision, str):
        try:
            return np.dtype(_DTYPE_ALIASES[precision])
        except KeyError:
            raise ValueError(f"unknown precision {precision!r}") from None
    dt = np.dtype(precision)
    if dt not in (np.dtype(np.float32), np.dtype(np.float64)):
        raise ValueError(f"unsupported precision {precision!r}")
    return dt


@dataclass(frozen=True)
class TransformSet:
    """Exact transform triple for F(m, r) (reference ``transforms.py:65-79``)."""

    m: int
    r: int
    points: tuple
    g: tuple
    b_t: tuple
    a_t: tuple

    @property
    def alpha(self) -> int:
        return self.m + self.r - 1


def _frac_rows(rows):
    return tuple(tuple(Fraction(x) for x in row) for row in rows)


@lru_cache(maxsize=None)
def get_transform(r: int, m: int = 2) -> TransformSet:
    """F(2, r) for r in 1..3, bit-for-bit the reference's ``get_transform``
    (``transforms.py:268-271``) restricted to the sizes DWM emits."""
    if m != 2 or r not in _TABLE:
        raise ValueError(
            f"the B200 DWM path ships F(2,1..3) only; F({m},{r}) is never produced "
            "by the decomposition planner")
    points, g, b_t, a_t = _TABLE[r]
    return TransformSet(m=2, r=r, points=tuple(Fraction(p) for p in points),
                        g=_frac_rows(g), b_t=_frac_rows(b_t), a_t=_frac_rows(a_t))


def to_float(ts: TransformSet, precision) -> dict:
    """Float rendering of a transform triple (reference ``transforms.py:250-258``)."""
    dt = precision_dtype(precision)
    conv = lambda rows: np.array([[float(x) for x in row] for row in rows], dtype=dt)
    return {"g": conv(ts.g), "b_t": conv(ts.b_t), "a_t": conv(ts.a_t)}
