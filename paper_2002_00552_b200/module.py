"""Plug-and-play DWM convolution operator for PyTorch.

The paper presents DWM as a drop-in replacement for a framework's conv
operator; the reference ships only the NumPy functions.
This module is that operator on B200:

* ``DWMConv2dFunction`` -- ``torch.autograd.Function``: forward through the C
  ABI (``dwm_conv2d_forward_prepared``), backward through ``dwm_backward``.
* ``DWMConv2d`` -- ``torch.nn.Module`` with ``nn.Conv2d``-like arguments
  (plus asymmetric 4-tuple padding, which the reference's ConvSpec allows).
* ``FilterCache`` -- the transformed filters U = G g G^T per weight version.
  Weights stay in the spatial domain (reference SPEC.md:327); U is a cache
  keyed by (storage pointer, ``tensor._version``, dtype, engine layout,
  geometry), so an optimizer step (an in-place update bumps ``_version``)
  invalidates it and inference re-uses it across calls.  The cache is used
  only when no gradient flows to the weights (inference, ``torch.no_grad``,
  frozen weights): during training U changes every step anyway, and writes
  through ``tensor.data`` (as ``gradcheck`` does) bypass version tracking.

CUDA tensors only: there is no CPU fallback.
"""

import weakref

import numpy as np
import torch

from . import _native
from .convspec import ConvSpec
from .decompose import DecompositionPlan, plan_decomposition
from .engines import _aligned, _as_spec, _check_plan, _workspace, dwm_backward


class FilterCache:
    """Transformed-filter cache, one entry per live weight tensor.

    An entry holds a weak reference to the caller's weight tensor and the
    ``_version`` it was transformed at; a hit needs the very same tensor
    object (not merely the same address: the caching allocator reuses
    addresses, and a fresh tensor starts at version 0) at the same version.
    Non-contiguous and inference tensors are never cached (their contiguous
    copy is a new object per call; an inference tensor has no version)."""

    def __init__(self, capacity: int = 64):
        self.capacity = capacity
        self._entries = {}
        self.hits = 0
        self.misses = 0

    def clear(self):
        self._entries.clear()

    @staticmethod
    def transform(lib, desc, code: int, algo_code: int, w: torch.Tensor, stream) -> torch.Tensor:
        w = w.contiguous()
        u = torch.empty(max(int(lib.dwm_filter_bytes(desc, code, algo_code)), 1), dtype=torch.uint8,
                        device=w.device)
        _native.check(lib.dwm_prepare_filter(desc, code, algo_code, w.data_ptr(), u.data_ptr(),
                                             stream.cuda_stream), "dwm_prepare_filter")
        return u

    @staticmethod
    def cacheable(w: torch.Tensor) -> bool:
        return w.is_contiguous() and not w.is_inference() and w.data_ptr() % 16 == 0

    def get(self, lib, desc, code: int, algo_code: int, w: torch.Tensor, stream) -> torch.Tensor:
        """U for the caller's weight tensor ``w`` (before any .contiguous())."""
        if not self.cacheable(w):
            self.misses += 1
            return self.transform(lib, desc, code, algo_code, w, stream)
        tc = lib.dwm_select_algo(desc, code, algo_code) == _native.ALGOS["tc"]
        key = (w.data_ptr(), w.device, w.dtype, tc, desc.f, desc.c, desc.r_h, desc.r_w,
               desc.s_h, desc.s_w)
        hit = self._entries.get(key)
        if hit is not None and hit[0]() is w and hit[1] == w._version:
            self.hits += 1
            return hit[2]
        self.misses += 1
        u = self.transform(lib, desc, code, algo_code, w, stream)
        self._entries.pop(key, None)
        if len(self._entries) >= self.capacity:
            self._entries.pop(next(iter(self._entries)))
        self._entries[key] = (weakref.ref(w), w._version, u)
        return u


DEFAULT_CACHE = FilterCache()


def _forward(x: torch.Tensor, w: torch.Tensor, spec: ConvSpec, algo: str, cache: FilterCache,
             check_finite: bool) -> torch.Tensor:
    if not (x.is_cuda and w.is_cuda):
        raise _native.NativeError("DWM operator needs CUDA tensors (B200); there is no CPU fallback")
    if x.dtype != w.dtype or x.dtype not in (torch.float32, torch.float64):
        raise TypeError(f"data and weights must share float32/float64, got {x.dtype} and {w.dtype}")
    if x.dim() != 4 or w.dim() != 4:
        raise ValueError("data and weights must have 4 axes (N,C,H,W) / (F,C,r_h,r_w)")
    if x.shape[1] != w.shape[1]:
        raise ValueError(f"channel mismatch: data has {x.shape[1]}, weights have {w.shape[1]}")
    if tuple(w.shape[2:]) != spec.kernel:
        raise ValueError(f"weights taps {tuple(w.shape[2:])} do not match kernel {spec.kernel}")
    if x.shape[0] == 0 or x.shape[1] == 0 or w.shape[0] == 0:
        oh, ow = spec.out_dims(int(x.shape[2]), int(x.shape[3]))
        return torch.zeros((x.shape[0], w.shape[0], oh, ow), dtype=x.dtype, device=x.device)
    lib = _native.load()
    code = _native.DWM_F64 if x.dtype == torch.float64 else _native.DWM_F32
    algo_code = _native.ALGOS[algo]
    n, c, h, wd = (int(v) for v in x.shape)
    desc = _native.make_desc(n, c, h, wd, int(w.shape[0]), spec.kernel, spec.stride, spec.pad)
    x = _aligned(x.contiguous())
    with torch.cuda.device(x.device):
        s = torch.cuda.current_stream(x.device)
        if cache is None:
            u = FilterCache.transform(lib, desc, code, algo_code, _aligned(w.contiguous()), s)
        else:
            u = cache.get(lib, desc, code, algo_code, w, s)
        y = torch.empty((n, desc.f, desc.oh, desc.ow), dtype=x.dtype, device=x.device)
        ws_bytes = int(lib.dwm_workspace_bytes(desc, code, algo_code))
        ws = _workspace(ws_bytes, x.device)
        flag = torch.zeros(1, dtype=torch.int32, device=x.device) if check_finite else None
        _native.check(lib.dwm_conv2d_forward_prepared(
            desc, code, algo_code, x.data_ptr(), u.data_ptr(), y.data_ptr(), ws.data_ptr(), ws_bytes,
            flag.data_ptr() if flag is not None else None, s.cuda_stream), "dwm_conv2d_forward_prepared")
        if check_finite and int(flag.item()) != 0:
            raise FloatingPointError("dwm_conv2d produced non-finite values")
    return y


def _cache_for(w: torch.Tensor, cache: FilterCache):
    """Bypass the cache while gradients flow to the weights (decided outside
    autograd.Function.forward, which always runs with grad mode off)."""
    return None if (torch.is_grad_enabled() and w.requires_grad) else cache


class DWMConv2dFunction(torch.autograd.Function):
    """y = dwm_conv2d(x, w) with gradients from ``dwm_backward``."""

    @staticmethod
    def forward(ctx, x, w, spec, plan, algo, cache, check_finite):
        ctx.save_for_backward(x, w)
        ctx.plan, ctx.algo = plan, algo
        return _forward(x, w, spec, algo, cache, check_finite)

    @staticmethod
    def backward(ctx, grad_y):
        x, w = ctx.saved_tensors
        gd, gw = dwm_backward(grad_y.contiguous(), ctx.plan, x.contiguous(), w.contiguous(),
                              algo=ctx.algo, need_data=ctx.needs_input_grad[0],
                              need_weights=ctx.needs_input_grad[1])
        return gd, gw, None, None, None, None, None


def dwm_conv2d_op(x: torch.Tensor, w: torch.Tensor, spec: ConvSpec, plan: DecompositionPlan = None,
                  algo: str = "auto", cache: FilterCache = None, check_finite: bool = True):
    """Functional, differentiable DWM convolution of CUDA tensors."""
    spec = _as_spec(spec)
    if plan is None:
        plan = plan_decomposition(spec)
    else:
        _check_plan(plan, spec)
    return DWMConv2dFunction.apply(x, w, spec, plan, algo, _cache_for(w, cache or DEFAULT_CACHE),
                                   check_finite)


def _pair(v):
    if isinstance(v, int):
        return (v, v)
    v = tuple(int(t) for t in v)
    if len(v) != 2:
        raise ValueError(f"expected an int or a pair, got {v}")
    return v


def _pad4(p):
    if isinstance(p, int):
        return (p,) * 4
    p = tuple(int(t) for t in p)
    if len(p) == 2:
        return (p[0], p[0], p[1], p[1])
    if len(p) == 4:
        return p
    raise ValueError(f"padding must be an int, (pad_h, pad_w) or (top, bottom, left, right), got {p}")


class DWMConv2d(torch.nn.Module):
    """``nn.Conv2d``-style layer computed by DWM on B200 (groups=1, dilation=1)."""

    def __init__(self, in_channels: int, out_channels: int, kernel_size, stride=1, padding=0,
                 bias: bool = True, algo: str = "auto", check_finite: bool = True, device=None,
                 dtype=None):
        super().__init__()
        self.spec = ConvSpec(kernel=_pair(kernel_size), stride=_pair(stride), pad=_pad4(padding))
        self.plan = plan_decomposition(self.spec)
        if algo not in _native.ALGOS:
            raise ValueError(f"unknown engine {algo!r}; choose one of {sorted(_native.ALGOS)}")
        self.algo = algo
        self.check_finite = check_finite
        self.cache = FilterCache(capacity=4)
        fk = dict(device=device, dtype=dtype)
        self.weight = torch.nn.Parameter(torch.empty((out_channels, in_channels, *self.spec.kernel), **fk))
        self.bias = torch.nn.Parameter(torch.empty(out_channels, **fk)) if bias else None
        self.reset_parameters()

    def reset_parameters(self):
        fan_in = self.weight.shape[1] * self.spec.kernel[0] * self.spec.kernel[1]
        bound = 1.0 / np.sqrt(fan_in)
        with torch.no_grad():
            self.weight.uniform_(-bound, bound)
            if self.bias is not None:
                self.bias.uniform_(-bound, bound)

    def forward(self, x):
        y = DWMConv2dFunction.apply(x, self.weight, self.spec, self.plan, self.algo,
                                    _cache_for(self.weight, self.cache), self.check_finite)
        if self.bias is not None:
            y = y + self.bias.view(1, -1, 1, 1)
        return y

    def extra_repr(self):
        return (f"{self.weight.shape[1]}, {self.weight.shape[0]}, kernel={self.spec.kernel}, "
                f"stride={self.spec.stride}, pad={self.spec.pad}, algo={self.algo}, "
                f"bias={self.bias is not None}")
