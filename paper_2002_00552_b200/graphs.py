"""CUDA-Graph path for small, latency-bound DWM convolutions.

For a single 56x56 image (BASELINE configs[0], cfg1) the three kernels of a
forward run in ~75 us while the host side of an eager ``dwm_conv2d`` call
(argument checks, descriptor, workspace and flag allocation, three launches,
the flag read) costs about as much again.  ``DWMConvGraph`` captures the
whole forward -- filter transform, input transform, contraction with the
fused output transform, non-finite flag -- for one fixed geometry into a CUDA
graph over static device buffers; a call is two copies into those buffers
and one graph launch.  Same kernels, same bits as ``dwm_conv2d``.
"""

import numpy as np
import torch

from . import _native
from .convspec import ConvSpec
from .engines import _as_spec


class DWMConvGraph:
    """Captured ``dwm_conv2d`` for fixed shapes (x: N,C,H,W; w: F,C,r_h,r_w).

    ``graph(x, w)`` copies ``x``/``w`` (CUDA or host tensors, or NumPy arrays)
    into the static inputs, replays the graph on the current stream and
    returns the static output (valid until the next call; pass ``out=`` or
    clone it to keep it).  ``check_finite`` raises FloatingPointError like
    the eager call (one 4-byte device->host read)."""

    def __init__(self, x_shape, w_shape, spec: ConvSpec, dtype=torch.float32, device=None, algo: str = "auto",
                 check_finite: bool = True):
        spec = _as_spec(spec)
        if not torch.cuda.is_available():
            raise _native.NativeError("DWMConvGraph needs a CUDA device (B200); there is no CPU fallback")
        self.lib = _native.load()
        self.spec, self.check_finite = spec, check_finite
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        n, c, h, w = (int(v) for v in x_shape)
        f = int(w_shape[0])
        if int(w_shape[1]) != c:
            raise ValueError(f"channel mismatch: data has {c}, weights have {w_shape[1]}")
        if tuple(int(v) for v in w_shape[2:]) != spec.kernel:
            raise ValueError(f"weights taps {tuple(w_shape[2:])} do not match kernel {spec.kernel}")
        self.code = _native.DWM_F64 if dtype == torch.float64 else _native.DWM_F32
        self.algo = _native.ALGOS[algo]
        self.desc = _native.make_desc(n, c, h, w, f, spec.kernel, spec.stride, spec.pad)
        d = self.desc
        kw = dict(dtype=dtype, device=self.device)
        self.x = torch.zeros((n, c, h, w), **kw)
        self.w = torch.zeros((f, c, *spec.kernel), **kw)
        self.y = torch.empty((n, f, d.oh, d.ow), **kw)
        self.ws_bytes = int(self.lib.dwm_workspace_bytes(d, self.code, self.algo))
        self.ws = torch.empty(max(self.ws_bytes, 16), dtype=torch.uint8, device=self.device)
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.device(self.device), torch.cuda.stream(side):
            self._launch(side)  # warm-up outside the capture (module load, attributes, tensor maps)
            side.synchronize()
            with torch.cuda.graph(self.graph, stream=side):
                self.flag.zero_()
                self._launch(side)
        torch.cuda.current_stream(self.device).wait_stream(side)

    def _launch(self, stream):
        _native.check(self.lib.dwm_conv2d_forward(self.desc, self.code, self.algo, self.x.data_ptr(),
                                                  self.w.data_ptr(), self.y.data_ptr(), self.ws.data_ptr(),
                                                  self.ws_bytes, self.flag.data_ptr(), stream.cuda_stream),
                      "dwm_conv2d_forward")

    @staticmethod
    def _copy_in(dst, src):
        if isinstance(src, np.ndarray):
            src = torch.from_numpy(np.ascontiguousarray(src))
        if src.data_ptr() != dst.data_ptr():
            dst.copy_(src, non_blocking=True)

    def __call__(self, x, w, out=None):
        """Replay on the current stream of the graph's device.  With
        ``check_finite=False`` nothing synchronizes: the result (and a host
        ``out``) is ready once that stream is."""
        with torch.cuda.device(self.device):
            self._copy_in(self.x, x)
            self._copy_in(self.w, w)
            self.graph.replay()
            y = self.y
            if out is not None:
                out.copy_(y, non_blocking=True)
                y = out
            if self.check_finite and int(self.flag.item()) != 0:
                raise FloatingPointError("dwm_conv2d produced non-finite values")
        return y
