"""Drop-in DWM forward entry point on B200.

``dwm_conv2d(data, weights, spec, plan=None, precision=None, counter=None)``
keeps the reference signature, argument meaning, error types and messages
(reference ``pkg/src/dwmconv/engines.py:219-255``) and runs the whole
forward on the GPU through the C ABI (``include/dwm_b200.h``):

  filter transform  (U = G g Gt per part)           dwm_transforms.cu
  input transform   (V = Bt d B, polyphase gather)   dwm_transforms.cu
  transform-domain contraction + fused At.m.A,
  plan-order part sum, tile interleave, finiteness   dwm_gemm_exact.cu / dwm_gemm_tc.cu

Inputs may be NumPy arrays (copied to the GPU, result copied back as NumPy,
exactly like the reference's return type) or torch tensors (CUDA tensors stay
on the device; CPU tensors are staged through the GPU and returned on the CPU).
binary32 and binary64 are supported; the exact-rational object dtype of the
reference's test mode is not (TypeError).  There is no CPU fallback: without
the native library or a CUDA device every call raises.
"""

import ctypes
import functools
from dataclasses import dataclass

import numpy as np

from . import _native
from .convspec import ConvSpec
from .decompose import DecompositionPlan, plan_decomposition
from .transforms import precision_dtype

FLOAT_DTYPES = (np.dtype(np.float32), np.dtype(np.float64))


@dataclass(frozen=True)
class ConvOutput:
    """Result plus the elementwise-product count (reference engines.py:32-41)."""

    y: object
    flops: object = None


class FlopCounter:
    """Mutable tally of transform-domain products (reference engines.py:44-48)."""

    def __init__(self):
        self.elementwise = 0


def _torch():
    import torch
    return torch


def _is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _require_tensor4(x, name: str):
    """reference tensor.py:16-24 (torch tensors accepted as well)."""
    if _is_torch(x):
        if x.dim() != 4:
            raise ValueError(f"{name} must have 4 axes (N,C,H,W), got shape {tuple(x.shape)}")
        torch = _torch()
        if x.dtype not in (torch.float32, torch.float64):
            raise TypeError(f"{name} must be float32 or float64, got {x.dtype}")
        return x
    if not isinstance(x, np.ndarray):
        raise TypeError(f"{name} must be a numpy array, got {type(x).__name__}")
    if x.ndim != 4:
        raise ValueError(f"{name} must have 4 axes (N,C,H,W), got shape {x.shape}")
    if x.dtype == np.dtype(object):
        raise TypeError(f"{name}: the exact-rational object dtype runs only in the reference's "
                        "CPU test mode; the B200 path computes in binary32/binary64")
    if x.dtype not in FLOAT_DTYPES:
        raise TypeError(f"{name} must be float32 or float64, got {x.dtype}")
    return x


def _np_dtype(x) -> np.dtype:
    if _is_torch(x):
        return np.dtype(np.float64) if x.dtype == _torch().float64 else np.dtype(np.float32)
    return x.dtype


def _check_pair(data, weights):
    """reference engines.py:63-68"""
    _require_tensor4(data, "data")
    _require_tensor4(weights, "weights")
    if data.shape[1] != weights.shape[1]:
        raise ValueError(
            f"channel mismatch: data has {data.shape[1]}, weights have {weights.shape[1]}")


def _zeros_like_io(ref, shape, dt, out=None):
    """Zeros of ``shape`` in the caller's container type (NumPy, or torch on
    the reference tensor's device) -- the result of an empty contraction."""
    if out is not None:
        out.zero_()
        return out
    if _is_torch(ref):
        torch = _torch()
        tdt = torch.float64 if np.dtype(dt) == np.dtype(np.float64) else torch.float32
        return torch.zeros(shape, dtype=tdt, device=ref.device)
    return np.zeros(shape, dtype=dt)


def _workspace(nbytes: int, device):
    """Per-call V/U scratch from torch's stream-ordered caching allocator,
    allocated on the *current* stream (callers run under
    ``torch.cuda.stream(s)``): a later call on another stream can never be
    handed this block while this call's kernels still use it, and two calls
    on two streams never share one."""
    torch = _torch()
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)


def _aligned(t):
    """The tensor itself when its base is 16-byte aligned, else an aligned copy
    (a view with an odd storage offset); the C ABI's workspace-style operands
    and the kernels' vector paths want 16-byte bases."""
    return t if t.data_ptr() % 16 == 0 else t.clone()


_SMALL_WORKSPACE = 256 << 20


def _batch_chunk(lib, desc, code, algo_code, spec, dev, budget=None) -> int:
    """Largest batch chunk whose workspace fits the device memory budget
    (free memory plus torch's cached-but-unused blocks, with 20 % headroom);
    the whole batch when it fits."""
    n = desc.n
    need = lib.dwm_workspace_bytes(desc, code, algo_code)
    if budget is None and need <= _SMALL_WORKSPACE:
        return max(n, 1)  # no device-memory query on the small-problem path
    if budget is None:
        torch = _torch()
        free, _ = torch.cuda.mem_get_info(dev)
        cached = torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
        budget = int(0.8 * (free + cached))
    if need <= budget or n <= 1:
        return max(n, 1)
    one = lib.dwm_workspace_bytes(_native.make_desc(1, desc.c, desc.h, desc.w, desc.f, spec.kernel,
                                                    spec.stride, spec.pad), code, algo_code)
    return int(max(1, min(n, budget // max(one, 1))))


def _as_spec(spec) -> ConvSpec:
    """Accept the reference's own ``ConvSpec`` (or any object with kernel /
    stride / pad) as well as ours: both normalise to the same int tuples
    (reference convspec.py:19-28)."""
    if isinstance(spec, ConvSpec):
        return spec
    try:
        return ConvSpec(kernel=spec.kernel, stride=spec.stride, pad=spec.pad)
    except AttributeError:
        raise TypeError(f"spec must be a ConvSpec, got {type(spec).__name__}") from None


def _check_plan(plan, spec: ConvSpec) -> None:
    """reference engines.py:233-236: a caller-supplied plan must be the plan
    for ``spec``.  Works for the reference's ``DecompositionPlan`` (fields
    ``spec`` and ``parts`` only, decompose.py:52-57) and ours."""
    try:
        pspec = _as_spec(plan.spec)
    except TypeError:
        pspec = None
    if pspec != spec:
        raise ValueError("plan was built for a different ConvSpec")


def _axis_parts_of(plan):
    """Row and column axis parts of a row-major cross-product plan, derived
    from ``plan.parts`` (the only part list the reference's plan has)."""
    parts = [((p.row.origin, p.row.step, p.row.count), (p.col.origin, p.col.step, p.col.count))
             for p in plan.parts]
    rows, cols = [], []
    for r, c in parts:
        if r not in rows:
            rows.append(r)
        if r == parts[0][0]:
            cols.append(c)
    if parts != [(r, c) for r in rows for c in cols]:
        raise ValueError("plan parts are not the row-major cross product of its axis parts")
    return rows, cols


@functools.lru_cache(maxsize=256)
def _cached_plan(spec: ConvSpec) -> DecompositionPlan:
    return plan_decomposition(spec)


@functools.lru_cache(maxsize=256)
def _cached_desc_key(n, c, h, w, f, kernel, stride, pad):
    d = _native.make_desc(n, c, h, w, f, kernel, stride, pad)
    # the native planner must agree with the host planner for this spec (checked once per geometry)
    _check_plan_matches(_cached_plan(ConvSpec(kernel=kernel, stride=stride, pad=pad)), d)
    return d


def _cached_desc(n, c, h, w, f, spec: ConvSpec):
    """Descriptor per geometry (read-only once built: the C ABI takes it by const pointer)."""
    return _cached_desc_key(n, c, h, w, f, spec.kernel, spec.stride, spec.pad)


def _check_plan_matches(plan, desc) -> None:
    rows, cols = _axis_parts_of(plan)
    if rows != desc.axis("row") or cols != desc.axis("col"):
        raise ValueError(f"plan parts {rows}/{cols} differ from the plan for this ConvSpec "
                         f"{desc.axis('row')}/{desc.axis('col')}")


def dwm_conv2d(data, weights, spec: ConvSpec, plan: DecompositionPlan = None,
               precision=None, counter: FlopCounter = None, *, algo: str = "auto",
               check_finite: bool = True, out=None, stream=None):
    """Decomposed Winograd convolution for any kernel size and stride, on B200.

    Same contract as the reference (engines.py:219-255): pads once, runs every
    plan part as a stride-1 F(2, <=3) Winograd convolution, sums parts in plan
    order, raises FloatingPointError on non-finite output.  Keyword-only
    extras: ``algo`` ("auto" | "exact" | "tc"), ``check_finite`` (skip the
    device->host flag read for fully asynchronous use), ``out`` (preallocated
    CUDA output tensor) and ``stream`` (torch.cuda.Stream; default current).
    """
    _check_pair(data, weights)
    spec = _as_spec(spec)
    if tuple(weights.shape[2:]) != spec.kernel:
        raise ValueError(f"weights taps {tuple(weights.shape[2:])} do not match kernel {spec.kernel}")
    own_plan = plan is None
    if own_plan:
        plan = _cached_plan(spec)
    else:
        _check_plan(plan, spec)
    dt = _np_dtype(data) if precision is None else precision_dtype(precision)
    n, c, h, w = (int(s) for s in data.shape)
    f = int(weights.shape[0])
    oh, ow = spec.out_dims(h, w)  # geometry errors with the reference's message
    if n == 0 or c == 0 or f == 0:
        # empty batch / filters -> empty output; no input channels -> zeros (the
        # empty sum), exactly as the reference's NumPy path returns
        if counter is not None:
            counter.elementwise += flops_dwm(plan, (oh, ow))
        return _zeros_like_io(data, (n, f, oh, ow), dt, out)

    torch = _torch()
    lib = _native.load()
    # host-side planning first (pure C++, no device): the native planner's
    # axis parts must be the caller's plan
    desc = _cached_desc(n, c, h, w, f, spec)
    if not own_plan:
        _check_plan_matches(plan, desc)
    if not torch.cuda.is_available():
        raise _native.NativeError("dwm_conv2d needs a CUDA device (B200); there is no CPU fallback")
    tdt = torch.float64 if dt == np.dtype(np.float64) else torch.float32
    code = _native.DWM_F64 if tdt == torch.float64 else _native.DWM_F32

    from_numpy = not _is_torch(data)
    host_in = from_numpy or not data.is_cuda
    dev = (data.device if (not from_numpy and data.is_cuda)
           else torch.device("cuda", torch.cuda.current_device()))
    oh, ow = desc.oh, desc.ow
    if out is not None:
        if not _is_torch(out) or tuple(out.shape) != (n, f, oh, ow) or out.dtype != tdt \
                or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous {(n, f, oh, ow)} {tdt} tensor")
        if host_in and out.is_cuda:
            raise ValueError("out must be a host tensor when data is on the host")
        if not host_in and out.device != dev:
            raise ValueError(f"out must be on {dev} (the device of data), got {out.device}")
    algo_code = _native.ALGOS[algo]

    with torch.cuda.device(dev):
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        # every allocation, conversion, launch and the flag read are ordered
        # on s (temporaries come from s's pool of the caching allocator)
        with torch.cuda.stream(s):
            w_d = _aligned((torch.from_numpy(np.ascontiguousarray(weights)) if not _is_torch(weights)
                            else weights).to(dev, dtype=tdt).contiguous())
            flag = torch.zeros(1, dtype=torch.int32, device=dev) if check_finite else None
            if host_in:
                x_h = (torch.from_numpy(np.ascontiguousarray(data)) if from_numpy else data.contiguous())
                if x_h.dtype != tdt:
                    x_h = x_h.to(tdt)
                y_h = out if out is not None else torch.empty((n, f, oh, ow), dtype=tdt, pin_memory=True)
                _forward_host(lib, desc, code, algo_code, spec, x_h, w_d, y_h, flag, s, dev)
                y_res = y_h
            else:
                x_d = data.to(dev, dtype=tdt).contiguous()
                y_d = out if out is not None else torch.empty((n, f, oh, ow), dtype=tdt, device=dev)
                # images are independent: when the V workspace of the whole batch
                # would not fit, run it in batch chunks (same bits per image)
                chunk = _batch_chunk(lib, desc, code, algo_code, spec, dev)
                for b0 in range(0, n, chunk):
                    b1 = min(n, b0 + chunk)
                    dk = desc if (b0, b1) == (0, n) else _native.make_desc(
                        b1 - b0, c, h, w, f, spec.kernel, spec.stride, spec.pad)
                    ws_bytes = lib.dwm_workspace_bytes(dk, code, algo_code)
                    ws = _workspace(ws_bytes, dev)
                    st = lib.dwm_conv2d_forward(dk, code, algo_code, x_d[b0].data_ptr(), w_d.data_ptr(),
                                                y_d[b0].data_ptr(), ws.data_ptr(), ws_bytes,
                                                flag.data_ptr() if flag is not None else None,
                                                s.cuda_stream)
                    _native.check(st, "dwm_conv2d_forward")
                    del ws
                y_res = y_d
            if counter is not None:
                counter.elementwise += int(lib.dwm_elementwise_count(desc))
            # .item() copies on s and waits for it
            if check_finite and int(flag.item()) != 0:
                raise FloatingPointError("dwm_conv2d produced non-finite values")
    if from_numpy:
        return y_res.numpy()
    return y_res


_SIDE_STREAMS = {}


def _side_streams(dev):
    torch = _torch()
    if dev not in _SIDE_STREAMS:
        _SIDE_STREAMS[dev] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    return _SIDE_STREAMS[dev]


def _host_chunks(lib, desc, code, algo_code, n, dev):
    """Chunk boundaries for the host-buffer forward.  The first chunk's H2D
    and the last chunk's D2H are exposed, so chunks are small (about n/8) --
    but each chunk is one launch of the persistent tcgen05 GEMM, whose work
    items (128 tiles x 64 filters) run in waves of one per SM: a chunk that
    fills 2.65 waves idles 12 % of the GEMM in its last wave.  For that
    engine the smallest chunk size in [n/16, n/6] with the least wave
    quantisation is picked (cfg4 11x11, N = 512: 48-image chunks = exactly
    2 waves; cfg5, N = 1024: 72 images = 3 waves)."""
    if n < 2:
        return [0, n]
    k = max(1, round(n / 8))
    if lib.dwm_select_algo(desc, code, algo_code) == _native.DWM_ALGO_TC:
        torch = _torch()
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        tiles_img = desc.tiles // desc.n
        nblk = -(-desc.f // 64)

        def waste(kk):
            items = -(-kk * tiles_img // 128) * nblk
            waves = -(-items // sms)
            return waves * sms / items

        cands = range(max(1, n // 16), max(2, n // 6) + 1)
        k = min(cands, key=lambda kk: (round(waste(kk), 3), kk))
    bounds = list(range(0, n, k)) + [n]
    return bounds


def _forward_host(lib, desc, code, algo_code, spec, x_h, w_d, y_h, flag, s, dev):
    """Host-resident input/output: the batch is cut into chunks whose
    host->device copy, forward and device->host copy run on three streams, so
    PCIe traffic in both directions overlaps the kernels (images are
    independent, so chunking changes no result bit).  Runs with ``s`` current."""
    torch = _torch()
    n = x_h.shape[0]
    bounds = _host_chunks(lib, desc, code, algo_code, n, dev)
    x_d = torch.empty(x_h.shape, dtype=x_h.dtype, device=dev)
    y_d = torch.empty(y_h.shape, dtype=y_h.dtype, device=dev)
    s_in, s_out = _side_streams(dev)
    s_in.wait_stream(s)
    s_out.wait_stream(s)
    descs = [_native.make_desc(b1 - b0, desc.c, desc.h, desc.w, desc.f, spec.kernel, spec.stride, spec.pad)
             for b0, b1 in zip(bounds, bounds[1:])]
    # one engine and one filter transform for all chunks (the engine choice
    # does not depend on the batch; resolve it once so U's layout matches)
    sel = lib.dwm_select_algo(descs[0], code, algo_code)
    if sel < 0:
        _native.check(lib.dwm_conv2d_forward(descs[0], code, algo_code, None, None, None, None, 0, None,
                                             s.cuda_stream), "dwm_conv2d_forward")
    u = _workspace(lib.dwm_filter_bytes(descs[0], code, sel), dev)
    _native.check(lib.dwm_prepare_filter(descs[0], code, sel, w_d.data_ptr(), u.data_ptr(), s.cuda_stream),
                  "dwm_prepare_filter")
    ws_bytes = max(lib.dwm_workspace_bytes(dk, code, sel) for dk in descs)
    ws = _workspace(ws_bytes, dev)
    for (b0, b1), dk in zip(zip(bounds, bounds[1:]), descs):
        with torch.cuda.stream(s_in):
            x_d[b0:b1].copy_(x_h[b0:b1], non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(s_in)
        s.wait_event(ev_in)
        # chunk bases need only natural alignment (the kernels take their
        # vector paths only on 16-/8-byte aligned bases)
        st = lib.dwm_conv2d_forward_prepared(dk, code, sel, x_d[b0].data_ptr(), u.data_ptr(),
                                             y_d[b0].data_ptr(), ws.data_ptr(), ws_bytes,
                                             flag.data_ptr() if flag is not None else None, s.cuda_stream)
        _native.check(st, "dwm_conv2d_forward_prepared")
        ev_done = torch.cuda.Event()
        ev_done.record(s)
        s_out.wait_event(ev_done)
        with torch.cuda.stream(s_out):
            y_h[b0:b1].copy_(y_d[b0:b1], non_blocking=True)
    # device buffers go back to the caching allocator only after the side
    # streams are done with them
    x_d.record_stream(s_in)
    y_d.record_stream(s_out)
    s.wait_stream(s_out)
    s_out.synchronize()


def _to_device(x, dev, tdt):
    torch = _torch()
    t = torch.from_numpy(np.ascontiguousarray(x)) if not _is_torch(x) else x
    return t.to(dev, dtype=tdt).contiguous()


def _phase_geometry(rho: int, s: int, r: int, pad_lo: int, size: int, out: int):
    """One axis of input-gradient phase rho (positions p = s*i + rho of the
    padded input).  Taps with k = rho (mod s) reach it: T = ceil((r-rho)/s).
    Returns (T, i_min, m, pad_lo', pad_hi') for the stride-1 correlation of
    grad_out with the reversed sub-kernel that yields rows i_min .. i_min+m-1
    (negative pads mean cropping grad_out)."""
    taps = max(0, -(-(r - rho) // s))
    i_min = -(-(pad_lo - rho) // s)
    i_max = (pad_lo + size - 1 - rho) // s
    m = i_max - i_min + 1
    lo = taps - 1 - i_min
    hi = m - 1 + taps - out - lo
    return taps, i_min, m, lo, hi


def _data_grad_polyphase(dy, wt, spec: ConvSpec, hw, algo: str, stream, flag):
    """Input gradient as s_h*s_w stride-1 DWM forwards (one per output phase):
    grad_pad[s*i + rho] = sum_t dY[i - t] * w[rho + s*t]  -- the DWM stride
    split applied to the adjoint, so no zero-inserted (dilated) grad_out and no
    multiply by an inserted zero.  Phases write disjoint positions.

    Each phase's filter is the channel-transposed, tap-reversed sub-kernel
    w[:, :, rho::s_h, sig::s_w]: its transform reads it in place through
    element strides (dwm_prepare_filter_strided), nothing is materialised.
    A stride-1 problem has one phase covering the whole gradient, written
    directly; the non-finite flag of every phase accumulates in ``flag``
    (one device->host read for the whole backward)."""
    torch = _torch()
    lib = _native.load()
    n, f, oh, ow = dy.shape
    c = wt.shape[1]
    h, w = hw
    r_h, r_w = spec.kernel
    s_h, s_w = spec.stride
    top, _, left, _ = spec.pad
    code = _native.DWM_F64 if dy.dtype == torch.float64 else _native.DWM_F32
    algo_code = _native.ALGOS[algo]
    rows = [_phase_geometry(rho, s_h, r_h, top, h, oh) for rho in range(s_h)]
    cols = [_phase_geometry(sig, s_w, r_w, left, w, ow) for sig in range(s_w)]
    covered = all(g[0] > 0 for g in rows + cols)
    gd = (torch.empty if covered else torch.zeros)((n, c, h, w), dtype=dy.dtype, device=dy.device)
    wc = wt.contiguous()
    for rho, (tr, i0, m, pt, pb) in enumerate(rows):
        if tr == 0 or m <= 0:
            continue
        for sig, (tc, j0, mc, pl, pr) in enumerate(cols):
            if tc == 0 or mc <= 0:
                continue
            src = dy
            if min(pt, pb, pl, pr) < 0:
                src = dy[:, :, max(0, -pt):oh - max(0, -pb), max(0, -pl):ow - max(0, -pr)].contiguous()
            adj = ConvSpec(kernel=(tr, tc), stride=(1, 1),
                           pad=(max(0, pt), max(0, pb), max(0, pl), max(0, pr)))
            # the phase problem: data = grad_out (F channels), filters = C
            desc = _native.make_desc(n, f, src.shape[2], src.shape[3], c, adj.kernel, adj.stride, adj.pad)
            # element (c', f', i, j) of the reversed sub-kernel is
            # w[f', c', rho + s_h*(tr-1-i), sig + s_w*(tc-1-j)]
            base = wc[0, 0, rho + s_h * (tr - 1), sig + s_w * (tc - 1)]
            strides = (ctypes.c_int64 * 4)(r_h * r_w, c * r_h * r_w, -s_h * r_w, -s_w)
            u = _workspace(lib.dwm_filter_bytes(desc, code, algo_code), dy.device)
            _native.check(lib.dwm_prepare_filter_strided(desc, code, algo_code, base.data_ptr(), strides,
                                                         u.data_ptr(), stream.cuda_stream),
                          "dwm_prepare_filter_strided")
            r0, c0 = s_h * i0 + rho - top, s_w * j0 + sig - left
            direct = (s_h, s_w) == (1, 1) and (r0, c0) == (0, 0) and (desc.oh, desc.ow) == (h, w)
            y = gd if direct else torch.empty((n, c, desc.oh, desc.ow), dtype=dy.dtype, device=dy.device)
            ws_bytes = lib.dwm_workspace_bytes(desc, code, algo_code)
            ws = _workspace(ws_bytes, dy.device)
            _native.check(lib.dwm_conv2d_forward_prepared(desc, code, algo_code, src.data_ptr(), u.data_ptr(),
                                                          y.data_ptr(), ws.data_ptr(), ws_bytes, flag.data_ptr(),
                                                          stream.cuda_stream), "dwm_conv2d_forward_prepared")
            if not direct:
                gd[:, :, r0::s_h, c0::s_w] = y
    return gd


def dwm_backward(grad_out, plan: DecompositionPlan, data, weights, precision=None, *,
                 algo: str = "auto", stream=None, need_data: bool = True, need_weights: bool = True,
                 wgrad_algo: str = "auto"):
    """Gradients of ``dwm_conv2d`` w.r.t. data and weights on B200 (SURVEY §8f
    rank 1; reference ``engines.py:342-399``, same signature, checks and
    messages).  Returns ``(grad_data, grad_weights)``.

    B200 design (not the reference's per-part Winograd adjoint):

    * data gradient -- the adjoint of a stride-s correlation splits, by the
      same stride decomposition DWM uses, into s_h*s_w stride-1 correlations
      of ``grad_out`` with reversed, channel-transposed sub-kernels
      w[:, :, rho::s, sig::s], one per phase of the input gradient.  Each is
      a DWM forward, so it runs on the forward engines (tcgen05 3xTF32 when
      the channel counts allow) with no zero-inserted grad_out.
    * weight gradient -- ``dwm_weight_grad`` (C ABI), ``wgrad_algo``:
      "tc" (AUTO for float32, C % 32 == 0, C, F >= 64) works in the Winograd
      domain like the reference: per frequency dU = V^T DM on tcgen05
      (3xTF32, K = tiles), then G^T dU G placed at each part's taps;
      "exact" is an implicit-im2col CUDA-core GEMM with a geometry-fixed
      split-K.  Both deterministic.

    Both are exact in exact arithmetic, so results agree with the reference's
    to rounding (binary64: <= 1e-10 absolute, the reference's own criterion).
    ``need_data`` / ``need_weights`` = False skip a gradient (returned as None).
    """
    _check_pair(data, weights)
    _require_tensor4(grad_out, "grad_out")
    spec = _as_spec(plan.spec)
    if tuple(weights.shape[2:]) != spec.kernel:
        raise ValueError(f"weights taps {tuple(weights.shape[2:])} do not match kernel {spec.kernel}")
    n, c, h, w = (int(s) for s in data.shape)
    f = int(weights.shape[0])
    oh, ow = spec.out_dims(h, w)
    if tuple(grad_out.shape) != (n, f, oh, ow):
        raise ValueError(f"grad_out shape {tuple(grad_out.shape)} != {(n, f, oh, ow)}")
    dt = _np_dtype(grad_out) if precision is None else precision_dtype(precision)
    if n == 0 or c == 0 or f == 0:
        # empty contraction: both gradients are zeros (the reference's result)
        gd = _zeros_like_io(grad_out, (n, c, h, w), dt) if need_data else None
        gw = _zeros_like_io(grad_out, (f, c, *spec.kernel), dt) if need_weights else None
        return gd, gw

    torch = _torch()
    lib = _native.load()
    if not torch.cuda.is_available():
        raise _native.NativeError("dwm_backward needs a CUDA device (B200); there is no CPU fallback")
    tdt = torch.float64 if dt == np.dtype(np.float64) else torch.float32
    code = _native.DWM_F64 if tdt == torch.float64 else _native.DWM_F32
    cuda_in = _is_torch(grad_out) and grad_out.is_cuda
    dev = grad_out.device if cuda_in else torch.device("cuda", torch.cuda.current_device())
    r_h, r_w = spec.kernel

    with torch.cuda.device(dev):
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        with torch.cuda.stream(s):
            dy = _to_device(grad_out, dev, tdt)
            x = _to_device(data, dev, tdt)
            wt = _to_device(weights, dev, tdt)

            # one device flag for every kernel of the backward, read once
            flag = torch.zeros(1, dtype=torch.int32, device=dev)
            gw = None
            if need_weights:
                gw = torch.empty((f, c, r_h, r_w), dtype=tdt, device=dev)
                desc = _native.make_desc(n, c, h, w, f, spec.kernel, spec.stride, spec.pad)
                wg_algo = _native.ALGOS[wgrad_algo]
                wg_bytes = int(lib.dwm_weight_grad_workspace_bytes(desc, code, wg_algo))
                wg_ws = _workspace(wg_bytes, dev)
                _native.check(lib.dwm_weight_grad(desc, code, wg_algo, x.data_ptr(), dy.data_ptr(),
                                                  gw.data_ptr(), wg_ws.data_ptr(), wg_bytes, flag.data_ptr(),
                                                  s.cuda_stream),
                              "dwm_weight_grad")
            gd = _data_grad_polyphase(dy, wt, spec, (h, w), algo, s, flag) if need_data else None
            if int(flag.item()) != 0:
                raise FloatingPointError("dwm_backward produced non-finite values")
    if not _is_torch(grad_out):
        return tuple(None if g is None else g.cpu().numpy() for g in (gd, gw))
    if not cuda_in:
        return tuple(None if g is None else g.cpu() for g in (gd, gw))
    return gd, gw


def convolve(data, weights, spec: ConvSpec, algo: str = "dwm", precision=None,
             plan: DecompositionPlan = None) -> ConvOutput:
    """Instrumented run by name (reference engines.py:402-421); only "dwm"
    is on the B200 path -- "direct"/"winograd" are the reference's CPU
    baselines and are out of scope here."""
    if algo != "dwm":
        raise ValueError(f"unknown algorithm {algo!r} for the B200 path; only 'dwm' is implemented "
                         "(direct and classic Winograd are the reference's CPU baselines)")
    counter = FlopCounter()
    y = dwm_conv2d(data, weights, spec, plan=plan, precision=precision, counter=counter)
    return ConvOutput(y=y, flops=counter.elementwise)


def flops_dwm(plan: DecompositionPlan, out) -> int:
    """tiles * sum over parts of alpha_r * alpha_c (reference flops.py:107-119;
    the transform terms are zero because F(2,<=3) is shift-free)."""
    oh, ow = out
    tiles = -(-oh // 2) * -(-ow // 2)
    return tiles * sum((p.row.count + 1) * (p.col.count + 1) for p in plan.parts)
