"""Operator wrapper: autograd.Function / nn.Module with the
transformed-filter cache.  The numerics reference for this float layer is
torch's own conv2d in float64 (a test oracle only); tolerances:
  * binary64 forward and both gradients: max abs diff <= 1e-10 (the
    reference's FP64 criterion, test_acceptance.py:65-78 / test_engines_backward.py:96-97);
  * binary32 forward: bit-identical to ``dwm_conv2d`` (same kernels, cached U);
  * ``torch.autograd.gradcheck`` in binary64 with its default tolerances.
"""

import numpy as np
import pytest
import torch

from paper_2002_00552_b200 import (ConvSpec, DWMConv2d, FilterCache, dwm_conv2d, dwm_conv2d_op,
                                   plan_decomposition)
from paper_2002_00552_b200._native import NativeError


def test_module_geometry_cpu():
    m = DWMConv2d(3, 8, 7, stride=2, padding=3, bias=False)
    assert m.spec == ConvSpec(kernel=(7, 7), stride=(2, 2), pad=(3, 3, 3, 3))
    assert m.weight.shape == (8, 3, 7, 7) and m.bias is None
    m2 = DWMConv2d(2, 4, (3, 5), stride=(1, 2), padding=(1, 0, 2, 2))
    assert m2.spec.pad == (1, 0, 2, 2) and m2.plan.spec == m2.spec
    with pytest.raises(ValueError):
        DWMConv2d(2, 4, 3, padding=(1, 2, 3))
    with pytest.raises(ValueError):
        DWMConv2d(2, 4, 3, algo="winograd")


def test_module_rejects_cpu_tensors():
    m = DWMConv2d(2, 4, 3)
    with pytest.raises(NativeError, match="CUDA"):
        m(torch.zeros(1, 2, 8, 8))


GEOMS = [((3, 3), (1, 1), (1, 1, 1, 1), 3, 4, 9),
         ((5, 5), (2, 2), (2, 1, 0, 2), 2, 3, 11),
         ((7, 7), (2, 2), (3, 3, 3, 3), 3, 8, 14),
         ((4, 3), (3, 1), (0, 0, 1, 1), 5, 2, 10),
         ((3, 3), (1, 1), (1, 1, 1, 1), 64, 64, 8)]


@pytest.mark.gpu
@pytest.mark.parametrize("k,s,p,c,f,hw", GEOMS)
def test_op_f64_matches_torch_conv2d(cuda, k, s, p, c, f, hw):
    g = torch.Generator().manual_seed(sum(k) + c)
    x = torch.randn(2, c, hw, hw, generator=g, dtype=torch.float64).to(cuda).requires_grad_()
    w = torch.randn(f, c, *k, generator=g, dtype=torch.float64).to(cuda).requires_grad_()
    spec = ConvSpec(kernel=k, stride=s, pad=p)
    y = dwm_conv2d_op(x, w, spec)
    xp = torch.nn.functional.pad(x, (p[2], p[3], p[0], p[1]))
    y_ref = torch.nn.functional.conv2d(xp, w, stride=s)
    assert y.shape == y_ref.shape
    assert (y - y_ref).abs().max().item() <= 1e-10
    gy = torch.randn(y.shape, generator=g, dtype=torch.float64).to(cuda)
    gx, gw = torch.autograd.grad(y, (x, w), gy)
    gx_ref, gw_ref = torch.autograd.grad(y_ref, (x, w), gy)
    assert (gx - gx_ref).abs().max().item() <= 1e-10
    assert (gw - gw_ref).abs().max().item() <= 1e-10


@pytest.mark.gpu
def test_gradcheck_f64(cuda):
    spec = ConvSpec(kernel=(5, 5), stride=(2, 2), pad=(1, 1, 1, 1))
    x = torch.randn(1, 2, 9, 9, dtype=torch.float64, device=cuda, requires_grad=True)
    w = torch.randn(2, 2, 5, 5, dtype=torch.float64, device=cuda, requires_grad=True)
    assert torch.autograd.gradcheck(lambda a, b: dwm_conv2d_op(a, b, spec), (x, w))


@pytest.mark.gpu
def test_filter_cache_hits_and_invalidation(cuda):
    torch.manual_seed(0)
    m = DWMConv2d(3, 16, 7, stride=2, padding=3, bias=False).to(cuda)
    x = torch.randn(2, 3, 20, 20, device=cuda)
    with torch.no_grad():
        y1 = m(x)
        y2 = m(x)
    assert m.cache.misses == 1 and m.cache.hits == 1
    assert torch.equal(y1, y2)
    want = dwm_conv2d(x, m.weight.detach(), m.spec)
    assert torch.equal(y1, want)
    # an optimizer step updates the weights in place -> new version -> recompute U
    opt = torch.optim.SGD(m.parameters(), lr=0.1)
    m(x).square().sum().backward()
    opt.step()
    with torch.no_grad():
        y3 = m(x)
    assert m.cache.misses == 2
    assert torch.equal(y3, dwm_conv2d(x, m.weight.detach(), m.spec))
    assert not torch.equal(y3, y1)


@pytest.mark.gpu
def test_tc_layer_cache_uses_split_layout(cuda):
    torch.manual_seed(1)
    m = DWMConv2d(64, 64, 3, padding=1, bias=True).to(cuda)
    x = torch.randn(2, 64, 16, 16, device=cuda)
    with torch.no_grad():
        y = m(x)
        y2 = m(x)
    want = dwm_conv2d(x, m.weight.detach(), m.spec, algo="tc") + m.bias.view(1, -1, 1, 1)
    assert torch.equal(y, want) and torch.equal(y, y2)


@pytest.mark.gpu
def test_training_matches_nn_conv2d(cuda):
    """Same init, same data, same SGD: the DWM layer trains like nn.Conv2d
    (binary64, so the two stay equal to rounding over the steps)."""
    torch.manual_seed(2)
    ref = torch.nn.Conv2d(4, 8, 5, stride=2, padding=2, dtype=torch.float64).to(cuda)
    m = DWMConv2d(4, 8, 5, stride=2, padding=2, dtype=torch.float64).to(cuda)
    with torch.no_grad():
        m.weight.copy_(ref.weight)
        m.bias.copy_(ref.bias)
    x = torch.randn(8, 4, 16, 16, device=cuda, dtype=torch.float64)
    y_t = torch.randn(8, 8, 8, 8, device=cuda, dtype=torch.float64)
    opts = [torch.optim.SGD(mod.parameters(), lr=0.05, momentum=0.9) for mod in (ref, m)]
    for _ in range(10):
        for mod, opt in zip((ref, m), opts):
            opt.zero_grad()
            (mod(x) - y_t).square().mean().backward()
            opt.step()
    assert (m.weight - ref.weight).abs().max().item() <= 1e-10
    assert (m.bias - ref.bias).abs().max().item() <= 1e-10
    with torch.no_grad():
        assert (m(x) - ref(x)).abs().max().item() <= 1e-10


class _FakeLib:
    """Host stand-in for the native library: FilterCache.get only asks it for
    the engine selection; the transform itself is stubbed."""

    def dwm_select_algo(self, desc, code, algo):
        return 2


def _desc():
    from types import SimpleNamespace
    return SimpleNamespace(f=4, c=3, r_h=3, r_w=3, s_h=1, s_w=1)


def test_filter_cache_identity_version_and_uncacheable(monkeypatch):
    """The cache hits only for the same live tensor object at the same
    version: a new tensor at a recycled address, an in-place update, a
    non-contiguous weight and an inference tensor all re-transform."""
    import torch
    from paper_2002_00552_b200.module import FilterCache
    calls = []

    def fake_transform(lib, desc, code, algo_code, w, stream):
        calls.append(w.data_ptr())
        return torch.tensor([float(len(calls))])
    monkeypatch.setattr(FilterCache, "transform", staticmethod(fake_transform))
    cache, lib, d = FilterCache(), _FakeLib(), _desc()
    w = torch.randn(4, 3, 3, 3)
    u1 = cache.get(lib, d, 0, 0, w, None)
    assert cache.get(lib, d, 0, 0, w, None) is u1 and len(calls) == 1        # same tensor, same version
    with torch.no_grad():
        w.add_(1.0)                                                          # optimizer-style update
    assert cache.get(lib, d, 0, 0, w, None) is not u1 and len(calls) == 2
    # a new tensor at (possibly) the same address starts at _version 0: must miss
    ptr = w.data_ptr()
    del w
    w2 = torch.empty(4, 3, 3, 3).normal_()
    n0 = len(calls)
    cache.get(lib, d, 0, 0, w2, None)
    assert len(calls) == n0 + 1, f"stale hit (same address reused: {w2.data_ptr() == ptr})"
    # non-contiguous (channels_last) weights: never cached, always re-transformed
    wc = torch.randn(4, 3, 3, 3).to(memory_format=torch.channels_last)
    assert not wc.is_contiguous()
    cache.get(lib, d, 0, 0, wc, None)
    cache.get(lib, d, 0, 0, wc, None)
    assert len(calls) == n0 + 3
    # inference tensors have no version counter: bypass, no error
    with torch.inference_mode():
        wi = torch.randn(4, 3, 3, 3)
    cache.get(lib, d, 0, 0, wi, None)
    assert len(calls) == n0 + 4
