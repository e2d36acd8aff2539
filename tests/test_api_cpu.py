"""Host-side behaviour of the drop-in entry point that runs before any device
work: argument validation with the reference's exception types/messages, and
the no-CPU-fallback rule (engines.py:63-68,230-236; tensor.py:16-24)."""

import numpy as np
import pytest

from paper_2002_00552_b200 import ConvSpec, dwm_conv2d, plan_decomposition, convolve


def test_rejects_channel_mismatch():             # test_engines_forward.py:209-213
    with pytest.raises(ValueError, match="channel"):
        dwm_conv2d(np.zeros((1, 2, 8, 8)), np.zeros((1, 3, 3, 3)), ConvSpec(kernel=(3, 3)))


def test_rejects_non_arrays_and_bad_rank():
    with pytest.raises(TypeError, match="numpy array"):
        dwm_conv2d([[1.0]], np.zeros((1, 1, 3, 3)), ConvSpec(kernel=(3, 3)))
    with pytest.raises(ValueError, match="4 axes"):
        dwm_conv2d(np.zeros((2, 8, 8)), np.zeros((1, 2, 3, 3)), ConvSpec(kernel=(3, 3)))
    with pytest.raises(TypeError, match="float32 or float64"):
        dwm_conv2d(np.zeros((1, 1, 8, 8), np.int32), np.zeros((1, 1, 3, 3)), ConvSpec(kernel=(3, 3)))
    with pytest.raises(TypeError, match="binary32/binary64"):
        dwm_conv2d(np.zeros((1, 1, 8, 8), object), np.zeros((1, 1, 3, 3)), ConvSpec(kernel=(3, 3)))


def test_rejects_tap_mismatch_and_foreign_plan():
    d, g = np.zeros((1, 1, 8, 8)), np.zeros((1, 1, 3, 3))
    with pytest.raises(ValueError, match="do not match kernel"):
        dwm_conv2d(d, g, ConvSpec(kernel=(5, 5)))
    with pytest.raises(ValueError, match="different ConvSpec"):
        dwm_conv2d(d, g, ConvSpec(kernel=(3, 3)), plan=plan_decomposition(ConvSpec(kernel=(3, 3), stride=(2, 2))))
    with pytest.raises(ValueError, match="unknown precision"):
        dwm_conv2d(d, g, ConvSpec(kernel=(3, 3)), precision="binary16")
    with pytest.raises(ValueError, match="too small"):
        dwm_conv2d(np.zeros((1, 1, 2, 2)), g, ConvSpec(kernel=(3, 3)))


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        dwm_conv2d(np.zeros((1, 1, 8, 8)), np.zeros((1, 1, 3, 3)), ConvSpec(kernel=(3, 3)))
    with pytest.raises(ValueError, match="only 'dwm'"):
        convolve(np.zeros((1, 1, 8, 8)), np.zeros((1, 1, 3, 3)), ConvSpec(kernel=(3, 3)), algo="direct")


@pytest.mark.parametrize("n,c,f", [(0, 3, 4), (2, 3, 0), (2, 0, 4), (0, 0, 0)])
def test_empty_tensors_like_reference(n, c, f):
    """Empty batch / filters give empty outputs and no input channels gives
    zeros, as the reference's NumPy path does; the counter still counts.
    (Shape-only: no device work happens, so this runs on CPU.)"""
    import numpy as np
    from paper_2002_00552_b200 import ConvSpec, FlopCounter, dwm_backward, dwm_conv2d, flops_dwm, plan_decomposition
    spec = ConvSpec(kernel=(3, 3), stride=(2, 1), pad=(1, 0, 1, 1))
    d = np.zeros((n, c, 8, 9), np.float32)
    g = np.ones((f, c, 3, 3), np.float32)
    counter = FlopCounter()
    y = dwm_conv2d(d, g, spec, counter=counter)
    oh, ow = spec.out_dims(8, 9)
    assert y.shape == (n, f, oh, ow) and y.dtype == np.float32 and not y.any()
    assert counter.elementwise == flops_dwm(plan_decomposition(spec), (oh, ow))
    gd, gw = dwm_backward(np.ones((n, f, oh, ow), np.float32), plan_decomposition(spec), d, g)
    assert gd.shape == d.shape and gw.shape == g.shape and not gd.any() and not gw.any()


def test_empty_tensors_match_live_reference(ref):
    import numpy as np
    from paper_2002_00552_b200 import ConvSpec, dwm_conv2d
    d = np.zeros((2, 0, 8, 8), np.float32)
    g = np.ones((4, 0, 3, 3), np.float32)
    want = ref.dwm_conv2d(d, g, ref.ConvSpec(kernel=(3, 3)))
    got = dwm_conv2d(d, g, ConvSpec(kernel=(3, 3)))
    assert got.shape == want.shape and got.dtype == want.dtype and np.array_equal(got, want)


@pytest.mark.parametrize("kernel,stride,pad", [((7, 7), (2, 2), (3, 3, 3, 3)), ((11, 5), (4, 1), (0, 1, 2, 0)),
                                               ((3, 3), (1, 1), (1, 1, 1, 1))])
def test_reference_spec_and_plan_objects_reach_native_planner(ref, monkeypatch, kernel, stride, pad):
    """Drop-in with the reference's own objects (engines.py:233-236,417-418):
    its ConvSpec and DecompositionPlan (fields spec/parts only) pass the plan
    check and reach dwm_desc_init; the first thing that fails on this CPU-only
    host is the device check, after all host-side planning."""
    import torch
    from paper_2002_00552_b200 import engines, flops_dwm
    seen = {}
    real = engines._check_plan_matches

    def spy(plan, desc):
        real(plan, desc)
        seen["rows"], seen["cols"] = desc.axis("row"), desc.axis("col")
    monkeypatch.setattr(engines, "_check_plan_matches", spy)
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    rspec = ref.ConvSpec(kernel=kernel, stride=stride, pad=pad)
    rplan = ref.plan_decomposition(rspec)
    d = np.zeros((1, 2, 23, 19), np.float32)
    g = np.zeros((3, 2, *kernel), np.float32)
    for sp, pl in ((rspec, rplan), (rspec, None), (ConvSpec(kernel=kernel, stride=stride, pad=pad), rplan)):
        seen.clear()
        engines._cached_desc_key.cache_clear()
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            dwm_conv2d(d, g, sp, plan=pl)
        if pl is None:
            continue  # own plan: checked against the native planner once per geometry (cached)
        want_rows = []
        for p in rplan.parts:
            r = (p.row.origin, p.row.step, p.row.count)
            if r not in want_rows:
                want_rows.append(r)
        assert seen["rows"] == want_rows
    # the reference's FlopCounter and plan work with the counting helpers
    oh, ow = rspec.out_dims(23, 19)
    assert flops_dwm(rplan, (oh, ow)) == ref.flops_dwm(rplan, (oh, ow))


def test_reference_plan_for_other_spec_is_rejected(ref):
    rspec = ref.ConvSpec(kernel=(5, 5), stride=(1, 1), pad=(2, 2, 2, 2))
    other = ref.plan_decomposition(ref.ConvSpec(kernel=(5, 5), stride=(2, 2), pad=(2, 2, 2, 2)))
    with pytest.raises(ValueError, match="different ConvSpec"):
        dwm_conv2d(np.zeros((1, 1, 8, 8)), np.zeros((1, 1, 5, 5)), rspec, plan=other)
