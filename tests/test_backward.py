"""DWM backward: ``dwm_backward`` against the reference's
own ``dwm_backward`` outputs (golden fixtures made by tests/golden/make_golden.py
on the reference's backward test geometries, test_engines_backward.py:81-132)
and against the binary64 analytic oracle.

Tolerances (written here):
  * binary64: max |gpu - oracle| <= 1e-10 (the reference's own criterion,
    test_engines_backward.py:96-97) and max |gpu - reference dwm64| <= 1e-10.
  * binary32: MSE vs the binary64 oracle <= the reference's binary32 MSE
    (<= 4x for gradients with fewer than 4096 entries, where the ratio is noise)
    (plus 1e-14 absolute for the all-but-exact tiny cases) -- the B200 data
    gradient runs the forward engine on the adjoint problem and the weight
    gradient is a different (fixed) summation order, so bits differ but the
    error must stay at the reference's level.
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle.dwm_oracle import direct_conv2d_grads_f64, mse
from paper_2002_00552_b200 import ConvSpec, dwm_backward, plan_decomposition

CASES = json.loads((GOLDEN / "backward_cases.json").read_text())
ARR = np.load(GOLDEN / "backward_cases.npz")


def _spec(case):
    return ConvSpec(kernel=tuple(case["kernel"]), stride=tuple(case["stride"]), pad=tuple(case["pad"]))


def _inputs(case):
    """The seeded inputs make_golden.py used (backward_inputs); their sums are
    recorded in the fixture, so a changed generator fails loudly."""
    rng = np.random.default_rng(case["seed"])
    n, c, h, w = case["shape"]
    spec = _spec(case)
    d = rng.standard_normal((n, c, h, w))
    g = rng.standard_normal((case["f"], c, *case["kernel"]))
    oh, ow = spec.out_dims(h, w)
    dy = rng.standard_normal((n, case["f"], oh, ow))
    assert np.allclose([d.sum(), g.sum(), dy.sum()], case["input_sums"], rtol=0, atol=1e-9)
    return d, g, dy


# ---------------------------------------------------------------- CPU (oracle)

@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_grads_match_reference_golden(case):
    """Pins the oracle restatement against the reference's dwm_backward."""
    d, g, dy = _inputs(case)
    gd, gw = direct_conv2d_grads_f64(d, g, _spec(case), dy)
    k = case["name"]
    assert np.max(np.abs(gd - ARR[f"{k}/gd64"])) <= 1e-10
    assert np.max(np.abs(gw - ARR[f"{k}/gw64"])) <= 1e-10


def test_oracle_grads_match_reference_module(ref):
    """Oracle vs the reference test-suite's literal-loop oracle_grads semantics
    (reference.py:48-71) re-derived through the reference dwm_backward."""
    rng = np.random.default_rng(5)
    spec = ConvSpec(kernel=(4, 3), stride=(3, 2), pad=(2, 1, 0, 2))
    d = rng.standard_normal((2, 3, 11, 10))
    g = rng.standard_normal((2, 3, 4, 3))
    rspec = ref.ConvSpec(kernel=(4, 3), stride=(3, 2), pad=(2, 1, 0, 2))
    oh, ow = rspec.out_dims(11, 10)
    dy = rng.standard_normal((2, 2, oh, ow))
    from dwmconv.engines import dwm_backward as ref_backward
    want_d, want_w = ref_backward(dy, ref.plan_decomposition(rspec), d, g)
    got_d, got_w = direct_conv2d_grads_f64(d, g, spec, dy)
    assert np.max(np.abs(got_d - want_d)) <= 1e-10
    assert np.max(np.abs(got_w - want_w)) <= 1e-10


def test_backward_rejects_bad_grad_shape():
    """reference test_engines_backward.py:135-141 (raised before any device work)."""
    spec = ConvSpec(kernel=(3, 3))
    with pytest.raises(ValueError, match="grad_out"):
        dwm_backward(np.zeros((1, 1, 2, 2)), plan_decomposition(spec),
                     np.zeros((1, 1, 8, 8)), np.zeros((1, 1, 3, 3)))


def test_backward_rejects_bad_taps_and_channels():
    spec = ConvSpec(kernel=(3, 3))
    plan = plan_decomposition(spec)
    with pytest.raises(ValueError, match="taps"):
        dwm_backward(np.zeros((1, 1, 6, 6)), plan, np.zeros((1, 1, 8, 8)), np.zeros((1, 1, 5, 5)))
    with pytest.raises(ValueError, match="channel mismatch"):
        dwm_backward(np.zeros((1, 1, 6, 6)), plan, np.zeros((1, 2, 8, 8)), np.zeros((1, 1, 3, 3)))
    with pytest.raises(TypeError):
        dwm_backward([[0.0]], plan, np.zeros((1, 1, 8, 8)), np.zeros((1, 1, 3, 3)))


# ---------------------------------------------------------------- GPU

@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_backward_f64_matches_reference(cuda, case):
    d, g, dy = _inputs(case)
    spec = _spec(case)
    gd, gw = dwm_backward(dy, plan_decomposition(spec), d, g)
    assert gd.dtype == np.float64 and gd.shape == d.shape and gw.shape == g.shape
    k = case["name"]
    want_d, want_w = direct_conv2d_grads_f64(d, g, spec, dy)
    assert np.max(np.abs(gd - want_d)) <= 1e-10
    assert np.max(np.abs(gw - want_w)) <= 1e-10
    assert np.max(np.abs(gd - ARR[f"{k}/gd64"])) <= 1e-10
    assert np.max(np.abs(gw - ARR[f"{k}/gw64"])) <= 1e-10


def _tc_wgrad_ok(case):
    c, f = case["shape"][1], case["f"]
    return c % 32 == 0 and c >= 64 and f >= 64


def _record(key, value):
    """Achieved error ratios vs the reference, appended to $DWM_RATIO_OUT."""
    import json
    import os
    out = os.environ.get("DWM_RATIO_OUT")
    if not out:
        return
    old = json.loads(open(out).read()) if os.path.exists(out) else {}
    old[key] = value
    with open(out, "w") as fh:
        json.dump(old, fh, indent=1, sort_keys=True)


@pytest.mark.gpu
@pytest.mark.parametrize("wgrad", ["exact", "tc"])
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_backward_f32_error_at_reference_level(cuda, case, wgrad):
    if wgrad == "tc" and not _tc_wgrad_ok(case):
        pytest.skip("tcgen05 weight gradient needs C % 32 == 0, C >= 64, F >= 64")
    d, g, dy = _inputs(case)
    spec = _spec(case)
    gd, gw = dwm_backward(dy, plan_decomposition(spec), d, g, precision=np.float32, wgrad_algo=wgrad)
    assert gd.dtype == np.float32 and gw.dtype == np.float32
    k = case["name"]
    want_d, want_w = ARR[f"{k}/gd64"], ARR[f"{k}/gw64"]
    rd, rw = mse(gd, want_d) / max(case["ref_mse_gd32"], 1e-300), mse(gw, want_w) / max(case["ref_mse_gw32"], 1e-300)
    _record(f"backward_f32/{k}/{wgrad}", {"data": rd, "weights": rw, "outputs": [int(gd.size), int(gw.size)]})
    # at or below the reference's binary32 error; with fewer than 4096 outputs
    # the MSE ratio is sampling noise (0.2-2.7x observed), 4x slack there
    slack_d = 1.0 if gd.size >= 4096 else 4.0
    slack_w = 1.0 if gw.size >= 4096 else 4.0
    assert mse(gd, want_d) <= slack_d * case["ref_mse_gd32"] + 1e-14, rd
    assert mse(gw, want_w) <= slack_w * case["ref_mse_gw32"] + 1e-14, rw


@pytest.mark.gpu
def test_backward_zero_grad_out(cuda):
    """reference test_engines_backward.py:12-27"""
    spec = ConvSpec(kernel=(5, 5), stride=(2, 2))
    d = np.ones((1, 1, 9, 9))
    w = np.ones((1, 1, 5, 5))
    oh, ow = spec.out_dims(9, 9)
    gd, gw = dwm_backward(np.zeros((1, 1, oh, ow)), plan_decomposition(spec), d, w)
    np.testing.assert_array_equal(gd, np.zeros_like(d))
    np.testing.assert_array_equal(gw, np.zeros_like(w))


@pytest.mark.gpu
def test_backward_ones_counts_windows(cuda):
    """reference test_engines_backward.py:44-50 through dwm_backward: every
    3x3 tap of a 4x4 all-ones input is covered by all four outputs."""
    spec = ConvSpec(kernel=(3, 3))
    gd, gw = dwm_backward(np.ones((1, 1, 2, 2)), plan_decomposition(spec),
                          np.ones((1, 1, 4, 4)), np.ones((1, 1, 3, 3)))
    np.testing.assert_array_equal(gw, np.full((1, 1, 3, 3), 4.0))


@pytest.mark.gpu
def test_backward_torch_io_and_determinism(cuda):
    import torch
    case = next(c for c in CASES if c["name"] == "bw_extra6")
    d, g, dy = _inputs(case)
    plan = plan_decomposition(_spec(case))
    t = [torch.from_numpy(a).float().to(cuda) for a in (dy, d, g)]
    gd1, gw1 = dwm_backward(t[0], plan, t[1], t[2])
    gd2, gw2 = dwm_backward(t[0], plan, t[1], t[2])
    assert gd1.is_cuda and gd1.dtype == torch.float32
    assert torch.equal(gd1, gd2) and torch.equal(gw1, gw2)
    gd_np, gw_np = dwm_backward(dy.astype(np.float32), plan, d.astype(np.float32), g.astype(np.float32))
    assert np.array_equal(gd1.cpu().numpy(), gd_np) and np.array_equal(gw1.cpu().numpy(), gw_np)


@pytest.mark.gpu
def test_backward_nonfinite_raises(cuda):
    spec = ConvSpec(kernel=(3, 3))
    d = np.ones((1, 1, 6, 6))
    d[0, 0, 2, 2] = np.inf
    with pytest.raises(FloatingPointError, match="dwm_backward"):
        dwm_backward(np.ones((1, 1, 4, 4)), plan_decomposition(spec), d, np.ones((1, 1, 3, 3)))


@pytest.mark.gpu
def test_backward_need_flags(cuda):
    case = next(c for c in CASES if c["name"] == "bw_r7_s2")
    d, g, dy = _inputs(case)
    plan = plan_decomposition(_spec(case))
    gd_all, gw_all = dwm_backward(dy, plan, d, g)
    gd, gw = dwm_backward(dy, plan, d, g, need_weights=False)
    assert gw is None and np.array_equal(gd, gd_all)
    gd, gw = dwm_backward(dy, plan, d, g, need_data=False)
    assert gd is None and np.array_equal(gw, gw_all)


@pytest.mark.gpu
def test_backward_batch_invariance(cuda):
    """Per-image data gradients do not depend on the batch they are in."""
    case = next(c for c in CASES if c["name"] == "bw_extra6")
    d, g, dy = _inputs(case)
    plan = plan_decomposition(_spec(case))
    gd, _ = dwm_backward(dy, plan, d, g, need_weights=False)
    for i in range(d.shape[0]):
        gdi, _ = dwm_backward(dy[i:i + 1], plan, d[i:i + 1], g, need_weights=False)
        assert np.array_equal(gd[i:i + 1], gdi)


@pytest.mark.gpu
def test_tc_weight_grad_tail_and_determinism(cuda):
    """tcgen05 weight gradient: odd tile counts (TMA zero fill of the K tail),
    C and F not multiples of the 128 x 64 block, run-to-run identical."""
    import torch
    from oracle.dwm_oracle import direct_conv2d_grads_f64
    rng = np.random.default_rng(77)
    spec = ConvSpec(kernel=(5, 5), stride=(1, 1), pad=(2, 2, 2, 2))
    d = rng.standard_normal((3, 96, 11, 13))
    g = rng.standard_normal((80, 96, 5, 5))
    dy = rng.standard_normal((3, 80, 11, 13))
    plan = plan_decomposition(spec)
    t = [torch.from_numpy(a).float().to(cuda) for a in (dy, d, g)]
    _, gw1 = dwm_backward(t[0], plan, t[1], t[2], need_data=False, wgrad_algo="tc")
    _, gw2 = dwm_backward(t[0], plan, t[1], t[2], need_data=False, wgrad_algo="tc")
    assert torch.equal(gw1, gw2)
    _, want = direct_conv2d_grads_f64(d.astype(np.float32), g.astype(np.float32), spec, dy.astype(np.float32))
    _, gw_exact = dwm_backward(t[0], plan, t[1], t[2], need_data=False, wgrad_algo="exact")
    e_tc = mse(gw1.cpu().numpy(), want)
    e_ex = mse(gw_exact.cpu().numpy(), want)
    assert e_tc <= 4 * e_ex + 1e-12, (e_tc, e_ex)


def _random_backward_geometries(count, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        k = tuple(int(v) for v in rng.integers(1, 10, size=2))
        st = tuple(int(v) for v in rng.integers(1, 4, size=2))
        pad = tuple(int(v) for v in rng.integers(0, 4, size=4))
        h, w = (int(v) for v in rng.integers(6, 24, size=2))
        try:
            ConvSpec(kernel=k, stride=st, pad=pad).out_dims(h, w)
        except ValueError:
            continue
        out.append((k, st, pad, h, w))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("geom", _random_backward_geometries(24, 7),
                         ids=lambda g: f"k{g[0]}s{g[1]}p{g[2]}_{g[3]}x{g[4]}")
def test_backward_random_geometries(cuda, geom):
    """Random kernels/strides/pads/extents: binary64 gradients <= 1e-10 from
    the FP64 oracle (polyphase data gradient + CUDA-core weight gradient);
    binary32 with the tcgen05 weight gradient close to the oracle."""
    k, st, pad, h, w = geom
    spec = ConvSpec(kernel=k, stride=st, pad=pad)
    plan = plan_decomposition(spec)
    rng = np.random.default_rng(h * 100 + w)
    oh, ow = spec.out_dims(h, w)
    d = rng.standard_normal((2, 3, h, w))
    g = rng.standard_normal((5, 3, *k))
    dy = rng.standard_normal((2, 5, oh, ow))
    gd, gw = dwm_backward(dy, plan, d, g)
    want_d, want_w = direct_conv2d_grads_f64(d, g, spec, dy)
    assert np.max(np.abs(gd - want_d)) <= 1e-10
    assert np.max(np.abs(gw - want_w)) <= 1e-10
    d = rng.standard_normal((2, 64, h, w)).astype(np.float32)
    g = rng.standard_normal((64, 64, *k)).astype(np.float32)
    dy = rng.standard_normal((2, 64, oh, ow)).astype(np.float32)
    gd, gw = dwm_backward(dy, plan, d, g, wgrad_algo="tc")
    want_d, want_w = direct_conv2d_grads_f64(d, g, spec, dy)
    assert np.max(np.abs(gd - want_d)) <= 2e-4 * max(1.0, np.abs(want_d).max())
    assert np.max(np.abs(gw - want_w)) <= 2e-4 * max(1.0, np.abs(want_w).max())
