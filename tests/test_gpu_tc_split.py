"""GPU tests of the tcgen05 engine's fp16 split (csrc/dwm_gemm_tc.cu).

The engine computes each FP32 contraction from three fp16 products of
power-of-two scaled operands (V per image by 2^(12 - floor(log2 max|x_n|)),
U per filter by 2^(12 - floor(log2 max|w_f|))).  Properties checked here, on top of
the MSE-vs-reference bars every tc workload already passes (test_gpu_parity,
test_gpu_acceptance):
  * the C-ABI stage pair (dwm_input_transform_ranged + dwm_gemm_output_tc)
    and dwm_gemm_output (range taken from V itself) give the forward's bits;
  * power-of-two scale invariance, bit for bit: y(2^a x, 2^b w) == 2^(a+b) y(x, w)
    far outside the fp16 range (the scales absorb it);
  * per-image scales: each image's bits are those of the image run alone,
    also when the batch mixes images of very different magnitudes;
  * one channel 2^20 larger than the rest (the shared V scale then puts the
    others' low parts near the fp16 subnormal range): MSE vs FP64 still at or
    below the reference DWM32's on the same data.
"""

import numpy as np
import pytest
import torch

from oracle.dwm_oracle import direct_conv2d_f64, dwm_conv2d_oracle, mse
from paper_2002_00552_b200 import ConvSpec, _native

pytestmark = pytest.mark.gpu

GEOMS = [  # (n, c, hw, f, r, stride, pad)
    (2, 128, 14, 96, 5, 1, 2),
    (3, 64, 11, 64, 3, 1, 1),
    (2, 96, 16, 130, 7, 2, 3),
]


def _forward(lib, x, w, spec, desc):
    ws_bytes = lib.dwm_workspace_bytes(desc, _native.DWM_F32, _native.DWM_ALGO_TC)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=x.device)
    y = torch.empty(x.shape[0], w.shape[0], desc.oh, desc.ow, device=x.device)
    flag = torch.zeros(1, dtype=torch.int32, device=x.device)
    s = torch.cuda.current_stream().cuda_stream
    _native.check(lib.dwm_conv2d_forward(desc, _native.DWM_F32, _native.DWM_ALGO_TC, x.data_ptr(), w.data_ptr(),
                                         y.data_ptr(), ws.data_ptr(), ws_bytes, flag.data_ptr(), s))
    torch.cuda.synchronize()
    assert int(flag.item()) == 0
    return y


def _setup(geom, seed=0):
    n, c, hw, f, r, st, p = geom
    spec = ConvSpec(kernel=(r, r), stride=(st, st), pad=(p, p, p, p))
    desc = _native.make_desc(n, c, hw, hw, f, spec.kernel, spec.stride, spec.pad)
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(n, c, hw, hw, generator=g).cuda()
    w = torch.randn(f, c, r, r, generator=g).cuda()
    return spec, desc, x, w


@pytest.mark.parametrize("geom", GEOMS)
def test_stage_pair_and_self_ranged_gemm_match_forward(cuda, geom):
    lib = _native.load()
    spec, desc, x, w = _setup(geom)
    y = _forward(lib, x, w, spec, desc)
    s = torch.cuda.current_stream().cuda_stream
    u = torch.empty(lib.dwm_filter_bytes(desc, _native.DWM_F32, _native.DWM_ALGO_TC), dtype=torch.uint8,
                    device="cuda")
    _native.check(lib.dwm_prepare_filter(desc, _native.DWM_F32, _native.DWM_ALGO_TC, w.data_ptr(), u.data_ptr(), s))
    v = torch.empty(desc.num_freqs * desc.tiles * desc.c, device="cuda")
    rng = torch.zeros(lib.dwm_range_bytes(desc) // 4, dtype=torch.int32, device="cuda")
    _native.check(lib.dwm_input_transform_ranged(desc, x.data_ptr(), v.data_ptr(), rng.data_ptr(), s))
    y2 = torch.full_like(y, float("nan"))
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _native.check(lib.dwm_gemm_output_tc(desc, v.data_ptr(), u.data_ptr(), rng.data_ptr(), y2.data_ptr(),
                                         flag.data_ptr(), s))
    # the stage API without a range: bound from max|V| (a different power of two, same bits)
    y3 = torch.full_like(y, float("nan"))
    rb = lib.dwm_range_bytes(desc)
    scratch = torch.empty(rb, dtype=torch.uint8, device="cuda")
    _native.check(lib.dwm_gemm_output(desc, _native.DWM_F32, _native.DWM_ALGO_TC, v.data_ptr(), u.data_ptr(),
                                      y3.data_ptr(), flag.data_ptr(), scratch.data_ptr(), rb, s))
    torch.cuda.synchronize()
    assert torch.equal(y, y2)
    assert torch.equal(y, y3)
    # no workspace -> a loud error, not a guess
    with pytest.raises(ValueError, match="workspace"):
        _native.check(lib.dwm_gemm_output(desc, _native.DWM_F32, _native.DWM_ALGO_TC, v.data_ptr(), u.data_ptr(),
                                          y3.data_ptr(), flag.data_ptr(), None, 0, s))


@pytest.mark.parametrize("a,b", [(-70, 0), (0, -60), (50, 20), (-100, 30), (24, -24)])
def test_power_of_two_scale_invariance(cuda, a, b):
    lib = _native.load()
    spec, desc, x, w = _setup(GEOMS[0], seed=1)
    y = _forward(lib, x, w, spec, desc)
    ys = _forward(lib, x * 2.0 ** a, w * 2.0 ** b, spec, desc)
    assert torch.equal(ys, y * 2.0 ** (a + b))


def test_outlier_channel_accuracy(cuda):
    lib = _native.load()
    spec, desc, x, w = _setup((2, 128, 14, 64, 5, 1, 2), seed=2)
    x[:, 7] *= 2.0 ** 20
    y = _forward(lib, x, w, spec, desc).cpu().numpy()
    xn, wn = x.cpu().numpy(), w.cpu().numpy()
    truth = direct_conv2d_f64(xn.astype(np.float64), wn.astype(np.float64), spec)
    ref32 = dwm_conv2d_oracle(xn, wn, spec, np.float32)
    ours, theirs = mse(y, truth), mse(ref32, truth)
    assert ours <= theirs, (ours, theirs)


def test_per_image_scale_independent_of_batch(cuda):
    """Images of very different magnitudes in one batch: every image's output
    is bit-identical to the image convolved alone (the V scale is per image)."""
    lib = _native.load()
    spec, desc, x, w = _setup((4, 128, 14, 64, 5, 1, 2), seed=3)
    x[1] *= 2.0 ** 30
    x[2] *= 2.0 ** -40
    y = _forward(lib, x, w, spec, desc)
    for i in range(4):
        d1 = _native.make_desc(1, 128, 14, 14, 64, spec.kernel, spec.stride, spec.pad)
        yi = _forward(lib, x[i:i + 1].contiguous(), w, spec, d1)
        assert torch.equal(yi[0], y[i]), i


def test_host_chunked_forward_matches_device_forward(cuda):
    """Host tensors go through the chunked three-stream path (chunk sizes
    picked to fill whole GEMM waves); with per-image scales every output bit
    equals the single device call on the whole batch."""
    from paper_2002_00552_b200 import dwm_conv2d, engines
    spec = ConvSpec(kernel=(5, 5), stride=(1, 1), pad=(2, 2, 2, 2))
    g = torch.Generator().manual_seed(4)
    x = torch.randn(40, 128, 14, 14, generator=g)
    x[3] *= 2.0 ** 12
    w = torch.randn(128, 128, 5, 5, generator=g)
    lib = _native.load()
    desc = _native.make_desc(40, 128, 14, 14, 128, spec.kernel, spec.stride, spec.pad)
    bounds = engines._host_chunks(lib, desc, _native.DWM_F32, _native.DWM_ALGO_AUTO, 40, torch.device("cuda"))
    assert len(bounds) > 2  # really chunked
    y_dev = dwm_conv2d(x.cuda(), w.cuda(), spec).cpu()
    y_host = dwm_conv2d(x.pin_memory(), w.cuda(), spec)
    assert y_host.device.type == "cpu"
    assert torch.equal(y_host, y_dev)
