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
