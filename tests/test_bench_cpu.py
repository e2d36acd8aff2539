"""bench.py host logic on CPU: the self-launch under torchrun for --gpus N
(gloo, world_size 2, kernel call stubbed), strong-scaling shards, the binary64
ground truth used for the bench's MSE line, and the reference arm."""

import json
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def _run(args, timeout=300):
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


def test_bench_self_launches_two_ranks_strong_scaling():
    """--gpus 2 re-launches under torch.distributed.run; cfg4 shards its batch
    of 512 into 2 x 256 and rank 0 prints one line for the job."""
    line = _run(["--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "3"])
    assert line["n_gpus"] == 2
    assert line["scaling"] == "strong"
    assert line["config"]["global_batch"] == 512
    assert line["config"]["batch_per_gpu"] == 256
    assert line["shard"] == [0, 256]
    assert line["calls"] == 5            # 3 warm-up + 2 timed steps per rank


def test_bench_weak_scaling_default_for_stem():
    line = _run(["--gpus", "2", "--dry-run", "--steps", "1", "--workload", "cfg2-resnet50-stem"])
    assert line["scaling"] == "weak"
    assert line["config"]["global_batch"] == 512 and line["config"]["batch_per_gpu"] == 256


@pytest.mark.parametrize("name", ["cfg1-5x5s1", "cfg3-alexnet-conv1", "cfg5-5x5s2"])
def test_bench_direct_f64_matches_oracle(name):
    sys.path.insert(0, str(ROOT))
    import bench
    from oracle.dwm_oracle import direct_conv2d_f64
    from paper_2002_00552_b200.configs import WORKLOADS
    wl = WORKLOADS[name]
    rng = np.random.default_rng(0)
    c = min(wl.c_in, 16)
    x = rng.standard_normal((c, wl.hw, wl.hw))
    w = rng.standard_normal((8, c, wl.kernel, wl.kernel))
    got = bench.direct_f64(x, w, wl.spec())
    want = direct_conv2d_f64(x[None], w, wl.spec())[0]
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-11)


def test_bench_draw_is_reference_recipe():
    sys.path.insert(0, str(ROOT))
    import bench
    from oracle.dwm_oracle import draw
    a = bench.draw(1, (5, 5), (1, 1), 56, 32, 32, 1)
    b = draw(1, (5, 5), (1, 1), 56, 32, 32, 1)
    assert all(np.array_equal(p, q) for p, q in zip(a, b))


def test_bench_reference_arm_line():
    line = _run(["--impl", "reference", "--workload", "cfg1-5x5s1", "--steps", "2", "--warmup", "1"])
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["unit"] == "images/s"
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["e2e"]["h2d_bytes_per_step"] == 0
