"""Generate the golden fixtures in this directory FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``dwmconv`` from /root/reference/pkg/src (read-only, never copied)
and writes:
  plans.json          plan_to_json for r_h, r_w in 1..11, s in 1..4, plus
                      rectangular/anisotropic-stride cases
  transforms.json     exact F(2,1..3) triples (get_transform)
  small_cases.npz     inputs + reference outputs (dwm binary32, dwm binary64,
                      direct binary64) on the reference's own test geometries
  cases.json          metadata for small_cases.npz
  baseline_samples.json  per BASELINE workload (one image, seed 1, the bench.py
                      _draw recipe): reference DWM32 / direct32 MSE vs direct64
                      and 512 sampled output values of DWM32 and direct64
  backward_cases.npz  inputs + reference dwm_backward (binary64 and binary32)
  backward_cases.json on the reference's backward test geometries plus
                      asymmetric/rectangular/channel-heavy extras
                      (``make_golden.py backward`` regenerates only these)
  accuracy_14x14.json the reference's binary32 acceptance sweep (C=F=256,
                      14x14, r=3..11, seeds 1-3): DWM32 / direct32 MSE
                      (``make_golden.py acceptance`` regenerates only this)
The GPU box has no /root/reference; the tests there read these files.
"""

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from dwmconv.convspec import ConvSpec  # noqa: E402
from dwmconv.decompose import plan_decomposition, plan_to_json  # noqa: E402
from dwmconv.engines import direct_conv2d, dwm_backward, dwm_conv2d  # noqa: E402
from dwmconv.tensor import mse  # noqa: E402
from dwmconv.transforms import get_transform, transform_to_json  # noqa: E402

sys.path.insert(0, str(HERE.parent.parent))
from paper_2002_00552_b200.configs import WORKLOADS  # noqa: E402


def plans():
    out = []
    for r_h in range(1, 12):
        for r_w in range(1, 12):
            for s in range(1, 5):
                out.append(plan_to_json(plan_decomposition(ConvSpec(kernel=(r_h, r_w), stride=(s, s)))))
    for k, s in [((4, 6), (2, 1)), ((7, 3), (1, 3)), ((11, 5), (4, 2)), ((2, 9), (3, 1))]:
        out.append(plan_to_json(plan_decomposition(ConvSpec(kernel=k, stride=s))))
    (HERE / "plans.json").write_text(json.dumps(out))


def transforms():
    (HERE / "transforms.json").write_text(json.dumps([transform_to_json(get_transform(r)) for r in (1, 2, 3)]))


def small_case_specs():
    cases = []
    # test_engines_forward.py:138-150 full grid r=1..11 x s=1..3, pad 1
    for r in range(1, 12):
        for s in range(1, 4):
            cases.append(dict(name=f"grid_r{r}_s{s}", seed=31 * r + s, kernel=(r, r), stride=(s, s),
                              pad=(1, 1, 1, 1), shape=(1, 2, r + 2 * s + 3, r + 2 * s + 3), f=1))
    # test_engines_forward.py:153-164 and test_acceptance.py:65-78 (incl. s=4)
    for r, s in [(1, 1), (3, 1), (5, 1), (7, 2), (9, 2), (11, 4)]:
        h = max(16, r + s)
        cases.append(dict(name=f"param_r{r}_s{s}", seed=100 + r + s, kernel=(r, r), stride=(s, s),
                          pad=(r // 3,) * 4, shape=(2, 3, h, h), f=2))
    for r in (1, 3, 5, 7, 9, 11):
        for s in (1, 2, 4):
            hw = {1: 14, 2: 18, 4: 21}[s] if r < 9 else {1: 18, 2: 22, 4: 27}[s]
            cases.append(dict(name=f"accept_r{r}_s{s}", seed=1000 + 10 * r + s, kernel=(r, r), stride=(s, s),
                              pad=(r // 2,) * 4, shape=(2, 3, hw, hw), f=4))
    # odd extents, asymmetric pads, rectangular kernels, anisotropic strides
    extra = [((5, 5), (2, 2), (0, 0, 0, 0), (1, 2, 7, 7), 2),
             ((3, 3), (1, 1), (0, 0, 0, 0), (1, 2, 7, 9), 2),
             ((4, 6), (2, 1), (1, 2, 0, 3), (2, 3, 13, 11), 3),
             ((7, 3), (1, 3), (3, 3, 1, 1), (1, 4, 12, 17), 5),
             ((11, 5), (4, 2), (2, 0, 2, 1), (1, 2, 30, 19), 3),
             ((2, 2), (1, 1), (0, 1, 0, 1), (1, 1, 5, 6), 1),
             ((1, 1), (3, 2), (0, 0, 0, 0), (1, 3, 9, 8), 2)]
    for i, (k, s, p, shp, f) in enumerate(extra):
        cases.append(dict(name=f"extra{i}", seed=500 + i, kernel=k, stride=s, pad=p, shape=shp, f=f))
    # channel counts the B200 kernels treat differently (small-C / tensor-core)
    for i, (k, s, c, f, hw) in enumerate([(7, 2, 3, 64, 20), (11, 4, 3, 96, 31), (5, 1, 32, 32, 12),
                                          (3, 1, 64, 64, 10), (3, 1, 256, 16, 8), (5, 2, 128, 64, 12)]):
        cases.append(dict(name=f"chan{i}_c{c}_f{f}", seed=700 + i, kernel=(k, k), stride=(s, s),
                          pad=(k // 2,) * 4, shape=(1, c, hw, hw), f=f))
    return cases


def small_cases():
    arrays = {}
    meta = []
    for case in small_case_specs():
        rng = np.random.default_rng(case["seed"])
        n, c, h, w = case["shape"]
        d = rng.standard_normal((n, c, h, w))
        g = rng.standard_normal((case["f"], c, *case["kernel"]))
        spec = ConvSpec(kernel=case["kernel"], stride=case["stride"], pad=case["pad"])
        key = case["name"]
        arrays[f"{key}/data"] = d
        arrays[f"{key}/weights"] = g
        arrays[f"{key}/dwm32"] = dwm_conv2d(d, g, spec, precision=np.float32)
        arrays[f"{key}/dwm64"] = dwm_conv2d(d, g, spec, precision=np.float64)
        arrays[f"{key}/direct64"] = direct_conv2d(d, g, spec, precision=np.float64)
        meta.append({k: (list(v) if isinstance(v, tuple) else v) for k, v in case.items()})
    np.savez_compressed(HERE / "small_cases.npz", **arrays)
    (HERE / "cases.json").write_text(json.dumps(meta, indent=1))


def draw(seed, kernel, stride, hw, channels, filters, batch):
    """reference bench.py:103-109"""
    entropy = [seed, *kernel, *stride, hw, channels, filters, batch]
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy)))
    return rng.standard_normal((batch, channels, hw, hw)), rng.standard_normal((filters, channels, *kernel))


def baseline_samples():
    out = {}
    for name, wl in WORKLOADS.items():
        t0 = time.time()
        spec = ConvSpec(kernel=(wl.kernel,) * 2, stride=(wl.stride,) * 2, pad=(wl.pad,) * 4)
        d, g = draw(1, (wl.kernel,) * 2, (wl.stride,) * 2, wl.hw, wl.c_in, wl.c_out, 1)
        y64 = direct_conv2d(d, g, spec, precision=np.float64)
        y32 = dwm_conv2d(d, g, spec, precision=np.float32)
        d32 = direct_conv2d(d, g, spec, precision=np.float32)
        rng = np.random.default_rng(12345)
        idx = [tuple(int(rng.integers(0, s)) for s in y64.shape) for _ in range(512)]
        out[name] = {
            "seed": 1, "batch": 1,
            "dwm32_mse": mse(y32, y64), "direct32_mse": mse(d32, y64),
            "index": idx,
            "dwm32": [float(y32[i]) for i in idx],
            "direct64": [float(y64[i]) for i in idx],
            "dwm32_sum": float(y32.astype(np.float64).sum()),
            "direct64_sum": float(y64.sum()),
        }
        print(f"{name}: dwm32 {out[name]['dwm32_mse']:.3e} direct32 {out[name]['direct32_mse']:.3e} "
              f"({time.time() - t0:.1f}s)", flush=True)
    (HERE / "baseline_samples.json").write_text(json.dumps(out))


def acceptance_14x14():
    """The reference's own binary32 acceptance sweep (data/accuracy_14x14.json:
    C=F=256, 14x14, r=3..11 stride 1, seeds 1-3; test_acceptance.py:137-168),
    run through the reference's accuracy harness (bench.run_accuracy_suite):
    DWM32 and direct32 MSE vs the binary64 direct conv per (r, seed)."""
    from dwmconv.bench import AccuracyConfig, run_accuracy_suite
    spec = json.loads(Path("/root/reference/pkg/src/dwmconv/data/accuracy_14x14.json").read_text())
    rows = []
    for c in spec["configs"]:
        cfg = AccuracyConfig(kernel=(c["kernel"],) * 2, stride=(c["stride"],) * 2, hw=c["hw"],
                             channels=c["channels"], filters=c["filters"], batch=c["batch"],
                             precisions=("binary32",))
        rep = run_accuracy_suite([cfg], seeds=spec["seeds"])
        for r in rep.rows:
            if r.precision == "binary32" and r.algorithm in ("dwm", "direct"):
                rows.append({"kernel": c["kernel"], "stride": c["stride"], "hw": c["hw"],
                             "channels": c["channels"], "filters": c["filters"], "batch": c["batch"],
                             "seed": r.seed, "algorithm": r.algorithm, "mse": r.mse})
        print(f"r={c['kernel']}: " + ", ".join(f"{x['algorithm']} s{x['seed']} {x['mse']:.3e}"
                                             for x in rows if x["kernel"] == c["kernel"]), flush=True)
    (HERE / "accuracy_14x14.json").write_text(json.dumps({"seeds": spec["seeds"], "rows": rows}, indent=1))


def backward_case_specs():
    cases = []
    # test_engines_backward.py:81-98 (+ the finite-difference and degenerate cases)
    for k, s, p in [((3, 3), (1, 1), (1, 1, 1, 1)), ((5, 5), (1, 1), (2, 2, 2, 2)),
                    ((5, 5), (2, 2), (1, 1, 1, 1)), ((7, 7), (2, 2), (3, 3, 3, 3))]:
        cases.append(dict(name=f"bw_r{k[0]}_s{s[0]}", seed=sum(k) + sum(s), kernel=k, stride=s, pad=p,
                          shape=(2, 2, 12, 12), f=2))
    cases.append(dict(name="bw_fd", seed=23, kernel=(5, 5), stride=(2, 2), pad=(1, 1, 1, 1),
                      shape=(1, 2, 9, 9), f=2))
    cases.append(dict(name="bw_degenerate", seed=21, kernel=(3, 3), stride=(1, 1), pad=(0, 0, 0, 0),
                      shape=(1, 2, 8, 8), f=2))
    extra = [((11, 11), (4, 4), (2, 2, 2, 2), (1, 3, 31, 31), 4),
             ((4, 6), (2, 1), (1, 2, 0, 3), (2, 3, 13, 11), 3),
             ((7, 3), (1, 3), (3, 3, 1, 1), (1, 4, 12, 17), 5),
             ((5, 5), (2, 2), (0, 0, 0, 0), (1, 2, 8, 8), 2),      # unused trailing row/col
             ((3, 3), (1, 1), (4, 0, 0, 3), (1, 2, 7, 6), 2),      # pad > r-1 (adjoint crops)
             ((1, 1), (3, 2), (0, 0, 0, 0), (1, 3, 9, 8), 2),
             ((7, 7), (2, 2), (3, 3, 3, 3), (2, 3, 20, 20), 64),   # ResNet stem shape, small
             ((3, 3), (1, 1), (1, 1, 1, 1), (1, 64, 10, 10), 64),  # tensor-core adjoint
             ((5, 5), (1, 1), (2, 2, 2, 2), (1, 32, 9, 9), 128),
             ((5, 5), (2, 2), (2, 2, 2, 2), (2, 64, 15, 15), 64),   # tcgen05 weight gradient
             ((7, 7), (1, 1), (3, 3, 3, 3), (1, 64, 12, 12), 64)]
    for i, (k, s, p, shp, f) in enumerate(extra):
        cases.append(dict(name=f"bw_extra{i}", seed=900 + i, kernel=k, stride=s, pad=p, shape=shp, f=f))
    return cases


def backward_inputs(case):
    """Seeded inputs of a backward case (tests regenerate them the same way)."""
    rng = np.random.default_rng(case["seed"])
    n, c, h, w = case["shape"]
    spec = ConvSpec(kernel=tuple(case["kernel"]), stride=tuple(case["stride"]), pad=tuple(case["pad"]))
    d = rng.standard_normal((n, c, h, w))
    g = rng.standard_normal((case["f"], c, *case["kernel"]))
    oh, ow = spec.out_dims(h, w)
    dy = rng.standard_normal((n, case["f"], oh, ow))
    return spec, d, g, dy


def backward_cases():
    arrays = {}
    meta = []
    for case in backward_case_specs():
        spec, d, g, dy = backward_inputs(case)
        plan = plan_decomposition(spec)
        key = case["name"]
        gd64, gw64 = dwm_backward(dy, plan, d, g, precision=np.float64)
        gd32, gw32 = dwm_backward(dy, plan, d, g, precision=np.float32)
        arrays[f"{key}/gd64"], arrays[f"{key}/gw64"] = gd64, gw64
        m = {k: (list(v) if isinstance(v, tuple) else v) for k, v in case.items()}
        m["ref_mse_gd32"], m["ref_mse_gw32"] = mse(gd32, gd64), mse(gw32, gw64)
        m["input_sums"] = [float(d.sum()), float(g.sum()), float(dy.sum())]
        meta.append(m)
    np.savez_compressed(HERE / "backward_cases.npz", **arrays)
    (HERE / "backward_cases.json").write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    if sys.argv[1:] == ["backward"]:
        backward_cases()
        sys.exit(0)
    if sys.argv[1:] == ["acceptance"]:
        acceptance_14x14()
        sys.exit(0)
    backward_cases()
    acceptance_14x14()
    plans()
    transforms()
    small_cases()
    baseline_samples()
