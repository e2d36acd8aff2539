"""DWM1 tensor files and the ``conv`` CLI (reference
tensorfile.py:1-58, cli.py:92-144, determinism criterion test_acceptance.py:187-229)."""

import json
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, reference_available
from paper_2002_00552_b200 import ConvSpec, flops_dwm, plan_decomposition, tensorfile
from paper_2002_00552_b200.cli import main

CASES = {c["name"]: c for c in json.loads((GOLDEN / "cases.json").read_text())}
ARR = np.load(GOLDEN / "small_cases.npz")


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_roundtrip(tmp_path, dtype):
    a = np.random.default_rng(0).standard_normal((2, 3, 5, 7)).astype(dtype)
    p = tmp_path / "a.dwm"
    tensorfile.write_tensor(p, a)
    b = tensorfile.read_tensor(p)
    assert b.dtype == dtype and np.array_equal(a, b)
    raw = p.read_bytes()
    assert raw[:4] == b"DWM1" and len(raw) == 25 + a.nbytes and raw[24] == (0 if dtype == np.float32 else 1)


def test_bytes_identical_to_reference_writer(tmp_path, ref):
    from dwmconv import tensorfile as rtf
    a = np.random.default_rng(1).standard_normal((1, 2, 3, 4))
    for dt in (np.float32, np.float64):
        rtf.write_tensor(tmp_path / "r.dwm", a.astype(dt))
        tensorfile.write_tensor(tmp_path / "o.dwm", a.astype(dt))
        assert (tmp_path / "r.dwm").read_bytes() == (tmp_path / "o.dwm").read_bytes()
        assert np.array_equal(rtf.read_tensor(tmp_path / "o.dwm"), tensorfile.read_tensor(tmp_path / "r.dwm"))


def test_malformed_files(tmp_path):
    good = tmp_path / "g.dwm"
    tensorfile.write_tensor(good, np.zeros((1, 1, 2, 2), np.float32))
    raw = good.read_bytes()
    cases = {"truncated header": raw[:10], "bad magic": b"XWM1" + raw[4:],
             "rank 3 unsupported": raw[:4] + (3).to_bytes(4, "little") + raw[8:],
             "unknown precision tag": raw[:24] + bytes([7]) + raw[25:],
             "payload is": raw[:-1]}
    for msg, blob in cases.items():
        p = tmp_path / "bad.dwm"
        p.write_bytes(blob)
        with pytest.raises(ValueError, match=msg):
            tensorfile.read_tensor(p)
    with pytest.raises(TypeError):
        tensorfile.write_tensor(tmp_path / "x.dwm", np.zeros((1, 1, 2, 2), np.int32))
    with pytest.raises(ValueError):
        tensorfile.write_tensor(tmp_path / "x.dwm", np.zeros((2, 2), np.float32))


def test_cli_errors_before_compute(tmp_path, capsys):
    tensorfile.write_tensor(tmp_path / "d.dwm", np.zeros((1, 1, 8, 8)))
    tensorfile.write_tensor(tmp_path / "w.dwm", np.zeros((1, 1, 3, 3)))
    base = ["conv", "--algo", "dwm", "--in", str(tmp_path / "d.dwm"), "--weights", str(tmp_path / "w.dwm")]
    assert main(base + ["--kernel", "5"]) == 1
    assert "does not match weights file taps" in capsys.readouterr().err
    assert main(base + ["--pad", "1,2"]) == 1
    assert main(["conv", "--algo", "dwm", "--in", str(tmp_path / "missing"), "--weights", "x"]) == 1
    with pytest.raises(SystemExit):
        main(base[:2] + ["direct"] + base[3:])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["param_r7_s2", "accept_r11_s4", "chan0_c3_f64"])
def test_cli_conv_matches_reference_and_is_deterministic(cuda, tmp_path, name):
    c = CASES[name]
    d, g = ARR[f"{name}/data"], ARR[f"{name}/weights"]
    tensorfile.write_tensor(tmp_path / "d.dwm", d)
    tensorfile.write_tensor(tmp_path / "w.dwm", g)
    stride = ",".join(str(s) for s in c["stride"])
    pad = ",".join(str(p) for p in c["pad"])
    outs, lines = [], []
    for i in range(2):
        out = tmp_path / f"y{i}.dwm"
        r = subprocess.run([sys.executable, "-m", "paper_2002_00552_b200.cli", "conv", "--algo", "dwm",
                            "--in", str(tmp_path / "d.dwm"), "--weights", str(tmp_path / "w.dwm"),
                            "--stride", stride, "--pad", pad, "--precision", "f32", "--out", str(out)],
                           cwd=ROOT, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        outs.append(out.read_bytes())
        lines.append(r.stdout)
    assert outs[0] == outs[1] and lines[0] == lines[1]
    y = tensorfile.read_tensor(tmp_path / "y0.dwm")
    want = ARR[f"{name}/dwm32"]
    assert y.dtype == np.float32 and y.shape == want.shape
    assert np.array_equal(y, want)  # C_in <= 4: bit-identical to the reference
    spec = ConvSpec(kernel=tuple(c["kernel"]), stride=tuple(c["stride"]), pad=tuple(c["pad"]))
    k = c["kernel"]
    flops = flops_dwm(plan_decomposition(spec), want.shape[2:])
    assert lines[0].strip() == (f"algo=dwm kernel={k[0]}x{k[1]} stride={c['stride'][0]}x{c['stride'][1]} "
                                f"out={want.shape[2]}x{want.shape[3]} mults_per_channel_filter={flops}")


@pytest.mark.gpu
def test_cli_verify_and_dump_plan(cuda, tmp_path, capsys):
    name = "grid_r5_s2"
    tensorfile.write_tensor(tmp_path / "d.dwm", ARR[f"{name}/data"])
    tensorfile.write_tensor(tmp_path / "w.dwm", ARR[f"{name}/weights"])
    rc = main(["conv", "--algo", "dwm", "--in", str(tmp_path / "d.dwm"), "--weights", str(tmp_path / "w.dwm"),
               "--stride", "2", "--pad", "1", "--verify", "--dump-plan"])
    assert rc == 0
    out = capsys.readouterr().out
    first, rest = out.split("\n", 1)
    diff = float(first.split("max_abs_diff_vs_direct=")[1])
    assert diff <= 1e-10  # binary64 input -> binary64 compute
    assert json.loads(rest)["kernel"] == [5, 5]
