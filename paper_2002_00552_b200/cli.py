"""``python -m paper_2002_00552_b200.cli conv ...`` -- the reference's
``dwmconv conv`` subcommand (``pkg/src/dwmconv/cli.py:92-128,131-144``) on the
B200 path: DWM1 files in, DWM1 file out, the same flags,
the same stdout stats line and the same exit codes (0 ok, 1 error on stderr).

Only ``--algo dwm`` runs here; ``direct``/``winograd`` are the reference's CPU
baselines (out of scope).  ``--verify`` compares against an independent
direct convolution (cuDNN through torch, in the compute precision) -- a
checking aid, not the computed result.  The other reference subcommands
(gen-transforms, bench, analyze) are host-side analysis tools, out of scope
per SURVEY §8.
"""

import argparse
import json
import sys

import numpy as np

from . import tensorfile
from .convspec import ConvSpec
from .decompose import plan_decomposition, plan_to_json
from .engines import convolve


def _fail(message: str, code: int = 1) -> int:
    print(f"error: {message}", file=sys.stderr)
    return code


def _pair(text: str, name: str):
    vals = [int(v) for v in text.split(",")]
    if len(vals) == 1:
        return vals[0], vals[0]
    if len(vals) == 2:
        return vals[0], vals[1]
    raise ValueError(f"{name} takes one or two comma-separated integers, got {text!r}")


def _pad(text: str):
    vals = [int(v) for v in text.split(",")]
    if len(vals) == 1:
        return (vals[0],) * 4
    if len(vals) == 4:
        return tuple(vals)
    raise ValueError(f"--pad takes one or four comma-separated integers, got {text!r}")


def _direct_check(data, weights, spec, dtype):
    import torch
    t = torch.float64 if dtype == np.float64 else torch.float32
    dev = torch.device("cuda", torch.cuda.current_device())
    x = torch.from_numpy(np.ascontiguousarray(data)).to(dev, t)
    w = torch.from_numpy(np.ascontiguousarray(weights)).to(dev, t)
    top, bottom, left, right = spec.pad
    x = torch.nn.functional.pad(x, (left, right, top, bottom))
    return torch.nn.functional.conv2d(x, w, stride=spec.stride).cpu().numpy()


def cmd_conv(args) -> int:
    try:
        data = tensorfile.read_tensor(args.input)
        weights = tensorfile.read_tensor(args.weights)
    except (OSError, ValueError) as exc:
        return _fail(str(exc))
    kernel = tuple(weights.shape[2:])
    try:
        if args.kernel is not None and _pair(args.kernel, "--kernel") != kernel:
            return _fail(f"--kernel {args.kernel} does not match weights file taps {kernel}")
        stride = _pair(args.stride, "--stride")
        spec = ConvSpec(kernel=kernel, stride=stride, pad=_pad(args.pad))
    except ValueError as exc:
        return _fail(str(exc))
    precision = {"f32": np.float32, "f64": np.float64, None: None}[args.precision]
    try:
        out = convolve(data, weights, spec, algo=args.algo, precision=precision)
    except (ValueError, FloatingPointError) as exc:
        return _fail(str(exc))
    line = (f"algo={args.algo} kernel={kernel[0]}x{kernel[1]} stride={stride[0]}x{stride[1]} "
            f"out={out.y.shape[2]}x{out.y.shape[3]} mults_per_channel_filter={out.flops}")
    if args.verify:
        want = _direct_check(data, weights, spec, precision or data.dtype)
        diff = float(np.max(np.abs(out.y - want))) if out.y.size else 0.0
        line += f" max_abs_diff_vs_direct={diff:.6E}"
    print(line)
    if args.dump_plan:
        print(json.dumps(plan_to_json(plan_decomposition(spec)), indent=2))
    if args.out:
        tensorfile.write_tensor(args.out, out.y)
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2002_00552_b200",
                                 description="DWM convolution on B200 (drop-in for `dwmconv conv`)")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("conv", help="run a single convolution on DWM1 tensor files")
    p.add_argument("--algo", choices=("dwm",), required=True)
    p.add_argument("--in", dest="input", required=True, help="input tensor file (DWM1)")
    p.add_argument("--weights", required=True, help="weights tensor file (F,C,r_h,r_w)")
    p.add_argument("--kernel", help="kernel taps, must match the weights file")
    p.add_argument("--stride", default="1", help="stride, one or two integers")
    p.add_argument("--pad", default="0", help="padding: symmetric value or top,bottom,left,right")
    p.add_argument("--precision", choices=("f32", "f64"), help="compute precision")
    p.add_argument("--out", help="write the output tensor here")
    p.add_argument("--verify", action="store_true", help="report max |dwm - direct|")
    p.add_argument("--dump-plan", action="store_true", help="print the decomposition plan as JSON")
    p.set_defaults(func=cmd_conv)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())
