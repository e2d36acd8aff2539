"""Time dwm_backward on the BASELINE workloads: data
gradient (forward engine on the adjoint problem) and weight gradient
(dwm_weight_grad) separately, CUDA events on the current stream, after warm-up.
Not a bench.py line (the north star is the forward); an engineering table.

    python tools/bench_backward.py [workload ...] [--batch B] [--steps K]
"""

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2002_00552_b200 import _native, dwm_backward  # noqa: E402
from paper_2002_00552_b200.configs import WORKLOADS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="*", default=list(WORKLOADS))
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--wgrad-algo", default="auto", choices=("auto", "exact", "tc"))
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    lib = _native.load()
    for name in args.workloads:
        wl = WORKLOADS[name]
        n = args.batch or wl.batch
        spec = wl.spec()
        from paper_2002_00552_b200 import plan_decomposition
        plan = plan_decomposition(spec)
        oh, ow = wl.out_hw()
        g = torch.Generator(device=dev).manual_seed(0)
        x = torch.randn(n, wl.c_in, wl.hw, wl.hw, device=dev, generator=g)
        w = torch.randn(wl.c_out, wl.c_in, wl.kernel, wl.kernel, device=dev, generator=g)
        dy = torch.randn(n, wl.c_out, oh, ow, device=dev, generator=g)
        desc = _native.make_desc(n, wl.c_in, wl.hw, wl.hw, wl.c_out, spec.kernel, spec.stride, spec.pad)
        gw = torch.empty_like(w)
        wg_algo = _native.ALGOS[args.wgrad_algo]
        wg_bytes = int(lib.dwm_weight_grad_workspace_bytes(desc, _native.DWM_F32, wg_algo))
        wg_ws = torch.empty(max(wg_bytes, 1), dtype=torch.uint8, device=dev)

        def wgrad():
            _native.check(lib.dwm_weight_grad(desc, _native.DWM_F32, wg_algo, x.data_ptr(), dy.data_ptr(),
                                              gw.data_ptr(),
                                              wg_ws.data_ptr(), wg_bytes, None, torch.cuda.current_stream().cuda_stream))

        def full():
            dwm_backward(dy, plan, x, w, wgrad_algo=args.wgrad_algo)

        res = {"workload": name, "batch": n, "wgrad_algo": args.wgrad_algo}
        for label, fn in (("backward", full), ("weight_grad", wgrad)):
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            res[f"{label}_ms"] = round(e0.elapsed_time(e1) / args.steps, 3)
        res["data_grad_ms_est"] = round(res["backward_ms"] - res["weight_grad_ms"], 3)
        flops = 2 * wl.direct_flops_per_image() * n  # data + weight gradient, direct-equivalent
        res["direct_equiv_tflops"] = round(flops / (res["backward_ms"] * 1e-3) / 1e12, 1)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
