"""One full-batch DWM forward of a BASELINE workload, bracketed by
cudaProfilerStart/Stop, for ncu captures:

    ncu --profile-from-start off --set full --clock-control none --import-source on \
        -o gpurun_out/ncu_cfg4r11 python tools/ncu_forward.py cfg4-11x11s1

A warm-up forward runs first (outside the profiled range) so module loading,
tensor-map encoding and allocator growth are not in the capture.
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2002_00552_b200 import _native  # noqa: E402
from paper_2002_00552_b200.configs import WORKLOADS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--algo", default="auto")
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--reps", type=int, default=1)
args = ap.parse_args()

wl = WORKLOADS[args.workload]
n = args.batch or wl.batch
spec = wl.spec()
lib = _native.load()
dev = torch.device("cuda", 0)
desc = _native.make_desc(n, wl.c_in, wl.hw, wl.hw, wl.c_out, spec.kernel, spec.stride, spec.pad)
algo = _native.ALGOS[args.algo]
ws_bytes = lib.dwm_workspace_bytes(desc, _native.DWM_F32, algo)
x = torch.randn(n, wl.c_in, wl.hw, wl.hw, device=dev)
w = torch.randn(wl.c_out, wl.c_in, wl.kernel, wl.kernel, device=dev)
y = torch.empty(n, wl.c_out, desc.oh, desc.ow, device=dev)
ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
flag = torch.zeros(1, dtype=torch.int32, device=dev)
s = torch.cuda.current_stream().cuda_stream


def fwd():
    _native.check(lib.dwm_conv2d_forward(desc, _native.DWM_F32, algo, x.data_ptr(), w.data_ptr(), y.data_ptr(),
                                         ws.data_ptr(), ws_bytes, flag.data_ptr(), s))


fwd()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(args.reps):
    fwd()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"{args.workload} n={n} engine={_native.ALGO_NAMES[lib.dwm_select_algo(desc, 0, algo)]} ok")
