"""Per-call latency of the small-problem path (cfg1: one 56x56 image, 32->32,
5x5): eager dwm_conv2d on device tensors, the same through DWMConvGraph,
and the kernels alone (CUDA events), in microseconds."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2002_00552_b200 import DWMConvGraph, dwm_conv2d  # noqa: E402
from paper_2002_00552_b200.configs import WORKLOADS  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg1-5x5s1"]
dev = torch.device("cuda", 0)
x = torch.randn(wl.batch, wl.c_in, wl.hw, wl.hw, device=dev)
w = torch.randn(wl.c_out, wl.c_in, wl.kernel, wl.kernel, device=dev)
spec = wl.spec()
out = {"workload": wl.name}
for name, fn in (("eager_us", lambda: dwm_conv2d(x, w, spec)),
                 ("eager_nocheck_us", lambda: dwm_conv2d(x, w, spec, check_finite=False)),
                 ("graph_us", None)):
    if fn is None:
        g = DWMConvGraph(x.shape, w.shape, spec, device=dev)
        fn = lambda: g(x, w)  # noqa: E731
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(500):
        fn()
    torch.cuda.synchronize()
    out[name] = 1e6 * (time.perf_counter() - t0) / 500
g = DWMConvGraph(x.shape, w.shape, spec, device=dev, check_finite=False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(500):
    g.graph.replay()
e1.record()
torch.cuda.synchronize()
out["graph_replay_device_us"] = 1e3 * e0.elapsed_time(e1) / 500
print(json.dumps(out))
