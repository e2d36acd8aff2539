"""Quick check of the tcgen05 engine against the oracle on small cases (GPU)."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from oracle.dwm_oracle import direct_conv2d_f64, dwm_conv2d_oracle, draw, mse
from paper_2002_00552_b200 import ConvSpec, dwm_conv2d

cases = [((3, 3), (1, 1), 8, 32, 64, 1), ((3, 3), (1, 1), 14, 64, 64, 2), ((5, 5), (2, 2), 16, 128, 128, 1),
         ((7, 7), (1, 1), 28, 256, 256, 1), ((11, 11), (1, 1), 28, 256, 256, 1), ((5, 5), (2, 2), 56, 128, 256, 1)]
for k, s, hw, c, f, n in cases:
    spec = ConvSpec(kernel=k, stride=s, pad=(k[0] // 2,) * 4)
    d, g = draw(1, k, s, hw, c, f, n)
    t = time.time()
    y = dwm_conv2d(d.astype(np.float32), g.astype(np.float32), spec, algo="tc")
    dt = time.time() - t
    y64 = direct_conv2d_f64(d, g, spec)
    ref = dwm_conv2d_oracle(d, g, spec)
    print(f"{k} {s} hw={hw} C={c} F={n}: mse tc {mse(y, y64):.3e} ref {mse(ref, y64):.3e} "
          f"max|tc-ref| {np.max(np.abs(y - ref)):.3e}  ({dt:.2f}s)", flush=True)
