"""Per-role wait profile of the tcgen05 GEMM (needs a -DDWM_TC_PROFILE build of
the library in place of the in-tree one; tools/ab/mklib.sh prof
dwm_gemm_tc.cu=... with ABFLAGS=-DDWM_TC_PROFILE).  Prints, per ablation flag
set, the GEMM time and each role's share of its cycles spent waiting."""
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2002_00552_b200 import _native  # noqa: E402
from paper_2002_00552_b200.configs import WORKLOADS  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg4-7x7s1"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else wl.batch
lib = _native.load()
lib.dwm_debug_tc_profile.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
lib.dwm_debug_tc_flags.argtypes = [ctypes.c_int]
spec = wl.spec()
desc = _native.make_desc(n, wl.c_in, wl.hw, wl.hw, wl.c_out, spec.kernel, spec.stride, spec.pad)
ws_bytes = lib.dwm_workspace_bytes(desc, 0, 2)
x = torch.randn(n, wl.c_in, wl.hw, wl.hw, device="cuda")
w = torch.randn(wl.c_out, wl.c_in, wl.kernel, wl.kernel, device="cuda")
y = torch.empty(n, wl.c_out, desc.oh, desc.ow, device="cuda")
ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
V = ws.data_ptr()
U = V + (desc.num_freqs * desc.tiles * desc.c * 4 + 255) // 256 * 256
R = U + (lib.dwm_filter_bytes(desc, 0, 2) + 255) // 256 * 256  # max|x| range slots (after V and U)
_native.check(lib.dwm_conv2d_forward(desc, 0, 2, x.data_ptr(), w.data_ptr(), y.data_ptr(), V, ws_bytes,
                                     flag.data_ptr(), s))
buf = (ctypes.c_ulonglong * 32)()
names = ["VTMA  wait v_empty", "MMA   wait acc_empty", "MMA   wait a_full", "MMA   wait u_full", "CONV  wait v_full",
         "CONV  wait a_empty", "EPI   wait acc_full"]
slots = [0, 4, 5, 6, 8, 9, 12]
for flags in [0, 1, 2, 4, 8, 1 | 2, 1 | 2 | 8, 1 | 2 | 4 | 8]:
    lib.dwm_debug_tc_flags(flags)
    lib.dwm_debug_tc_profile(buf, 1)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    _native.check(lib.dwm_gemm_output_tc(desc, V, U, R, y.data_ptr(), flag.data_ptr(), s))
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    lib.dwm_debug_tc_profile(buf, 1)
    tot = {r: buf[r * 4 + 3] or 1 for r in range(4)}
    parts = [f"{nm} {100 * buf[sl] / tot[sl // 4]:5.1f}%" for nm, sl in zip(names, slots)]
    print(f"flags={flags:2d} gemm {ms:7.3f} ms | " + " | ".join(parts), flush=True)
lib.dwm_debug_tc_flags(0)
