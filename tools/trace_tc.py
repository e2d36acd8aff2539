"""Run one tcgen05 GEMM launch of a workload under the trace build (debug)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2002_00552_b200 import _native
from paper_2002_00552_b200.configs import WORKLOADS
wl = WORKLOADS[sys.argv[1]]
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 64
lib = _native.load()
spec = wl.spec()
d = _native.make_desc(batch, wl.c_in, wl.hw, wl.hw, wl.c_out, spec.kernel, spec.stride, spec.pad)
x = torch.randn(batch, wl.c_in, wl.hw, wl.hw, device="cuda"); w = torch.randn(wl.c_out, wl.c_in, wl.kernel, wl.kernel, device="cuda")
y = torch.empty(batch, wl.c_out, d.oh, d.ow, device="cuda")
ws = torch.empty(lib.dwm_workspace_bytes(d, 0, 2), dtype=torch.uint8, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    _native.check(lib.dwm_conv2d_forward(d, 0, 2, x.data_ptr(), w.data_ptr(), y.data_ptr(), ws.data_ptr(), ws.numel(), flag.data_ptr(), s))
torch.cuda.synchronize()
print("ok")
