import sys, time, faulthandler, ctypes
faulthandler.enable()
sys.path.insert(0, "/root/repo")
print("start", flush=True)
import numpy as np, torch
print("torch ok", torch.cuda.is_available(), flush=True)
from paper_2002_00552_b200 import _native
lib = _native.load()
d = _native.make_desc(1, 32, 8, 8, 64, (3, 3), (1, 1), (1, 1, 1, 1))
print("desc", d.tiles, d.num_freqs, flush=True)
x = torch.randn(1, 32, 8, 8, device="cuda"); w = torch.randn(64, 32, 3, 3, device="cuda")
y = torch.empty(1, 64, 8, 8, device="cuda")
algo = _native.DWM_ALGO_TC
print("select", lib.dwm_select_algo(d, 0, algo), flush=True)
ws_bytes = lib.dwm_workspace_bytes(d, 0, algo)
ws = torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
v_bytes = d.num_freqs * d.tiles * d.c * 4
V = ws.data_ptr(); U = V + ((v_bytes + 255) // 256) * 256
print("filter", lib.dwm_filter_transform(d, 0, w.data_ptr(), U, s), flush=True)  # plain (not split) just to run
torch.cuda.synchronize(); print("filter done", flush=True)
print("input", lib.dwm_input_transform(d, 0, x.data_ptr(), V, s), flush=True)
torch.cuda.synchronize(); print("input done", flush=True)
st = lib.dwm_gemm_output(d, 0, algo, V, U, y.data_ptr(), flag.data_ptr(), None, 0, s)
print("gemm launched", st, _native.last_error(), flush=True)
t = time.time()
while not torch.cuda.current_stream().query():
    time.sleep(0.5)
    if time.time() - t > 20:
        print("gemm still running after 20 s", flush=True); break
print("query done", time.time() - t, flush=True)
torch.cuda.synchronize()
print("sync ok", flush=True)
