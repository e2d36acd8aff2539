"""Is the tcgen05 GEMM L2-bandwidth bound?  Time gemm_output per unit of MMA
work for F = 64 (V read once per m-block) vs F = 256 (V read by 4 n-block CTAs)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2002_00552_b200 import _native
lib = _native.load()
s = torch.cuda.current_stream().cuda_stream
for F, N in [(64, 512), (256, 512), (128, 512)]:
    d = _native.make_desc(N, 256, 28, 28, F, (7, 7), (1, 1), (3, 3, 3, 3))
    x = torch.randn(N, 256, 28, 28, device="cuda"); w = torch.randn(F, 256, 7, 7, device="cuda")
    y = torch.empty(N, F, 28, 28, device="cuda")
    ws = torch.empty(lib.dwm_workspace_bytes(d, 0, 2), dtype=torch.uint8, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _native.check(lib.dwm_conv2d_forward(d, 0, 2, x.data_ptr(), w.data_ptr(), y.data_ptr(), ws.data_ptr(), ws.numel(), flag.data_ptr(), s))
    vb = d.num_freqs * d.tiles * 256 * 4
    V = ws.data_ptr(); U = V + ((vb + 255) // 256) * 256
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        lib.dwm_gemm_output(d, 0, 2, V, U, y.data_ptr(), flag.data_ptr(), None, 0, s)
    e0.record()
    for _ in range(5):
        lib.dwm_gemm_output(d, 0, 2, V, U, y.data_ptr(), flag.data_ptr(), None, 0, s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    flops = 2.0 * 256 * F * d.tiles * d.num_freqs * 3
    print(f"F={F}: {ms:.3f} ms  {flops/ms/1e9:.1f} TFLOP/s tensor (3xTF32)", flush=True)
    del x, w, y, ws
