# Small tcgen05 forward through the fused and the staged C-ABI paths on odd shapes (partial filter block,
# odd width); prints whether both paths agree bit for bit.  (compute-sanitizer is not available on the pool.)
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2002_00552_b200 import ConvSpec, dwm_conv2d, _native
spec = ConvSpec(kernel=(5, 5), stride=(1, 1), pad=(2, 2, 2, 2))
x = torch.randn(3, 64, 9, 11, device="cuda"); w = torch.randn(70, 64, 5, 5, device="cuda")
y = dwm_conv2d(x, w, spec, algo="tc") if "algo" in dwm_conv2d.__code__.co_varnames else dwm_conv2d(x, w, spec)
torch.cuda.synchronize(); print("ok", y.shape)
lib = _native.load(); d = _native.make_desc(3, 64, 9, 11, 70, spec.kernel, spec.stride, spec.pad)
u = torch.empty(lib.dwm_filter_bytes(d, 0, 2), dtype=torch.uint8, device="cuda")
_native.check(lib.dwm_prepare_filter(d, 0, 2, w.data_ptr(), u.data_ptr(), None))
v = torch.empty(d.num_freqs * d.tiles * 64, device="cuda"); rb = lib.dwm_range_bytes(d)
sc = torch.empty(rb, dtype=torch.uint8, device="cuda"); flag = torch.zeros(1, dtype=torch.int32, device="cuda")
_native.check(lib.dwm_input_transform(d, 0, x.data_ptr(), v.data_ptr(), None))
y2 = torch.empty_like(y)
_native.check(lib.dwm_gemm_output(d, 0, 2, v.data_ptr(), u.data_ptr(), y2.data_ptr(), flag.data_ptr(), sc.data_ptr(), rb, None))
torch.cuda.synchronize(); print("ok2", torch.equal(y, y2))
