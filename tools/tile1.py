"""One single-pass column plan (len from argv) on N=2^30 c64, run 3 times (ncu target)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1409_5757_b200 import _native
n = 1 << 30
length = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dt = sys.argv[2] if len(sys.argv) > 2 else "c64"
tdt = torch.complex64 if dt == "c64" else torch.complex128
n = n if dt == "c64" else n // 2
x = torch.randn(n, dtype=tdt, device="cuda")
y = torch.empty_like(x)
p = _native.NativePlan(length, _native.EFFT_C64 if dt == "c64" else _native.EFFT_C128, -1, 0, 0,
                       columns=(n // length, 0, 0))
for _ in range(3):
    p.execute(x.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", p.describe())
