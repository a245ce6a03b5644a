"""Time single-pass column plans (one tile type, no staging) on an N=2^30 c64 array."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1409_5757_b200 import _native
n = 1 << 30
x = torch.randn(n, dtype=torch.complex64, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
for length in (16, 64, 256, 512, 1024, 32768):
    for tw in (0, n):
        try:
            p = _native.NativePlan(length, _native.EFFT_C64, -1, 0, 0, columns=(n // length, tw, 0))
        except Exception as e:
            print(length, "fail", e); continue
        for _ in range(2): p.execute(x.data_ptr(), y.data_ptr(), s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): p.execute(x.data_ptr(), y.data_ptr(), s)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"len={length:6d} tw={'N' if tw else '-'} {ms:.3f} ms  {2*n*8/ms/1e6:.0f} GB/s  {p.describe().splitlines()[1][:90]}", flush=True)
# plain copy for reference
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): y.copy_(x)
e1.record(); torch.cuda.synchronize()
print("torch copy", e0.elapsed_time(e1) / 5, "ms")
