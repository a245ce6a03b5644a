"""Single-pass column plans on an L2-resident array (n=2^21 c64): SM-compute throughput of a tile."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1409_5757_b200 import _native
for n in (1 << 21, 1 << 30):
    x = torch.randn(n, dtype=torch.complex64, device="cuda")
    y = torch.empty_like(x)
    s = torch.cuda.current_stream().cuda_stream
    for length in (16, 256, 512):
        for tw in (0, n):
            p = _native.NativePlan(length, _native.EFFT_C64, -1, 0, 0, columns=(n // length, tw, 0))
            reps = 200 if n < (1 << 25) else 5
            for _ in range(3): p.execute(x.data_ptr(), y.data_ptr(), s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps): p.execute(x.data_ptr(), y.data_ptr(), s)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            print(f"n=2^{n.bit_length()-1} len={length:4d} tw={'N' if tw else '-'} {ms*1e3:9.1f} us  -> {ms * (1<<30) / n:.3f} ms per 2^30", flush=True)
