"""Direct single-pass column plans on N=2^30 c64 (EFFT_DIRECT_TP selects the TMA kernel)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1409_5757_b200 import _native
n = 1 << 30
x = torch.randn(n, dtype=torch.complex64, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
for length in (16, 64, 256, 512):
    for tw in (0, n):
        p = _native.NativePlan(length, _native.EFFT_C64, -1, 0, 0, columns=(n // length, tw, 0))
        for _ in range(2): p.execute(x.data_ptr(), y.data_ptr(), s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): p.execute(x.data_ptr(), y.data_ptr(), s)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"len={length:4d} tw={'N' if tw else '-'} {ms:.3f} ms {p.describe().splitlines()[1][:70]}", flush=True)
# correctness of one small column plan vs numpy
m, cols = 512, 4096
a = (np.random.default_rng(0).standard_normal(m * cols) + 1j * np.random.default_rng(1).standard_normal(m * cols)).astype(np.complex64)
ad = torch.from_numpy(a).cuda(); bd = torch.empty_like(ad)
p = _native.NativePlan(m, _native.EFFT_C64, -1, 0, 0, columns=(cols, 0, 0))
p.execute(ad.data_ptr(), bd.data_ptr(), s); torch.cuda.synchronize()
ref = np.fft.fft(a.reshape(m, cols).astype(np.complex128), axis=0).reshape(-1)
print("colplan rel err", np.linalg.norm(bd.cpu().numpy() - ref) / np.linalg.norm(ref))
