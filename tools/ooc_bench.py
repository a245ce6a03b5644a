"""Dev tool: out-of-core transform throughput (host array -> host array) vs the in-HBM e2e path."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1409_5757_b200 import _native, outofcore  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 30
budget = int(float(sys.argv[2])) if len(sys.argv) > 2 else 1 << 32
n = 1 << lg
x = torch.randn(n, dtype=torch.complex64).numpy()
out = np.empty_like(x)
print("blocks", outofcore.plan_blocks(n, "complex64", budget), flush=True)
for pinned in (False, True):
    if pinned:
        xt = torch.from_numpy(x).pin_memory()
        ot = torch.empty(n, dtype=torch.complex64).pin_memory()
        xi, oi = xt.numpy(), ot.numpy()
    else:
        xi, oi = x, out
    for rep in range(2):
        t0 = time.perf_counter()
        outofcore.transform(xi, device_bytes=budget, out=oi)
        dt = time.perf_counter() - t0
        print(f"2^{lg} c64 budget={budget >> 20} MiB pinned={pinned} rep={rep}: {dt * 1e3:.1f} ms "
              f"= {5 * n * lg / dt / 1e9:.0f} GFLOP/s, {4 * n * 8 / dt / 1e9:.1f} GB/s PCIe (both directions)",
              flush=True)
# spot check against the in-HBM transform
xd = torch.from_numpy(x).cuda()
yd = torch.empty_like(xd)
p = _native.NativePlan(n, _native.EFFT_C64, -1, 0)
p.execute(xd.data_ptr(), yd.data_ptr(), torch.cuda.current_stream().cuda_stream)
ref = yd.cpu().numpy()
print("rel diff vs in-HBM:", float(np.linalg.norm(oi - ref) / np.linalg.norm(ref)))
