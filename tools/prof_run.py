"""Run a config's transform a few times (target for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1409_5757_b200 import _native, workloads  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = workloads.CONFIGS[cfg_name]
n, dt = cfg["n"], cfg["dtype"]
x = workloads.make_input(n, dt, cfg["kind"], 1)
y = torch.empty_like(x)
p = _native.NativePlan(n, _native.EFFT_C64 if dt == "complex64" else _native.EFFT_C128, -1, 0)
print(p.describe())
for _ in range(reps):
    p.execute(x.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok")
