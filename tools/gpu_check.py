"""Quick GPU sanity sweep: CUDA path vs numpy fp64 FFT (dev tool, not a test)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1409_5757_b200 as efft
from paper_1409_5757_b200 import _native

def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))

sizes = [int(s) for s in sys.argv[1].split(",")] if len(sys.argv) > 1 else \
    [2, 4, 8, 16, 64, 256, 512, 1024, 3*1024, 4096, 2**14, 3*2**14, 2**16, 2**18, 2**19, 2**20, 2**21, 3*2**20, 2**22]
rng = np.random.default_rng(0)
for n in sizes:
    for dt in ("complex64", "complex128"):
        x = (rng.standard_normal(n) + 1j * rng.standard_normal(n))
        ref = np.fft.fft(x)
        try:
            p = _native.NativePlan(n, _native.EFFT_C64 if dt == "complex64" else _native.EFFT_C128, -1, 0)
            tdt = torch.complex64 if dt == "complex64" else torch.complex128
            xi = torch.from_numpy(x.astype(np.complex64 if dt == "complex64" else np.complex128)).cuda()
            yo = torch.empty_like(xi)
            p.execute(xi.data_ptr(), yo.data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            y = yo.cpu().numpy()
            pi = _native.NativePlan(n, p.dtype, 1, 0)
            zo = torch.empty_like(xi)
            pi.execute(yo.data_ptr(), zo.data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            z = zo.cpu().numpy()
            print(f"n={n:>9} {dt:10s} fwd_err={rel(y, ref):.3e} rt_err={rel(z, x):.3e} | {p.describe().splitlines()[1:] }", flush=True)
        except Exception as exc:
            print(f"n={n} {dt} FAILED {type(exc).__name__}: {exc}", flush=True)
