"""Dev tool: device time of one transform per size (warm, L2-flushed between runs).
Usage: python tools/size_times.py c64|c128 n1,n2,...  (n as integers or like 3x2^20)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1409_5757_b200 import _native


def parse(tok):
    if "x2^" in tok:
        m, e = tok.split("x2^")
        return int(m) << int(e)
    if tok.startswith("2^"):
        return 1 << int(tok[2:])
    return int(tok)


dt = sys.argv[1]
tdt, ndt = (torch.complex64, _native.EFFT_C64) if dt == "c64" else (torch.complex128, _native.EFFT_C128)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for tok in sys.argv[2].split(","):
    n = parse(tok)
    x = torch.randn(n, dtype=tdt, device="cuda")
    y = torch.empty_like(x)
    p = _native.NativePlan(n, ndt, -1, 0, _native.EFFT_FLAG_CHECK_FINITE)
    for _ in range(3):
        p.execute(x.data_ptr(), y.data_ptr(), s)
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p.execute(x.data_ptr(), y.data_ptr(), s)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ref = torch.fft.fft(x)
    err = (torch.linalg.vector_norm((y - ref).to(torch.complex128)) / torch.linalg.vector_norm(ref.to(torch.complex128))).item()
    print(f"{dt} n={tok:>8s} median {ts[5]*1e3:8.1f} us  min {ts[0]*1e3:8.1f} us  rel-L2 vs torch.fft {err:.2e}", flush=True)
