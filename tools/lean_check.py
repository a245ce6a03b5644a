"""Dev tool: lean c64 path vs cuFFT (torch.fft) and vs the generic path; timings."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1409_5757_b200 import _native  # noqa: E402


def rel(a, b):
    return float(torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b))


def run(p, x, y, reps=1):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p.execute(x.data_ptr(), y.data_ptr(), s.cuda_stream)
    e0.record()
    for _ in range(reps):
        p.execute(x.data_ptr(), y.data_ptr(), s.cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


logs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["26", "27", "28", "29", "30"]
c128 = len(sys.argv) > 2 and sys.argv[2] == "c128"
tdt, ndt, esz = (torch.complex128, _native.EFFT_C128, 16) if c128 else (torch.complex64, _native.EFFT_C64, 8)
for tok in logs:
    L = int(tok.split("x")[-1])
    n = (int(tok.split("x")[0]) if "x" in tok else 1) << L
    g = torch.Generator(device="cuda").manual_seed(L)
    x = torch.randn(n, dtype=tdt, device="cuda", generator=g)
    y = torch.empty_like(x)
    p = _native.NativePlan(n, ndt, -1, 0)
    print(p.describe().strip(), flush=True)
    p.enable_timing(True)
    ms = run(p, x, y, 3)
    pt = p.launch_times_ms()
    if n * esz <= (16 << 30):
        ref = torch.fft.fft(x)
        err = rel(y, ref)
        del ref
    else:
        err = float("nan")
    pi = _native.NativePlan(n, ndt, 1, 0)
    torch.cuda.empty_cache()
    z = torch.empty_like(x) if n * esz <= (32 << 30) else None
    if z is None:  # 64 GiB arrays: round trip in place of the input (x regenerated for the check)
        pi.execute(y.data_ptr(), x.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        z, x = x, None
        torch.cuda.empty_cache()
        x = torch.randn(n, dtype=tdt, device="cuda", generator=torch.Generator(device="cuda").manual_seed(L)) \
            if False else None
        rt = float("nan")
    else:
        pi.execute(y.data_ptr(), z.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        rt = rel(z, x)
    gbs = [2 * n * esz / (t * 1e-3) / 1e9 for t in pt]
    print(f"N={tok} lean: {ms:.3f} ms  passes {['%.3f' % t for t in pt]} ms = {['%.0f' % v for v in gbs]} GB/s  "
          f"err_vs_cufft={err:.3e} roundtrip={rt:.3e}", flush=True)
    del z, x, y
    torch.cuda.empty_cache()
