"""Dev check of the pipelined pair kernel (EFFT_LEAN_PIPE) against the default lean
path: rel-L2 between the two (and vs torch.fft where it fits), per-pass device times.
Usage: python tools/pipe_check.py [log2n,...] [masks e.g. 0,1,2,3] [steps].  GPU only."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1409_5757_b200 import _native  # noqa: E402


def rel(a, b):
    return (torch.linalg.vector_norm((a - b).to(torch.complex128)) /
            torch.linalg.vector_norm(b.to(torch.complex128))).item()


def main():
    logs = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "30").split(",")]
    masks = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0,1,2,3").split(",")]
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    var = sys.argv[4] if len(sys.argv) > 4 else "EFFT_LEAN_PIPE"
    s = torch.cuda.current_stream().cuda_stream
    for L in logs:
        n = 1 << L
        g = torch.Generator(device="cuda").manual_seed(L)
        x = torch.randn(n, dtype=torch.complex64, device="cuda", generator=g)
        ref = None
        for m in masks:
            os.environ[var] = str(m)
            p = _native.NativePlan(n, _native.EFFT_C64, -1, 0, _native.EFFT_FLAG_CHECK_FINITE)
            y = torch.empty_like(x)
            p.execute(x.data_ptr(), y.data_ptr(), s)
            torch.cuda.synchronize()
            if ref is None:
                ref = y.clone()
                if L <= 28:
                    print(f"2^{L} {var}={m}: rel-L2 vs torch.fft {rel(y, torch.fft.fft(x)):.3e}", flush=True)
            else:
                print(f"2^{L} {var}={m}: rel-L2 vs first {rel(y, ref):.3e}  flag {p.nonfinite_seen(s)}", flush=True)
            p.enable_timing(steps)
            for _ in range(3):
                p.execute(x.data_ptr(), y.data_ptr(), s)
            p.enable_timing(steps)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                p.execute(x.data_ptr(), y.data_ptr(), s)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            lt = p.launch_times_ms()
            print(f"2^{L} {var}={m}: {ms:.3f} ms  {5 * n * L / ms / 1e6:.0f} GFLOP/s  passes "
                  f"{[round(v, 3) for v in lt]} ms", flush=True)
            print("   ", " || ".join(p.describe().strip().splitlines()[-2:]), flush=True)
            del p, y
        del x, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
