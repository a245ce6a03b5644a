"""Dev check of the TMA pass path (tpass.cu) against the lean path and the oracle
at N = 2^30 complex64: rel-L2 between the two GPU paths, fp64-oracle spot
values, round trip, and per-pass device times of both.  GPU only."""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1409_5757_b200 import _native, workloads  # noqa: E402
import oracle  # noqa: E402


def make_plan(n, direction, tpass):
    os.environ["EFFT_TPASS"] = "1" if tpass else "0"
    p = _native.NativePlan(n, _native.EFFT_C64, direction, 0, _native.EFFT_FLAG_CHECK_FINITE)
    return p


def rel(a, b):
    return (torch.linalg.vector_norm((a - b).to(torch.complex128)) /
            torch.linalg.vector_norm(b.to(torch.complex128))).item()


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    x = workloads.make_input(n, "complex64", "normal", workloads.seed_for("c3"))
    s = torch.cuda.current_stream().cuda_stream
    pt = make_plan(n, -1, True)
    pl = make_plan(n, -1, False)
    print(pt.describe())
    yt = torch.empty_like(x)
    yl = torch.empty_like(x)
    pt.execute(x.data_ptr(), yt.data_ptr(), s)
    pl.execute(x.data_ptr(), yl.data_ptr(), s)
    torch.cuda.synchronize()
    print("nonfinite flag (must be False):", pt.nonfinite_seen(s))
    print(f"rel-L2 tpass vs lean: {rel(yt, yl):.3e}")
    ks = np.array([0, 1, 2, 12345, n // 2, n - 1] + list(np.random.default_rng(3).integers(0, n, 6)))
    xh = x.cpu().numpy()
    ex = oracle.dft_at(xh, ks)
    yk = yt[torch.from_numpy(ks).cuda()].cpu().numpy().astype(np.complex128)
    scale = np.sqrt(np.mean(np.abs(ex) ** 2))
    print(f"spot max err vs fp64 direct sums: {np.max(np.abs(yk - ex) / np.maximum(np.abs(ex), scale)):.3e}")
    pi = make_plan(n, 1, True)
    z = torch.empty_like(x)
    pi.execute(yt.data_ptr(), z.data_ptr(), s)
    torch.cuda.synchronize()
    print(f"round trip rel-L2: {rel(z, x):.3e}")
    del z
    for name, p, y in (("tpass", pt, yt), ("lean", pl, yl)):
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
        gf = 5 * n * math.log2(n) / (ms * 1e-3) / 1e9
        print(f"{name}: {ms:.3f} ms/transform  {gf:.0f} GFLOP/s  passes {[round(v, 3) for v in lt]} ms "
              f"-> {[round(2 * n * 8 / (v * 1e-3) / 1e9) for v in lt]} GB/s")


if __name__ == "__main__":
    main()
