"""Time the generic two-pass plans over EFFT_SPLIT_T1 for sizes below the lean
range (c128 N < 2^26, c64 N < 2^24, M * 2^t).  Prints ms per transform for
each t1 (L2 flushed before every timed transform).  GPU only; experiment tool."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1:  # child: one (n, dtype, t1)
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1409_5757_b200 import _native
    n, dt = int(sys.argv[1]), sys.argv[2]
    tdt = torch.complex128 if dt == "c128" else torch.complex64
    x = torch.randn(n, dtype=tdt, device="cuda")
    y = torch.empty_like(x)
    p = _native.NativePlan(n, _native.EFFT_C128 if dt == "c128" else _native.EFFT_C64, -1, 0)
    sid = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(5):
        p.execute(x.data_ptr(), y.data_ptr(), sid)
    ts = []
    for _ in range(30):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p.execute(x.data_ptr(), y.data_ptr(), sid)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    # every timed split must also be right: rel-L2 against torch's fp64 FFT
    ref = torch.fft.fft(x.to(torch.complex128))
    err = (torch.linalg.vector_norm(y.to(torch.complex128) - ref) / torch.linalg.vector_norm(ref)).item()
    lg = max(1.0, float(torch.tensor(float(n)).log2()))
    assert err <= (1e-12 if dt == "c128" else 1e-5) * lg, (n, dt, os.environ.get("EFFT_SPLIT_T1"), err)
    plan = [l.split(" grid")[0] for l in p.describe().splitlines()[1:]]
    print(json.dumps({"n": n, "dtype": dt, "t1": os.environ.get("EFFT_SPLIT_T1", "default"),
                      "ms_median": round(ts[len(ts) // 2], 4), "rel_l2": err, "plan": plan}))
    sys.exit(0)

cases = [(1 << 21, "c128"), (1 << 23, "c128"), (1 << 25, "c128"), (3 << 20, "c128"), (5 << 20, "c128"),
         (1 << 21, "c64"), (1 << 22, "c64"), (1 << 23, "c64"), (3 << 21, "c64")]
for n, dt in cases:
    t = (n & -n).bit_length() - 1
    for t1 in ["default"] + list(range(7, t - 6)):
        env = dict(os.environ)
        env.pop("EFFT_SPLIT_T1", None)
        if t1 != "default":
            env["EFFT_SPLIT_T1"] = str(t1)
        r = subprocess.run([sys.executable, __file__, str(n), dt], env=env, capture_output=True, text=True,
                           timeout=120)
        out = [l for l in r.stdout.splitlines() if l.startswith("{")]
        print(out[-1] if out else json.dumps({"n": n, "dtype": dt, "t1": t1, "error": r.stderr[-300:]}),
              flush=True)
