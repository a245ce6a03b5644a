"""Command-line front end on the B200 path: transform, scan, check, bench.

Mirrors the reference CLI (reference pkg/src/efft/cli.py:46-247): the same
subcommands and flags, measurement rows on stdout under one stable CSV
header, diagnostics on stderr, sizes as integers or ``2^K`` (here also
``3x2^K`` for the M x 2^s sizes).  Extensions:
``--dtype float32|complex64|complex128`` (float32 = the reference's real
input and packed PERM output), ``--device``, and the CSV header of
``metrics.CSV_HEADER`` = the reference's columns + gbps, roofline_frac, ngpus,
dtype, rt_err.  Runtimes are device time of the transform (CUDA events), best of
``--repeats``; GFLOP/s uses 2.5 n log2 n for real input (reference
bench.py:27-31) and 5 N log2 N for complex input.

    python -m paper_1409_5757_b200 bench --size 2^30 --splits 3 --dtype complex64
"""

import argparse
import json
import math
import os
import sys

import numpy as np

from .core import handle_create, plan_create
from .errors import EfftError
from .metrics import CSV_HEADER, RunMetrics, algorithmic_bytes

DEFAULT_SEED = 12345  # reference bench.py:23
DEFAULT_REPEATS = 3
FULL_CHECK_LIMIT = 1 << 24      # complex dtypes: full rel-L2 against numpy fp64 up to here
REF_FULL_CHECK_LIMIT = 1 << 14  # float32 (the reference's own path): reference cli.py:33
REF_L2_TOLERANCE = 5e-6         # reference cli.py:34
REF_SPOT_TOLERANCE = 1e-5       # reference cli.py:35
ELEM = {"float32": 8, "complex64": 8, "complex128": 16}  # bytes per complex element the passes move


def parse_size(text: str) -> int:
    """'4096', '2^22' or '3x2^28' -> int (reference bench.py:154-163, plus M x 2^K)."""
    t = text.strip().replace("*", "x")
    mult = 1
    if "x" in t:
        m, t = t.split("x", 1)
        mult = int(m)
    v = (1 << int(t.split("^", 1)[1])) if t.startswith("2^") else int(t)
    if v * mult <= 0:
        raise ValueError(f"size must be positive: {text}")
    return v * mult


def parse_int_list(text: str) -> list:
    return [int(v) for v in text.split(",") if v.strip()]


def roofline_peak_gbs() -> float:
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json next to the package), else the recipe fallback."""
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6650.0


def signal(n: int, dtype: str, seed: int = DEFAULT_SEED) -> np.ndarray:
    rng = np.random.default_rng(seed)
    if dtype == "float32":  # reference bench.py:109-112
        return rng.random(n, dtype=np.float32) - np.float32(0.5)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    return x.astype(np.complex64 if dtype == "complex64" else np.complex128)


def _time_device(handle, repeats: int) -> float:
    """Best-of-`repeats` device time (seconds) of the transform on resident buffers."""
    import torch

    handle.run_device()  # warm-up
    best = math.inf
    for _ in range(max(1, repeats)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        handle.run_device()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return best


def _bench_row(n, splits, workers, dtype, repeats, device, test_mode=False) -> RunMetrics:
    plan = plan_create(n, splits, workers, test_mode=test_mode, dtype=dtype, device=device)
    with handle_create(plan) as h:
        h.data[:] = signal(n, dtype)
        h.run()  # stage the input on the device
        t = _time_device(h, repeats)
        passes = h.launches_per_run()
        nc = n // 2 if dtype == "float32" else n
        gbps = algorithmic_bytes(nc, ELEM[dtype], passes) / t / 1e9
        mem = int(2 * nc * ELEM[dtype] + h._native.workspace_bytes())
    return RunMetrics.from_timing(n, splits, workers, t, complex_input=dtype != "float32",
                                  peak_mem_bytes=mem, gbps=gbps, roofline_frac=gbps / roofline_peak_gbs(),
                                  dtype=dtype)


def _failed(n, splits, workers, dtype) -> str:
    return f"{n},{splits},{workers},,,,,failed,,,1,{dtype},"


def _exact_dft_at(x: np.ndarray, ks, chunk: int = 1 << 22) -> np.ndarray:
    """Direct O(N) sums in fp64 with the exact integer phase (k n) mod N."""
    n = x.shape[0]
    xc = x.astype(np.complex128)
    out = np.zeros(len(ks), dtype=np.complex128)
    for j, k in enumerate(ks):
        acc = 0j
        for s in range(0, n, chunk):
            idx = np.arange(s, min(n, s + chunk), dtype=np.int64)
            ph = (idx * int(k)) % n
            acc += np.sum(xc[s:s + len(idx)] * np.exp(-2j * np.pi * ph / n))
        out[j] = acc
    return out


def _full_spectrum(y: np.ndarray, dtype: str) -> np.ndarray:
    if dtype != "float32":
        return y.astype(np.complex128)
    from .core import PermSpectrum

    return PermSpectrum(y).to_full_complex()


def cmd_bench(n, splits, workers, repeats, dtype, device, test_mode=False) -> int:
    print(CSV_HEADER)
    try:
        print(_bench_row(n, splits, workers, dtype, repeats, device, test_mode).csv_row())
    except EfftError as exc:
        print(f"error: {exc}", file=sys.stderr)
        print(_failed(n, splits, workers, dtype))
        return 1
    return 0


def cmd_scan(n, splits_list, repeats, dtype, device, test_mode=False) -> int:
    """One bench row per splits value (the GPU planner is split-invariant; the
    reference's validation still applies per value)."""
    print(CSV_HEADER)
    rc = 0
    for s in splits_list:
        try:
            print(_bench_row(n, s, 1, dtype, repeats, device, test_mode).csv_row(), flush=True)
        except EfftError as exc:
            print(f"error: splits={s}: {exc}", file=sys.stderr)
            print(_failed(n, s, 1, dtype), flush=True)
            rc = 1
    return rc


def _roundtrip_error(y: np.ndarray, x: np.ndarray, dtype: str, device: int) -> float:
    """Inverse transform (scaled 1/N) of the forward result against the input."""
    plan = plan_create(len(x), 0, 1, test_mode=True, dtype=dtype, device=device, direction=1)
    with handle_create(plan) as h:
        h.data[:] = y
        z = np.array(h.run(), dtype=np.complex128)
    xd = x.astype(np.complex128)
    return float(np.linalg.norm(z - xd) / np.linalg.norm(xd))


def cmd_check(n, splits, spot_checks, dtype, device, test_mode=False, corrupt=False) -> int:
    """Accuracy row (reference cli.py:103-150).  float32 (the reference's own
    real-input path) keeps the reference contract exactly: full relative L2 up
    to 2^14 points (<= 5e-6), else the worst of `spot_checks` exact direct sums
    at coefficients in [0, n/2] (<= 1e-5); status ``failed`` and exit 1 on a
    miss.  Complex dtypes: full relative L2 against numpy's fp64 FFT up to
    2^24 points, spot checks above, with BASELINE.json's tolerances
    (1e-12 / 1e-5 x log2 N), plus the forward -> inverse round-trip error in
    the rt_err column.  ``--corrupt`` perturbs the result before the
    comparison (the reference's fault-injection hook, cli.py:125-126)."""
    try:
        plan = plan_create(n, splits, 1, test_mode=test_mode, dtype=dtype, device=device)
    except EfftError as exc:
        print(f"error: {exc}", file=sys.stderr)
        print(CSV_HEADER)
        print(_failed(n, splits, 1, dtype))
        return 1
    x = signal(n, dtype)
    with handle_create(plan) as h:
        h.data[:] = x
        import time

        t0 = time.perf_counter()
        y = np.array(h.run())
        wall = time.perf_counter() - t0
    rt = None if dtype == "float32" else _roundtrip_error(y, x, dtype, device)
    if corrupt:
        y = y.copy()
        y[0] += 1.0
    full = _full_spectrum(y, dtype)
    xd = x.astype(np.float64 if dtype == "float32" else np.complex128)
    limit = REF_FULL_CHECK_LIMIT if dtype == "float32" else FULL_CHECK_LIMIT
    if n <= limit:
        ref = np.fft.fft(xd)
        err = float(np.linalg.norm(full - ref) / np.linalg.norm(ref))
        tol = REF_L2_TOLERANCE if dtype == "float32" else (1e-12 if dtype == "complex128" else 1e-5) * math.log2(n)
    else:
        hi = n // 2 + 1 if dtype == "float32" else n
        rng = np.random.default_rng(DEFAULT_SEED + 1)
        ks = np.unique(np.concatenate([[0, 1, n // 2], rng.integers(0, hi, max(0, spot_checks - 3))]))
        ex = _exact_dft_at(xd, ks)
        scale = np.sqrt(np.mean(np.abs(ex) ** 2))
        err = float(np.max(np.abs(full[ks] - ex) / np.maximum(np.abs(ex), scale)))
        tol = REF_SPOT_TOLERANCE if dtype == "float32" else (1e-12 if dtype == "complex128" else 1e-5) * math.log2(n)
    ok = err <= tol
    m = RunMetrics.from_timing(n, splits, 1, wall, complex_input=dtype != "float32", l2=err,
                               status="ok" if ok else "failed", dtype=dtype, rt_err=rt)
    print(CSV_HEADER)
    print(m.csv_row())
    print(f"# check: error {err:.3e} vs tolerance {tol:.3e}", file=sys.stderr)
    if not ok:
        print(f"error: accuracy check failed, measured {err:.3e}", file=sys.stderr)
        return 1
    return 0


def _read_raw(path: str, n: int, dtype: str) -> np.ndarray:
    npdt = {"float32": "<f4", "complex64": "<c8", "complex128": "<c16"}[dtype]
    need = n * np.dtype(npdt).itemsize
    size = os.path.getsize(path)
    if size != need:
        kind = "short read" if size < need else "trailing data"
        raise ValueError(f"{path}: expected exactly {need} bytes, found {size} ({kind})")
    return np.fromfile(path, dtype=npdt, count=n)


def cmd_transform(input_path, output_path, n, splits, dtype, device, test_mode=False, device_bytes=0) -> int:
    """Raw little-endian file in, spectrum out (float32: packed PERM; complex: natural order).
    With --device-bytes (complex dtypes) the transform streams the host array
    through that much device memory (outofcore.py)."""
    import time

    try:
        x = _read_raw(input_path, n, dtype)
        if device_bytes and dtype != "float32":
            from . import outofcore

            t0 = time.perf_counter()
            y = outofcore.transform(x, device=device, device_bytes=device_bytes)
            wall = time.perf_counter() - t0
            y.tofile(output_path)
            print(CSV_HEADER)
            print(RunMetrics.from_timing(n, splits, 1, wall, dtype=dtype).csv_row())
            return 0
        plan = plan_create(n, splits, 1, test_mode=test_mode, dtype=dtype, device=device)
    except (OSError, ValueError, EfftError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1

    with handle_create(plan) as h:
        h.data[:] = x
        t0 = time.perf_counter()
        y = h.run()
        wall = time.perf_counter() - t0
        np.asarray(y).tofile(output_path)
    print(CSV_HEADER)
    print(RunMetrics.from_timing(n, splits, 1, wall, complex_input=dtype != "float32", dtype=dtype).csv_row())
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_1409_5757_b200",
                                 description="EFFT entry points on the B200 path")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p, repeats=False):
        p.add_argument("--size", required=True, help="transform size: 4096, 2^22 or 3x2^28")
        p.add_argument("--dtype", default="float32", choices=["float32", "complex64", "complex128"])
        p.add_argument("--device", type=int, default=0, help="CUDA device index")
        p.add_argument("--test-mode", action="store_true", help="relax the size rule (reference test_mode)")
        if repeats:
            p.add_argument("--repeats", type=int, default=DEFAULT_REPEATS)

    p = sub.add_parser("transform", help="transform a raw little-endian file")
    common(p)
    p.add_argument("--splits", type=int, required=True)
    p.add_argument("--input", required=True)
    p.add_argument("--output", required=True)
    p.add_argument("--device-bytes", type=int, default=0,
                   help="stream the array through this much device memory (complex dtypes; out of core)")
    p = sub.add_parser("scan", help="bench rows over a list of split counts")
    common(p, repeats=True)
    p.add_argument("--splits", required=True, help="comma-separated split counts")
    p = sub.add_parser("check", help="accuracy against an independent fp64 reference")
    common(p)
    p.add_argument("--splits", type=int, required=True)
    p.add_argument("--spot-checks", type=int, default=64)
    p.add_argument("--corrupt", action="store_true", help=argparse.SUPPRESS)
    p = sub.add_parser("bench", help="device time and throughput of one configuration")
    common(p, repeats=True)
    p.add_argument("--splits", type=int, required=True)
    p.add_argument("--workers", type=int, default=1, help="validated like the reference; no effect on the GPU")
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        n = parse_size(args.size)
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    if args.cmd == "transform":
        return cmd_transform(args.input, args.output, n, args.splits, args.dtype, args.device, args.test_mode,
                             args.device_bytes)
    if args.cmd == "scan":
        return cmd_scan(n, parse_int_list(args.splits), args.repeats, args.dtype, args.device, args.test_mode)
    if args.cmd == "check":
        return cmd_check(n, args.splits, args.spot_checks, args.dtype, args.device, args.test_mode, args.corrupt)
    return cmd_bench(n, args.splits, args.workers, args.repeats, args.dtype, args.device, args.test_mode)


if __name__ == "__main__":
    sys.exit(main())
