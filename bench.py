#!/usr/bin/env python
"""Benchmark: GFLOP/s (5*N*log2 N) and HBM GB/s of one large 1D FFT on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Default workload (BASELINE.json metric, north-star target config): C3, a forward
complex64 DFT of N = 2^30 (8 GiB), seeded N(0,1) synthetic input.  A "step" is one
transform (C2/C5: one forward + one inverse transform).  The input (8 GiB) is far
larger than the 126 MB L2, so no L2 flush is needed between steps; configs that fit
in L2 (C1) are timed per step with an L2 flush between steps.

Prints ONE JSON line (rank 0).  Keys beyond the base contract:
  roofline      dominant kernel (a pass kernel): algorithmic bytes per launch
                (2*N*sizeof(element): one read + one write of the array) over its
                average CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the CPU restatement of the reference algorithm (oracle/, float32
                arithmetic with the reference's twiddle recipe for c64 configs, fp64
                for c128) timed on the host cores on a bounded sample
  e2e           the same metric through the C-ABI host-buffer entry
                (efft_execute_host_batch): per transform pinned host in -> H2D ->
                passes -> D2H -> host out, with transform k+1's H2D overlapping
                transform k's passes and D2H (the two PCIe directions at once);
                forward+inverse configs run a forward batch then an inverse batch
  fp64          complex128 configs: the fp64 arithmetic rate (nominal 5NlogN and
                executed DADD+DMUL+2*DFMA from the committed ncu counts) against
                the measured DFMA peak (tools/dfma_peak.cu) -- 20 % of it: the
                passes are HBM bound, not fp64 bound
--impl reference times that CPU restatement (the reference itself is Python and
cannot travel to the GPU box) and prints the same line shape.
Multi-GPU (torchrun): ONE transform of the config's N, six-step sharded over the
ranks with NCCL all-to-alls (strong scaling; --replicas runs independent per-GPU
transforms instead); the time is the max over ranks.
"""
import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DTYPE_NAME = {"complex64": "f32", "complex128": "f64", "float32": "f32"}
# complex input: BASELINE.json's 5 N log2 N; real input: the reference's own 2.5 N log2 N
METRIC = {False: "GFLOP/s (5N*log2N) per 1D FFT", True: "GFLOP/s (2.5N*log2N, real input) per 1D FFT"}
ELEM = {"complex64": 8, "complex128": 16, "float32": 4}


def flops_of(cfg):
    """5 N log2 N for complex input (BASELINE.json), 2.5 N log2 N for real input
    (the reference's own model, bench.py:27-31)."""
    n = cfg["n"]
    return (2.5 if cfg["dtype"] == "float32" else 5.0) * n * math.log2(n)


def pass_alg_bytes(cfg):
    """One read + one write of the array a pass kernel transforms (real input:
    the N/2-point complex64 transform)."""
    n = cfg["n"]
    return 2 * (n // 2) * 8 if cfg["dtype"] == "float32" else 2 * n * ELEM[cfg["dtype"]]


def as_oracle_complex(x_np, cfg):
    """The complex array the oracle transforms: real input as complex."""
    import numpy as np

    if cfg["dtype"] == "float32":
        return x_np.astype(np.complex128)
    return x_np


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    NAMES = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device_index):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        s = sorted(self.samples)
        names = [v for k, v in self.NAMES.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(s)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, local, world


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_baseline(cfg_name, cfg, x_dev, max_seconds=25.0):
    """Time the oracle (CPU restatement of the reference algorithm) on a bounded
    sample; returns (cpu_baseline dict, oracle output or None).  The output is
    the oracle's float32 reference-recipe transform (c64) or fp64 transform
    (c128) of the WHOLE input when the sample is the whole input -- reused as
    the full-array parity comparator."""
    import numpy as np

    import oracle

    threads = oracle.host_threads()
    prec = "c128" if cfg["dtype"] == "complex128" else "c64"
    if cfg["dtype"] == "float32":
        return cpu_baseline_real(cfg_name, cfg, x_dev, threads, max_seconds)
    n_full = cfg["n"]
    # bounded sample: the largest power-of-two prefix (x 3 for C4) that runs in ~max_seconds
    m = 3 if n_full % 3 == 0 else 1
    n = min(n_full, m << 22)
    elem = 8 if prec == "c64" else 16
    host = x_dev[:n_full].cpu().numpy() if n_full * elem <= (16 << 30) else None
    best = None
    while True:
        if host is not None:
            x = host[:n] if n == n_full else np.ascontiguousarray(host[:n])
        else:
            x = x_dev[:n].cpu().numpy()
        t0 = time.perf_counter()
        out = oracle.transform(x, precision=prec, threads=threads)
        dt = time.perf_counter() - t0
        best = (n, dt)
        if n >= n_full or dt * 2.3 > max_seconds:
            break
        n *= 2
    n, dt = best
    gflops = 5.0 * n * math.log2(n) / dt / 1e9
    kind = ("float32 arithmetic with the reference's twiddle recipe" if prec == "c64"
            else "fp64 arithmetic")
    line = {"value": round(gflops, 3), "unit": "GFLOP/s", "cores": threads, "kind": "port",
            "sample": f"one {prec} transform of N={n} ({'the whole' if n == n_full else 'prefix of'} "
                      f"{cfg_name}'s N={n_full} input), {dt:.2f} s, oracle/efft_oracle.c "
                      f"({kind}) with {threads} OpenMP threads",
            "python_reference_context": PY_REFERENCE_CONTEXT}
    return line, (out if n == n_full else None), (host if n == n_full else None)


def cpu_baseline_real(cfg_name, cfg, x_dev, threads, max_seconds):
    """Real input: the oracle's float32 transform of the N/2-point complex
    packing x[2j] + i x[2j+1] -- the core of the reference's real algorithm
    (leaf_dft.py:93-125) -- on the largest prefix that runs in ~max_seconds."""
    import numpy as np

    import oracle

    n_full = cfg["n"]
    n = min(n_full, 1 << 22)
    best = None
    while True:
        xr = x_dev[:n].cpu().numpy()
        z = np.ascontiguousarray(xr[0::2] + 1j * xr[1::2]).astype(np.complex64)
        t0 = time.perf_counter()
        oracle.transform(z, precision="c64", threads=threads)
        dt = time.perf_counter() - t0
        best = (n, dt)
        if n >= n_full or dt * 2.3 > max_seconds:
            break
        n *= 2
    n, dt = best
    return {"value": round(2.5 * n * math.log2(n) / dt / 1e9, 3), "unit": "GFLOP/s", "cores": threads,
            "kind": "port",
            "sample": f"the oracle's float32 c64 transform of the N/2 = {n // 2} point complex packing of a "
                      f"{'whole' if n == n_full else 'prefix of the'} {cfg_name} real input ({dt:.2f} s, "
                      f"2.5 N log2 N), oracle/efft_oracle.c with {threads} OpenMP threads",
            "python_reference_context": PY_REFERENCE_CONTEXT}, None, None


# The reference package itself (Python, real float32 two-real composition) is
# not installable on the GPU box; its own numbers, measured in the build
# container, are kept beside the C restatement's.
PY_REFERENCE_CONTEXT = ("reference efft package (Python/numpy, real f32, two-real composition): "
                        "2.71 GFLOP/s at N=2^30, 2.70 at 2^27, 1.31 at 2^21 on 8 cores "
                        "(BASELINE.md section 2, build container)")


def rel_l2_chunked(a, b, chunk=1 << 26):
    """Relative L2 of a against b (numpy arrays), fp64 accumulation, bounded temporaries."""
    import numpy as np

    num = den = 0.0
    for i in range(0, a.shape[0], chunk):
        bb = b[i:i + chunk].astype(np.complex128)
        d = a[i:i + chunk].astype(np.complex128) - bb
        num += float(np.vdot(d, d).real)
        den += float(np.vdot(bb, bb).real)
    return math.sqrt(num / den)


def device_rel_l2(a, b, chunk=1 << 26):
    """Relative L2 of device tensors a against b, fp64 accumulation, chunked."""
    import torch

    num = den = 0.0
    for i in range(0, a.numel(), chunk):
        bb = torch.view_as_real(b[i:i + chunk]).double()
        d = torch.view_as_real(a[i:i + chunk]).double() - bb
        num += float(d.pow(2).sum())
        den += float(bb.pow(2).sum())
    return math.sqrt(num / den)


def parity_report_real(cfg, x, y):
    """Real input (PERM output): relative L2 over the packed slots against the
    fp64 restatement of the same input, the reference's own acceptance measure
    and tolerance (test_acceptance.py:33-51: <= 1e-6; oracle.py:115-127)."""
    import numpy as np

    import oracle

    n = cfg["n"]
    out = {"tolerance": 1e-6, "comparator": "oracle fp64 restatement, packed as the reference's PERM layout"}
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 0
    if avail < n * 48 + (8 << 30):
        out["rel_l2"] = None
        out["note"] = "host memory too small for the full-array comparator"
        return out
    xh = x.cpu().numpy()
    f = oracle.transform(xh.astype(np.complex128))
    packed = np.empty(n)
    packed[0], packed[1] = f[0].real, f[n // 2].real
    packed[2::2], packed[3::2] = f[1:n // 2].real, f[1:n // 2].imag
    del f
    yh = y.cpu().numpy().astype(np.float64)
    err = float(np.linalg.norm(yh - packed) / np.linalg.norm(packed))
    out["rel_l2"] = float(f"{err:.4e}")
    out["within_tolerance"] = err <= 1e-6
    return out


def parity_report(cfg, x, y, inv_plan, oracle_out, x_host, sid):
    """Full-array parity of the timed transform's output y = F(x) (north star:
    rel-L2 <= 1e-5 log2N (c64) / 1e-12 log2N (c128) against the reference CPU
    path on the same input, round-trip error reported)."""
    import numpy as np
    import torch

    import oracle

    n, dtype = cfg["n"], cfg["dtype"]
    if dtype == "float32":
        return parity_report_real(cfg, x, y)
    tol = (1e-5 if dtype == "complex64" else 1e-12) * math.log2(n)
    out = {"tolerance": tol}
    # forward -> inverse round trip on the device (the inverse plan scales by 1/N)
    if inv_plan is not None:
        z = torch.empty_like(x)
        inv_plan.execute(y.data_ptr(), z.data_ptr(), sid)
        torch.cuda.synchronize()
        out["rt_err"] = device_rel_l2(z, x)
        del z
    y_host = None
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 0
    elem = 8 if dtype == "complex64" else 16
    if oracle_out is not None:
        y_host = y.cpu().numpy()
        key = "rel_l2_vs_f32_reference_recipe" if dtype == "complex64" else "rel_l2"
        out[key] = rel_l2_chunked(y_host, oracle_out)
        out["comparator"] = ("oracle/efft_oracle.c float32 path (the reference's twiddle recipe, "
                             "recombine.py:49-59) on the whole input" if dtype == "complex64"
                             else "oracle/efft_oracle.c fp64 restatement on the whole input")
    if dtype == "complex64" and x_host is not None and avail > n * 40 + (8 << 30):
        # fp64 restatement of the same complex64 input: the ground truth
        t0 = time.perf_counter()
        exact = oracle.transform(x_host.astype(np.complex128), precision="c128")
        if y_host is None:
            y_host = y.cpu().numpy()
        out["rel_l2"] = rel_l2_chunked(y_host, exact)
        out["comparator_fp64"] = f"oracle fp64 restatement of the same input ({time.perf_counter() - t0:.1f} s)"
        del exact
    elif "rel_l2" not in out and oracle_out is None:
        out["rel_l2"] = None
        out["note"] = (f"full-array oracle skipped: {n * elem * 2 >> 30} GiB of host arrays "
                       f"(tests/test_gpu_parity.py checks this config by spots, Parseval and round trip)")
    ok = all(v is None or v <= (2 * tol if k == "rt_err" else tol)
             for k, v in out.items() if k.startswith("rel_l2") or k == "rt_err")
    out["within_tolerance"] = ok
    for k in list(out):
        if isinstance(out[k], float) and k != "tolerance":
            out[k] = float(f"{out[k]:.4e}")
    return out


def run_reference(args):
    """--impl reference: the CPU restatement of the reference path (oracle/,
    C + OpenMP on all host cores), rank 0 only, on the SAME config as our arm:
    each step is one transform (C2/C5: forward + inverse) of the config's full N
    on the same seeded input (generated on the GPU when one is present, as our
    arm does, then copied to the host outside the timed region)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    import oracle
    from paper_1409_5757_b200 import workloads

    cfg = workloads.CONFIGS[args.config]
    real = cfg["dtype"] == "float32"
    prec = "c128" if cfg["dtype"] == "complex128" else "c64"
    threads = oracle.host_threads()
    n = cfg["n"]
    elem = 8 if prec == "c64" else 16
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 1 << 62
    same = True
    if 2 * n * elem + (4 << 30) > avail:  # C5 (2 x 64 GiB) on a small host: largest pow2 prefix that fits
        same = False
        while 2 * n * elem + (4 << 30) > avail and n > (1 << 20):
            n //= 2
    seed = workloads.seed_for(args.config)
    try:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError
        x = workloads.make_input(cfg["n"], cfg["dtype"], cfg["kind"], seed)[:n].cpu().numpy()
        gen = "workloads.make_input (torch CUDA generator, same seed as our arm), copied to the host"
    except Exception:
        rng = np.random.default_rng(seed)
        x = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(
            np.complex64 if prec == "c64" else np.complex128)
        gen = "numpy default_rng(seed) N(0,1) (no GPU visible: same distribution, different values)"
    if real:  # the real transform's core: the N/2-point complex packing (leaf_dft.py:93-125)
        x = np.ascontiguousarray(x[0::2] + 1j * x[1::2]).astype(np.complex64)
    out = np.empty_like(x)
    per_step = 2 if cfg["roundtrip"] else 1
    for _ in range(args.warmup):
        oracle.transform(x, precision=prec, threads=threads, out=out)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for r in range(per_step):
            oracle.transform(x if r == 0 else out, direction=-1 if r == 0 else 1, precision=prec,
                             threads=threads, out=out if r == 0 else x)
    dt = time.perf_counter() - t0
    flops = (2.5 if real else 5.0) * n * math.log2(n) * per_step * args.steps
    gflops = flops / dt / 1e9
    what = (f"one c64 transform of the N/2 = {n // 2} point complex packing of the real input" if real else
            f"{per_step} {prec} transform(s) of N={n}") + ("" if same else f" (host RAM caps the full N={cfg['n']})")
    line = {
        "impl": "reference", "metric": METRIC[real],
        "value": round(gflops, 3), "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": DTYPE_NAME[cfg["dtype"]], "data": "synthetic",
        "config": {"workload": f"{args.config}: {'forward+inverse' if cfg['roundtrip'] else 'forward'} "
                               f"1D {cfg['dtype']} DFT, N={cfg['n']}",
                   "n": n, "same_config": same, "input": gen, "roundtrip": cfg["roundtrip"]},
        "cpu_baseline": {"value": round(gflops, 3), "unit": "GFLOP/s", "cores": threads,
                         "kind": "port",
                         "sample": f"each step = {what}; oracle/efft_oracle.c, the C restatement of the "
                                   f"reference EFFT algorithm ({'float32 with the reference twiddle recipe' if prec == 'c64' else 'fp64'}), "
                                   f"{threads} OpenMP threads (the reference is Python-only and cannot travel "
                                   f"to the GPU box)",
                         "python_reference_context": PY_REFERENCE_CONTEXT},
        "e2e": {"value": round(gflops, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_sharded(args, rank, local, world):
    """N > 1: ONE transform of the config's N, block-sharded over the ranks
    (six-step, 3 NCCL all-to-alls; paper_1409_5757_b200/sharded.py); strong scaling."""
    import torch

    from paper_1409_5757_b200 import sharded, workloads

    cfg = workloads.CONFIGS[args.config]
    n, dtype = cfg["n"], cfg["dtype"]
    shard = n // world
    x = workloads.make_input(shard, dtype, cfg["kind"], workloads.seed_for(args.config) * 1000 + rank)
    y = torch.empty_like(x)
    w = torch.empty_like(x)
    backend = sharded.GpuBackend(dtype, local)
    fwd = sharded.ShardedTransform(n, world, rank, -1, backend)
    inv = sharded.ShardedTransform(n, world, rank, 1, backend) if cfg["roundtrip"] else None
    per_step = 2 if inv else 1

    def step():
        fwd.execute(x, y, w)
        if inv is not None:
            inv.execute(y, x, w)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    total_ms = max_over_ranks(e0.elapsed_time(e1), world)
    barrier(world)
    ms_per_step = total_ms / args.steps
    value = per_step * 5.0 * n * math.log2(n) * args.steps / (total_ms * 1e-3) / 1e9
    elem = ELEM[dtype]
    exch = sharded.ShardedTransform.exchanged_bytes(n, world, elem)
    peak, peak_src = measured_peaks()
    # additive roofline of one sharded transform per rank: the local HBM passes
    # (2 FFT passes + pack + unpack) plus 3 all-to-alls over NVLink (770 GB/s
    # measured peer BW); the north-star minimum is 2 local passes
    hbm_bytes = sharded.ShardedTransform.local_passes() * 2 * shard * elem
    t_roof = hbm_bytes / (peak * 1e9) + exch / 770e9
    if rank == 0:
        line = {
            "metric": METRIC[cfg["dtype"] == "float32"],
            "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": DTYPE_NAME[dtype], "data": "synthetic (seeded torch generator, see workloads.py)",
            "config": {"workload": f"{args.config}: {'forward+inverse' if cfg['roundtrip'] else 'forward'} "
                                   f"1D {dtype} DFT, N={n}, six-step sharded over {world} GPUs",
                       "n": n, "input": cfg["kind"], "parallelism": f"six-step x{world} (NCCL all-to-all)",
                       "l2": "inputs larger than L2", "n1_n2": [fwd.n1, fwd.n2]},
            "roofline": {"bound": "hbm+nvlink", "achieved": round(per_step * t_roof / (ms_per_step * 1e-3), 4),
                         "peak": 1.0, "unit": "fraction of additive HBM+NVLink roofline",
                         "frac": round(per_step * t_roof / (ms_per_step * 1e-3), 4), "traffic": None,
                         "exchange_bytes_per_rank": exch, "t_roof_ms": round(t_roof * 1e3, 4),
                         "peak_source": peak_src + "; NVLink 770 GB/s measured peer copy (B200_PROFILING.md)"},
            "gpu_launches": None,
            "clocks": clocks.summary(),
            "e2e": None,
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    import torch.distributed as dist

    dist.destroy_process_group()


def run_ours(args):
    import torch

    import paper_1409_5757_b200 as efft
    from paper_1409_5757_b200 import _native, workloads

    rank, local, world = dist_init()
    if world > 1 and not args.replicas:
        return run_sharded(args, rank, local, world)
    torch.cuda.set_device(local)
    cfg = workloads.CONFIGS[args.config]
    n, dtype = cfg["n"], cfg["dtype"]
    seed = workloads.seed_for(args.config) + rank
    x = workloads.make_input(n, dtype, cfg["kind"], seed, device="cuda")
    y = torch.empty_like(x)
    ndt = {"complex64": _native.EFFT_C64, "complex128": _native.EFFT_C128, "float32": _native.EFFT_R32}[dtype]
    # the flags the drop-in handle uses (core.TransformHandle): the non-finite
    # input check of the reference's scatter (scatter.py:38-39) is timed too
    flags = _native.EFFT_FLAG_CHECK_FINITE
    fwd = _native.NativePlan(n, ndt, -1, local, flags)
    # (real input has no inverse entry: the reference's PERM path is forward only)
    inv = None if dtype == "float32" else _native.NativePlan(n, ndt, 1, local, flags | _native.EFFT_FLAG_SCALE_INVERSE)
    fwd.enable_timing(args.steps)  # per-launch events of every timed step (averaged)
    stream = torch.cuda.current_stream()
    sid = stream.cuda_stream
    per_step = 2 if cfg["roundtrip"] else 1
    l2_resident = n * ELEM[dtype] * 2 <= 96 << 20
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if l2_resident else None

    def step():
        fwd.execute(x.data_ptr(), y.data_ptr(), sid)
        if cfg["roundtrip"]:
            inv.execute(y.data_ptr(), x.data_ptr(), sid)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    launches = fwd.launches() + (inv.launches() if cfg["roundtrip"] else 0)
    fwd.enable_timing(args.steps)  # drop the warm-up executions
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        if flush is None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(args.steps):
                step()
                if i == args.steps - 1:
                    pass
            e1.record()
            torch.cuda.synchronize()
            total_ms = e0.elapsed_time(e1)
        else:
            total_ms = 0.0
            for _ in range(args.steps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                step()
                e1.record()
                torch.cuda.synchronize()
                total_ms += e0.elapsed_time(e1)
    warm = None
    cold_launch_ms = fwd.launch_times_ms()  # per-launch averages over the timed steps
    if flush is not None:
        # L2-resident size (SURVEY 7 hard part 7; reference bench.py:129-136 best-of):
        # also the warm time, steps back to back with the arrays left in L2
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        warm = e0.elapsed_time(e1) / args.steps
    torch.cuda.synchronize()
    barrier(world)
    total_ms = max_over_ranks(total_ms, world)
    ms_per_step = total_ms / args.steps
    flops_per_transform = flops_of(cfg)
    value = world * per_step * flops_per_transform * args.steps / (total_ms * 1e-3) / 1e9

    # dominant kernel roofline (pass kernels move 2*N*elem algorithmic bytes each)
    peak, peak_src = measured_peaks()
    # per-launch durations averaged over every timed step (events on the launching stream)
    avg = cold_launch_ms
    dom = max(range(len(avg)), key=lambda k: avg[k])
    alg_bytes = pass_alg_bytes(cfg)
    achieved = alg_bytes / (avg[dom] * 1e-3) / 1e9
    traffic = None  # DRAM bytes per launch of that kernel from the committed ncu capture
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh).get(args.config)
        if tr:
            traffic = tr["pass_bytes"][dom]
    except (OSError, ValueError, KeyError, IndexError):
        traffic = None
    whole_gbs = per_step * fwd.launches() * alg_bytes / (ms_per_step * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                "kernel": None, "pass_ms": [round(a, 4) for a in avg], "peak_source": peak_src,
                "alg_bytes_per_launch": alg_bytes}
    if warm is not None:
        # L2-resident (P_min = 1): the roofline of the whole transform is one
        # read + one write of the array; cold = L2 flushed before each step, warm = back to back
        t_alg = 2 * n * ELEM[dtype]
        roofline.update(achieved=round(t_alg / (ms_per_step * 1e-3) / 1e9, 1),
                        frac=round(t_alg / (ms_per_step * 1e-3) / 1e9 / peak, 4),
                        alg_bytes_per_launch=None, alg_bytes_per_transform=t_alg, p_min=1,
                        cold_ms=round(ms_per_step, 4), warm_ms=round(warm, 4),
                        warm_frac=round(t_alg / (warm * 1e-3) / 1e9 / peak, 4))
    desc = fwd.describe()
    kname = (("lean_pair" if dtype == "complex64" else "lean_pass") if "lean" in desc
             else "generic staged/direct pass")
    roofline["traffic"] = traffic
    roofline["kernel"] = (f"pass {dom} of {len(avg)} ({kname} kernel), {avg[dom]:.4f} ms avg over "
                          f"{args.steps} timed steps")
    fp64 = None  # complex128: fp64 arithmetic rate vs the measured DFMA peak
    if dtype == "complex128":
        try:
            with open(os.path.join(ROOT, "profiles", "fp64.json")) as fh:
                f64 = json.load(fh)
            ratio = f64.get(args.config, {}).get("executed_over_nominal")
            dpk = f64["dfma_peak"]["dfma_tflops"]
            nominal = value / 1e3
            fp64 = {"nominal_tflops": round(nominal, 3), "dfma_peak_tflops": dpk,
                    "executed_over_nominal": ratio,
                    "executed_tflops": round(nominal * ratio, 3) if ratio else None,
                    "frac": round(nominal * (ratio or 1.0) / dpk, 4),
                    "source": "profiles/fp64.json (ncu DADD+DMUL+2*DFMA counts; tools/dfma_peak.cu)"}
        except (OSError, ValueError, KeyError):
            fp64 = None

    # e2e through the C-ABI host-buffer entry (rank-local), fewer steps: PCIe bound
    e2e = None
    x_host = None
    if not args.no_e2e:
        hin = torch.empty(n, dtype=x.dtype, pin_memory=True)
        hout = torch.empty(n, dtype=x.dtype, pin_memory=True)
        hin.copy_(x)
        if 4 * n * ELEM[dtype] > torch.cuda.mem_get_info()[1] * 0.9:
            # C5: the host-buffer entry owns its own device in/out arrays; the
            # device-resident pair of the kernel timing must go first
            x_host = hin
            del x, y
            torch.cuda.empty_cache()
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        fwd.execute_host(hin.data_ptr(), hout.data_ptr(), sid)  # warm (allocates device buffers)
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        if not cfg["roundtrip"]:
            # pipelined: transform k+1's H2D overlaps transform k's passes + D2H
            fwd.execute_host_batch([hin.data_ptr()] * e2e_steps, [hout.data_ptr()] * e2e_steps, sid)
        else:
            # e2e_steps forward transforms, then e2e_steps inverse ones, each
            # batch pipelined like the forward-only configs (sequential inside
            # the library when two device pairs do not fit, as for C5)
            fwd.execute_host_batch([hin.data_ptr()] * e2e_steps, [hout.data_ptr()] * e2e_steps, sid)
            inv.execute_host_batch([hout.data_ptr()] * e2e_steps, [hin.data_ptr()] * e2e_steps, sid)
        dt = max_over_ranks(time.perf_counter() - t0, world)
        e2e = {"value": round(world * per_step * flops_per_transform * e2e_steps / dt / 1e9, 3),
               "unit": "GFLOP/s",
               "h2d_bytes_per_step": per_step * n * ELEM[dtype],
               "d2h_bytes_per_step": per_step * n * ELEM[dtype],
               "ms_per_step": round(dt / e2e_steps * 1e3, 3),
               "path": ("efft_execute_host_batch (C ABI): per transform pinned host -> H2D -> passes -> D2H "
                        "-> host, consecutive transforms overlapped (H2D of k+1 with D2H of k)") if not cfg["roundtrip"]
                       else ("efft_execute_host_batch (C ABI) of the forward plan, then of the inverse plan: "
                             "per transform pinned host -> H2D -> passes -> D2H -> host, overlapped")}
        del hin, hout

    cpu = None
    oracle_out = host_in = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu, oracle_out, host_in = cpu_baseline(args.config, cfg, x if x_host is None else x_host)
    parity = None
    if rank == 0 and not args.no_parity and x_host is None:
        if cfg["roundtrip"]:  # x was overwritten by the timed inverse: y = F(x) holds again
            fwd.execute(x.data_ptr(), y.data_ptr(), sid)
            torch.cuda.synchronize()
        parity = parity_report(cfg, x, y, inv, oracle_out, host_in, sid)
    del oracle_out, host_in

    if rank == 0:
        line = {
            "metric": METRIC[cfg["dtype"] == "float32"],
            "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": DTYPE_NAME[dtype], "data": "synthetic (seeded torch generator, see workloads.py)",
            "config": {"workload": f"{args.config}: {'forward+inverse' if cfg['roundtrip'] else 'forward'} "
                                   f"1D {dtype} DFT, N={n}",
                       "n": n, "input": cfg["kind"], "parallelism": f"replicas x{world}",
                       "l2": "flushed between steps (512 MiB write)" if flush is not None
                             else f"inputs ({n * ELEM[dtype] >> 20} MiB) larger than L2",
                       "plan": desc.strip().splitlines()},
            "hbm_gbs_whole_step": round(whole_gbs, 1),
            "roofline": roofline,
            "fp64": fp64,
            "gpu_launches": launches * args.steps,
            "clocks": clocks.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5", "r24", "r27", "r30"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-parity", action="store_true", help="skip the full-array parity leg")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent per-GPU transforms instead of one sharded transform")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: launch the ranks ourselves (the driver uses torchrun directly)
        import subprocess

        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", os.environ.get("MASTER_PORT", "29533"),
               os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
