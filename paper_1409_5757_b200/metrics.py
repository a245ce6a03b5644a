"""FLOP model, roofline and run metrics (reference bench.py:27-73, extended).

The reference reports 2.5*n*log2(n) for its real transform (bench.py:27-31);
complex transforms use the conventional 5*N*log2(N) of BASELINE.json.  The HBM
roofline of one transform is ``passes * 2 * N * sizeof(element)`` bytes.
"""

import math
from dataclasses import dataclass
from typing import Optional

from .errors import MissingBaseline, NonPositiveSize

CSV_HEADER = "size,splits,workers,runtime_s,gflops,l2,mem_bytes,status,gbps,roofline_frac,ngpus,dtype,rt_err"


def flops_model(n: int, complex_input: bool = False) -> float:
    """2.5*n*log2(n) for real input (reference), 5*n*log2(n) for complex."""
    if n <= 0:
        raise NonPositiveSize(f"transform size must be positive, got {n}")
    return (5.0 if complex_input else 2.5) * n * math.log2(n)


def efficiency(perf_by_workers: dict) -> dict:
    """Parallel efficiency P(T) / (T * P(1)) per worker count T (the reference's
    definition, bench.py:34-39; on the GPU the worker count has no effect)."""
    base = perf_by_workers.get(1)
    if base is None or not base > 0:
        raise MissingBaseline("need a positive single-worker performance P(1)")
    return {workers: perf / (workers * base) for workers, perf in perf_by_workers.items()}


def algorithmic_bytes(n: int, elem_bytes: int, passes: int) -> int:
    """Bytes one transform must move through HBM: each pass reads and writes N elements."""
    return passes * 2 * n * elem_bytes


@dataclass
class RunMetrics:
    n: int
    splits: int
    workers: int
    wall_seconds: float
    gflops: float
    l2: Optional[float] = None
    peak_mem_bytes: Optional[int] = None
    status: str = "ok"
    gbps: Optional[float] = None
    roofline_frac: Optional[float] = None
    ngpus: int = 1
    dtype: str = "complex64"
    rt_err: Optional[float] = None  # forward -> inverse round-trip relative L2 (north star)

    @classmethod
    def from_timing(cls, n, splits, workers, wall_seconds, complex_input=True, **kw):
        if not wall_seconds > 0:
            raise ValueError("wall time must be positive")
        gflops = flops_model(n, complex_input) / wall_seconds / 1e9
        return cls(n, splits, workers, wall_seconds, gflops, **kw)

    def csv_row(self) -> str:
        f = lambda v, fmt: "" if v is None else format(v, fmt)  # noqa: E731
        return (f"{self.n},{self.splits},{self.workers},{self.wall_seconds:.6e},{self.gflops:.6g},"
                f"{f(self.l2, '.6e')},{f(self.peak_mem_bytes, 'd')},{self.status},"
                f"{f(self.gbps, '.6g')},{f(self.roofline_frac, '.4f')},{self.ngpus},{self.dtype},"
                f"{f(self.rt_err, '.6e')}")
