"""CPU oracle for the large-1D-FFT hot path -- TEST INFRASTRUCTURE ONLY.

A ctypes wrapper over ``oracle/efft_oracle.c``, the C restatement of the
reference EFFT algorithm (scatter.py / leaf_dft.py / recombine.py in complex
form, oracle.py's direct sum).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (cpu_baseline and ``--impl reference``) import this module,
as the checker or the timed CPU baseline.  The product package
``paper_1409_5757_b200`` never imports it.

Parity status: pinned -- see tests/test_oracle.py (reference KATs and golden
fixtures generated from the reference package by tests/golden/make_golden.py).
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libefft_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the restatement with gcc (make) into oracle/_build/."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "efft_oracle.c"))
    ):
        subprocess.run(["make", "-C", _HERE], check=True, stdout=subprocess.DEVNULL)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        lib.efo_transform_c128.argtypes = [i64, i32, vp, vp, i32, i32]
        lib.efo_transform_c128.restype = i32
        lib.efo_transform_c64.argtypes = [i64, i32, vp, vp, i32, i32]
        lib.efo_transform_c64.restype = i32
        lib.efo_dft_at_many.argtypes = [i64, vp, vp, i64, i32, vp, i32]
        lib.efo_dft_at_many.restype = None
        lib.efo_bitrev.argtypes = [i64, i32]
        lib.efo_bitrev.restype = i64
        lib.efo_pass_c128.argtypes = [vp, vp] + [i64] * 13 + [i32, i32]
        lib.efo_pass_c128.restype = i32
        _lib = lib
    return _lib


def host_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def default_splits(n: int, leaf_log2: int = 16) -> int:
    """Bins of ~2^16 elements keep each leaf in cache (the paper's tuning rule)."""
    t = (n & -n).bit_length() - 1
    return max(0, t - leaf_log2)


def transform(x, direction: int = -1, splits=None, precision: str = "c128", threads=None,
              out=None) -> np.ndarray:
    """Restated EFFT of complex x (forward unnormalised; inverse scaled 1/N)."""
    lib = _load()
    if precision == "c128":
        x = np.ascontiguousarray(x, dtype=np.complex128)
        fn = lib.efo_transform_c128
    elif precision == "c64":
        x = np.ascontiguousarray(x, dtype=np.complex64)
        fn = lib.efo_transform_c64
    else:
        raise ValueError(precision)
    n = x.shape[0]
    if out is None:
        out = np.empty_like(x)
    s = default_splits(n) if splits is None else splits
    rc = fn(n, s, x.ctypes.data, out.ctypes.data, direction, threads or host_threads())
    if rc != 0:
        raise ValueError(f"oracle transform failed rc={rc} (n={n}, splits={s})")
    return out


def dft_at(x, ks, direction: int = -1, threads=None) -> np.ndarray:
    """Direct O(N) coefficients X_k (oracle.py:79-89 for complex input)."""
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.complex128)
    ks = np.ascontiguousarray(np.atleast_1d(ks), dtype=np.int64)
    out = np.empty(ks.shape[0], dtype=np.complex128)
    lib.efo_dft_at_many(x.shape[0], x.ctypes.data, ks.ctypes.data, ks.shape[0], direction,
                        out.ctypes.data, threads or host_threads())
    return out


def pass_c128(inp, out, *, length, cols, batch, in_col, in_stride, in_batch, out_col,
              out_stride, out_batch, tw_mod=0, tw_base=0, tw_col=0, tw_batch=0,
              direction=-1, threads=None):
    """CPU mirror of the device sub-FFT pass contract (see efft_oracle.c)."""
    lib = _load()
    assert inp.dtype == np.complex128 and out.dtype == np.complex128
    rc = lib.efo_pass_c128(inp.ctypes.data, out.ctypes.data, length, cols, batch, in_col,
                           in_stride, in_batch, out_col, out_stride, out_batch, tw_mod,
                           tw_base, tw_col, tw_batch, direction, threads or host_threads())
    if rc != 0:
        raise ValueError(f"oracle pass failed rc={rc}")
    return out


def bitrev(j: int, bits: int) -> int:
    return int(_load().efo_bitrev(j, bits))


def rel_l2(computed, exact) -> float:
    """Relative L2 deviation (oracle.py:115-127, complex form)."""
    a = np.asarray(computed, dtype=np.complex128)
    b = np.asarray(exact, dtype=np.complex128)
    den = np.sqrt(np.sum(np.abs(b) ** 2))
    return float(np.sqrt(np.sum(np.abs(a - b) ** 2)) / den)
