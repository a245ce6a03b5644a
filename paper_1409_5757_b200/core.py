"""Plans, handles and the packed-spectrum contract, backed by the B200 library.

Mirrors the reference's public surface (reference pkg/src/efft/core.py):

* ``plan_create`` validates exactly like core.py:63-111 (ValueError,
  SplitsTooLarge, SizeConstraintViolation, BinsizeNotPowerOfTwo) and adds the
  keywords ``dtype`` ("float32" = the reference's real-input PERM layout,
  "complex64", "complex128"), ``direction`` (-1 forward unnormalised, +1
  inverse scaled by 1/N) and ``device``.  Complex plans accept n = M * 2^t with
  M in {1, 3, 5, 7} (the paper's M x 2^s sizes); the real path keeps
  the reference's power-of-two bin rule byte for byte.
* ``TransformHandle`` owns the device buffers (torch CUDA tensors), pinned host
  views ``data`` (writable, preserved across runs, core.py:146-149) and
  ``result`` (read-only, core.py:151-157), and one native plan
  (libefft_b200.so).  ``run()`` = H2D copy, the sm_100a passes, D2H copy.
  ``run_device()`` runs on the device tensors only (what the bench times).
* ``splits``, ``workers``, ``i_tile`` and ``k_tile`` are validated and kept on
  the plan for API compatibility; the GPU planner picks its own decomposition
  (outputs are split-invariant, reference test_recombine.py:154-163).
"""

from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import (
    BinsizeNotPowerOfTwo,
    IndexOutOfRange,
    SizeConstraintViolation,
    SizeMismatch,
    SplitsTooLarge,
)

DEFAULT_I_TILE = 16
DEFAULT_K_TILE = 64
SIZE_GRAIN_BITS = 8  # core.py:33-40
MIN_LEAF = 4

DTYPES = ("float32", "complex64", "complex128")


def _is_pow2(v: int) -> bool:
    return v > 0 and (v & (v - 1)) == 0


def _is_m_pow2(v: int) -> bool:
    """v = M * 2^k with M in {1, 3, 5, 7}."""
    if v < 1:
        return False
    while v % 2 == 0:
        v //= 2
    return v in (1, 3, 5, 7)


def build_scatter_index(splits: int) -> np.ndarray:
    """Bit-reversal permutation over `splits` bits (reference scatter.py:18-28)."""
    if splits < 0:
        raise ValueError("splits must be >= 0")
    idx = np.arange(1 << splits, dtype=np.int64)
    rev = np.zeros_like(idx)
    for _ in range(splits):
        rev = (rev << 1) | (idx & 1)
        idx >>= 1
    rev.setflags(write=False)
    return rev


@dataclass(frozen=True, eq=False)
class TransformPlan:
    n: int
    splits: int
    bins: int
    binsize: int
    scatter_index: np.ndarray = field(repr=False)
    i_tile: int
    k_tile: int
    workers: int
    test_mode: bool = False
    dtype: str = "float32"
    direction: int = -1
    device: int = 0

    def __repr__(self):
        return (
            f"TransformPlan(n={self.n}, splits={self.splits}, bins={self.bins}, "
            f"binsize={self.binsize}, i_tile={self.i_tile}, k_tile={self.k_tile}, "
            f"workers={self.workers}, test_mode={self.test_mode}, dtype={self.dtype!r}, "
            f"direction={self.direction}, device={self.device})"
        )


def plan_create(
    n: int,
    splits: int,
    workers: int = 1,
    *,
    test_mode: bool = False,
    i_tile: int = DEFAULT_I_TILE,
    k_tile: int = DEFAULT_K_TILE,
    dtype: str = "float32",
    direction: int = -1,
    device: int = 0,
) -> TransformPlan:
    """Validate a configuration (reference core.py:63-111 plus dtype/direction/device)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if splits < 0:
        raise ValueError("splits must be >= 0")
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if i_tile < 1 or k_tile < 1:
        raise ValueError("tile lengths must be >= 1")
    if dtype not in DTYPES:
        raise ValueError(f"dtype must be one of {DTYPES}, got {dtype!r}")
    if direction not in (-1, 1):
        raise ValueError("direction must be -1 (forward) or +1 (inverse)")
    if dtype == "float32" and direction != -1:
        raise ValueError("the real-input PERM path is forward only (reference SPEC.md:114)")
    if device < 0:
        raise ValueError("device must be >= 0")

    bins = 1 << splits
    if bins > n:
        raise SplitsTooLarge(f"2**{splits} bins exceed transform size {n}")
    if not test_mode and n % (1 << (splits + SIZE_GRAIN_BITS)) != 0:
        raise SizeConstraintViolation(
            f"n={n} is not a multiple of 2**{splits + SIZE_GRAIN_BITS}; "
            f"pass test_mode=True to relax (test sizes only)"
        )
    binsize = n // bins
    if dtype == "float32":
        if binsize * bins != n or not _is_pow2(binsize) or binsize < MIN_LEAF:
            raise BinsizeNotPowerOfTwo(
                f"bin size {n}/{bins} must be a power of two >= {MIN_LEAF} "
                f"for the real-input path"
            )
    else:
        if binsize * bins != n or not _is_m_pow2(binsize) or n < 2:
            raise BinsizeNotPowerOfTwo(
                f"bin size {n}/{bins} must be M*2^k with M in (1, 3, 5, 7) for complex transforms"
            )
    return TransformPlan(
        n=n, splits=splits, bins=bins, binsize=binsize,
        scatter_index=build_scatter_index(splits), i_tile=i_tile, k_tile=k_tile,
        workers=workers, test_mode=test_mode, dtype=dtype, direction=direction, device=device,
    )


def _torch():
    import torch

    return torch


class TransformHandle:
    """Device buffers, pinned host views and the native plan for one TransformPlan.

    Buffers are allocated on first use, each once for the handle's life: the
    pinned host pair by ``data`` / ``result`` / ``run()``, the device pair by
    ``run()`` / ``device_data`` / ``run_device()``.  A device-only user
    (``execute_tensors`` on its own tensors) never pays for the mirrors -- at
    C5 size each of the four arrays is 64 GiB."""

    def __init__(self, plan: TransformPlan):
        torch = _torch()
        self.plan = plan
        if not torch.cuda.is_available():
            raise RuntimeError("TransformHandle needs a CUDA device (there is no CPU fallback)")
        self._dev = torch.device("cuda", plan.device)
        if plan.dtype == "float32":
            native_dtype = _native.EFFT_R32
            self._tdt = torch.float32
        elif plan.dtype == "complex64":
            native_dtype, self._tdt = _native.EFFT_C64, torch.complex64
        else:
            native_dtype, self._tdt = _native.EFFT_C128, torch.complex128
        self._native = _native.NativePlan(plan.n, native_dtype, plan.direction, plan.device,
                                          _native.EFFT_FLAG_CHECK_FINITE)
        self._dev_in = self._dev_out = None
        self._host_in = self._host_out = None
        self._data = self._result = None
        self._closed = False

    def _alloc(self, what):
        torch = _torch()
        try:
            if what == "host" and self._host_in is None:
                # contents before the first run are undefined in the reference (core.py:155);
                # zero-filled here
                self._host_in = torch.zeros(self.plan.n, dtype=self._tdt, pin_memory=True)
                self._host_out = torch.zeros(self.plan.n, dtype=self._tdt, pin_memory=True)
                self._data = self._host_in.numpy()
                self._result = self._host_out.numpy().view()
                self._result.setflags(write=False)
            elif what == "device" and self._dev_in is None:
                self._dev_in = torch.zeros(self.plan.n, dtype=self._tdt, device=self._dev)
                self._dev_out = torch.zeros(self.plan.n, dtype=self._tdt, device=self._dev)
        except RuntimeError as exc:  # CUDA OOM / pinning failure
            from .errors import AllocationFailure

            raise AllocationFailure(str(exc)) from exc

    # -- reference surface -------------------------------------------------
    @property
    def data(self) -> np.ndarray:
        """Writable pinned host view of the input; preserved across transforms."""
        if self._data is None:
            self._check_open()
            self._alloc("host")
        return self._data

    @property
    def result(self) -> np.ndarray:
        """Read-only pinned host view of the output of the last ``run()``."""
        if self._result is None:
            self._check_open()
            self._alloc("host")
        return self._result

    def run(self) -> np.ndarray:
        """H2D copy of ``data``, the transform, D2H copy into ``result``."""
        self._check_open()
        self._alloc("host")
        self._alloc("device")
        torch = _torch()
        with torch.cuda.device(self.plan.device):
            stream = torch.cuda.current_stream()
            # read-and-clear: a flag left by run_device / execute_* on other data
            # must not reject this input
            self._native.nonfinite_seen(stream.cuda_stream)
            self._dev_in.copy_(self._host_in, non_blocking=True)
            self._native.execute(self._dev_in.data_ptr(), self._dev_out.data_ptr(),
                                 stream.cuda_stream)
            # the reference rejects the input before writing any output
            # (scatter.py:38-39): check before the copy-back, result untouched
            if self._native.nonfinite_seen(stream.cuda_stream):
                raise ValueError("input contains non-finite values")
            self._host_out.copy_(self._dev_out, non_blocking=True)
            stream.synchronize()
        return self._result

    def close(self) -> None:
        if getattr(self, "_closed", True):
            return
        self._closed = True
        self._native.close()
        self._dev_in = self._dev_out = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    # -- device-side surface (B200 extension) ---------------------------------
    @property
    def device_data(self):
        """Device input tensor (never written by a transform)."""
        self._check_open()
        self._alloc("device")
        return self._dev_in

    @property
    def device_result(self):
        """Device output tensor."""
        self._check_open()
        self._alloc("device")
        return self._dev_out

    def run_device(self, stream=None):
        """Enqueue the transform device_data -> device_result on `stream` (no copies, no sync)."""
        self._check_open()
        self._alloc("device")
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(self.plan.device)
        self._native.execute(self._dev_in.data_ptr(), self._dev_out.data_ptr(), s.cuda_stream)
        return self._dev_out

    def execute_tensors(self, src, dst, stream=None):
        """Transform caller-owned device tensors src -> dst (same length/dtype as the plan)."""
        self._check_open()
        torch = _torch()
        if src.numel() != self.plan.n or dst.numel() != self.plan.n:
            raise SizeMismatch(f"tensors must have {self.plan.n} elements")
        if src.dtype != self._tdt or dst.dtype != self._tdt:
            raise SizeMismatch("tensor dtype does not match the plan")
        if not (src.is_contiguous() and dst.is_contiguous()):
            raise SizeMismatch("tensors must be contiguous")
        s = stream if stream is not None else torch.cuda.current_stream(self.plan.device)
        self._native.execute(src.data_ptr(), dst.data_ptr(), s.cuda_stream)
        return dst

    def execute_host(self, h_in: np.ndarray, h_out: np.ndarray) -> np.ndarray:
        """The C-ABI host-buffer entry (efft_execute_host): H2D, passes, D2H, sync."""
        self._check_open()
        torch = _torch()
        if h_in.shape != (self.plan.n,) or h_out.shape != (self.plan.n,):
            raise SizeMismatch(f"host buffers must have length {self.plan.n}")
        want = np.dtype({"float32": np.float32, "complex64": np.complex64, "complex128": np.complex128}[
            self.plan.dtype])
        if h_in.dtype != want or h_out.dtype != want:
            raise SizeMismatch(f"host buffers must be {want} (the plan dtype)")
        if not (h_in.flags.c_contiguous and h_out.flags.c_contiguous):
            raise SizeMismatch("host buffers must be C-contiguous")
        if not h_out.flags.writeable:
            raise SizeMismatch("h_out must be writable")
        with torch.cuda.device(self.plan.device):
            s = torch.cuda.current_stream()
            self._native.execute_host(h_in.ctypes.data, h_out.ctypes.data, s.cuda_stream)
        return h_out

    def describe(self) -> str:
        return self._native.describe()

    def launches_per_run(self) -> int:
        return self._native.launches()

    def _check_open(self):
        if self._closed:
            raise ValueError("handle is closed")


def handle_create(plan: TransformPlan) -> TransformHandle:
    """Allocate device buffers and the native plan; reuse the handle for all runs."""
    return TransformHandle(plan)


def data_view(handle: TransformHandle) -> np.ndarray:
    return handle.data


def result_view(handle: TransformHandle) -> np.ndarray:
    return handle.result


def run_transform(handle: TransformHandle) -> np.ndarray:
    """Run the transform; the input is preserved (reference recombine.py:298-308)."""
    return handle.run()


class PermSpectrum:
    """View of a real-input spectrum in the packed layout of the reference
    (core.py:10-15, contract of core.py:199-249): slot 0 = F_0, slot 1 = F_{M/2},
    slots 2k, 2k+1 = Re, Im of F_k for 0 < k < M/2; the upper half follows from
    F_{M-k} = conj(F_k)."""

    def __init__(self, packed: np.ndarray):
        buf = np.asarray(packed)
        m = buf.shape[0] if buf.ndim == 1 else 0
        if m < 2 or m & 1:
            raise ValueError("packed spectrum must be 1-D with even length >= 2")
        self.packed = buf

    def __len__(self) -> int:
        return len(self.packed)

    @property
    def dc(self) -> float:
        return float(self.packed[0])

    @property
    def nyquist(self) -> float:
        return float(self.packed[1])

    def coefficient(self, k: int) -> complex:
        """F_k for any 0 <= k < M."""
        m = len(self.packed)
        if k < 0 or k >= m:
            raise IndexOutOfRange(f"coefficient index {k} outside [0, {m})")
        h = m // 2
        mirrored = k > h
        j = m - k if mirrored else k
        if j == 0:
            val = complex(self.packed[0])
        elif j == h:
            val = complex(self.packed[1])
        else:
            val = complex(float(self.packed[2 * j]), float(self.packed[2 * j + 1]))
        return val.conjugate() if mirrored else val

    def to_complex(self) -> np.ndarray:
        """F_0 .. F_{M/2} as complex128."""
        p = np.asarray(self.packed, dtype=np.float64)
        inner = p[2:].reshape(-1, 2)
        return np.concatenate(([p[0]], inner[:, 0] + 1j * inner[:, 1], [p[1]])).astype(np.complex128)

    def to_full_complex(self) -> np.ndarray:
        """All M coefficients, the upper half by conjugate symmetry."""
        lower = self.to_complex()
        return np.concatenate((lower, np.conj(lower[1:-1][::-1])))


def pack_perm(coeffs) -> np.ndarray:
    """Coefficients F_0 .. F_{M/2} of a real length-M input -> the packed layout
    [R_0, R_{M/2}, R_1, I_1, ..., R_{M/2-1}, I_{M/2-1}] (the reference's layout
    contract, core.py:10-15 / oracle.py:92-112); F_0 and F_{M/2} must be real."""
    from .errors import NotRealSpectrum

    f = np.asarray(coeffs, dtype=np.complex128)
    if f.ndim != 1 or f.shape[0] < 2:
        raise ValueError("need the coefficients k = 0 .. M/2 of an M >= 2 point real transform")
    m = 2 * (f.shape[0] - 1)
    tol = 1e-9 * max(float(np.linalg.norm(f)), 1.0)
    if abs(f[0].imag) > tol or abs(f[-1].imag) > tol:
        raise NotRealSpectrum("DC and Nyquist terms must be real")
    out = np.empty(m)
    out[0], out[1] = f[0].real, f[-1].real
    out[2::2], out[3::2] = f[1:-1].real, f[1:-1].imag
    return out


def l2_norm(computed, exact) -> float:
    """Relative L2 deviation of `computed` from `exact` over packed slots, in fp64
    (the reference's accuracy measure, oracle.py:115-127)."""
    from .errors import ZeroReference

    a = np.asarray(computed, dtype=np.float64)
    b = np.asarray(exact, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"length mismatch: {a.shape} vs {b.shape}")
    den = float(np.linalg.norm(b))
    if den == 0.0:
        raise ZeroReference("the comparator has zero norm")
    return float(np.linalg.norm(a - b)) / den

