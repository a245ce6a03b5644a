"""Out-of-core transform: one 1D DFT of a HOST array streamed through one GPU.

SURVEY.md section 8f row f3 (reference bench.py:115-126 reads binary32 only;
the paper's "enormous" N): when the array, its output and the
plan workspace do not fit in HBM, the four-step form runs over host memory
with bounded device buffers.  With N = N1 N2, x viewed as (N1 x N2) row-major
(n = n1 N2 + n2) and X[k1 + N1 k2]:

  step 1  for every block of C columns n2:  Yt[n2][k1] = sum_n1 x[n1][n2] W_N1^(n1 k1)
          (strided H2D of the block, a batched column plan, a device
          transpose, contiguous D2H into rows c0.. of Yt, which lives in `out`)
  step 2  for every block of Rr columns k1:  X[k1 + N1 k2] = sum_n2 Yt[n2][k1] W_N^(n2 k1) W_N2^(n2 k2)
          (strided H2D of the block, a column plan with the four-step
          twiddle on its input, strided D2H back into the same columns of
          `out`, now viewed as X[k2][k1])

The streaming runs natively (efft_execute_outofcore in efft_capi.cu): the
caller's arrays are page-locked for the call, every block moves by strided
DMA (no host-side reshuffle), step 1 writes Y transposed (Yt[n2][k1]) into the
output array and step 2 transforms it in place block by block, with two
streams and two device buffer sets so one block's copies overlap the other's.
Inverse = direction +1 with 1/N1 and 1/N2 scaling in the two column plans
(1/N in total).  Sizes N = M 2^t, M in {1, 3, 5, 7}, N1, N2 <= 2^17.
"""

import math

import numpy as np

from . import _native
from .errors import BinsizeNotPowerOfTwo

ELEM = {"complex64": 8, "complex128": 16}
LANES = {"complex64": 16, "complex128": 8}  # columns per 128-byte line (column-plan granularity)
MAX_COLUMN_LEN = 1 << 17


def split(n: int):
    """N = N1 * N2 as balanced as possible, N1 takes the odd factor M."""
    m, t = n, 0
    while m % 2 == 0:
        m //= 2
        t += 1
    if m not in (1, 3, 5, 7):
        raise BinsizeNotPowerOfTwo(f"n={n} is not M*2^t with M in {{1, 3, 5, 7}}")
    t1 = t // 2
    n1, n2 = m << t1, 1 << (t - t1)
    if n1 > MAX_COLUMN_LEN or n2 > MAX_COLUMN_LEN:
        raise BinsizeNotPowerOfTwo(f"n={n} exceeds the out-of-core range (N1, N2 <= 2^17)")
    return n1, n2


def plan_blocks(n: int, dtype: str, device_bytes: int):
    """Columns per step-1 block and rows per step-2 block for a device budget
    (mirror of efft_outofcore_blocks).

    Two streams each hold two device buffers of a block (in/out of the column
    plan or of the transpose).  Blocks are multiples of the 128-byte line width
    and divide the array dimension."""
    n1, n2 = split(n)
    e, f = ELEM[dtype], LANES[dtype]
    per = max(1, device_bytes // (4 * e))  # elements per buffer

    def fit(length, dim):
        b = max(f, min(dim, per // length))
        b -= b % f
        b = max(f, b)
        while dim % b:
            b -= f
        if b < f or dim % b:
            raise BinsizeNotPowerOfTwo(f"no block of {dim} columns fits {device_bytes} bytes")
        return b

    return n1, n2, fit(n1, n2), fit(n2, n1)


def transform(x: np.ndarray, direction: int = -1, device: int = 0, device_bytes: int = 1 << 30,
              out: np.ndarray = None) -> np.ndarray:
    """DFT of host array `x` (complex64 / complex128, natural order) with at most
    about `device_bytes` of device memory for the data blocks."""
    if x.dtype not in (np.complex64, np.complex128) or x.ndim != 1:
        raise ValueError("x must be a 1D complex64 or complex128 array")
    dtype = "complex64" if x.dtype == np.complex64 else "complex128"
    n = x.shape[0]
    plan_blocks(n, dtype, device_bytes)  # validates (same rule as the library)
    x = np.ascontiguousarray(x)
    res = out if out is not None else np.empty(n, dtype=x.dtype)
    if res.dtype != x.dtype or res.shape != (n,) or not res.flags.c_contiguous:
        raise ValueError("out must be a contiguous array like x")
    ndt = _native.EFFT_C64 if dtype == "complex64" else _native.EFFT_C128
    # non-finite input is rejected like the in-core handle (reference scatter.py:38-39)
    flags = _native.EFFT_FLAG_CHECK_FINITE | (_native.EFFT_FLAG_SCALE_INVERSE if direction == 1 else 0)
    _native.execute_outofcore(n, ndt, direction, device, flags, x.ctypes.data, res.ctypes.data, device_bytes)
    return res


def flops(n: int) -> float:
    return 5.0 * n * math.log2(n)
