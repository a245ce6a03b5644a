"""Out-of-core transform: one 1D DFT of a HOST array streamed through one GPU.

SURVEY.md section 8f row f3 (reference bench.py:115-126 reads binary32 only;
the paper's "enormous" N): when the array, its output and the
plan workspace do not fit in HBM, the four-step form runs over host memory
with bounded device buffers.  With N = N1 N2, x viewed as (N1 x N2) row-major
(n = n1 N2 + n2) and X[k1 + N1 k2]:

  step 1  for every block of C columns n2:  Y[k1][n2] = sum_n1 x[n1][n2] W_N1^(n1 k1)
          (gather the block, H2D, a batched column plan, D2H into Y)
  step 2  for every block of Rr rows k1:    X[k1 + N1 k2] = sum_n2 Y[k1][n2] W_N^(n2 k1) W_N2^(n2 k2)
          (contiguous rows H2D, device transpose, a column plan with the
          four-step twiddle on its input, D2H into X viewed as (N2 x N1))

Both steps use the library's column plans (efft_plan_create_columns) and the
permutation kernel (efft_permute_swap01); the host side only reshuffles
blocks.  Inverse = direction +1 with 1/N1 and 1/N2 scaling in the two column
plans (1/N in total).  Sizes N = M 2^t, M in {1, 3, 5, 7}, N1, N2 <= 2^17.
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
    """Columns per step-1 block and rows per step-2 block for a device budget.

    Each step holds two device buffers of its block (in/out of the column plan
    or of the transpose).  Blocks are multiples of the 128-byte line width and
    divide the array dimension."""
    n1, n2 = split(n)
    e, f = ELEM[dtype], LANES[dtype]
    per = max(1, device_bytes // (2 * e))  # elements per buffer

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
    import torch

    dtype = "complex64" if x.dtype == np.complex64 else "complex128"
    if x.dtype not in (np.complex64, np.complex128) or x.ndim != 1:
        raise ValueError("x must be a 1D complex64 or complex128 array")
    n = x.shape[0]
    n1, n2, cblk, rblk = plan_blocks(n, dtype, device_bytes)
    ndt = _native.EFFT_C64 if dtype == "complex64" else _native.EFFT_C128
    flags = _native.EFFT_FLAG_SCALE_INVERSE if direction == 1 else 0
    tdt = torch.complex64 if dtype == "complex64" else torch.complex128
    dev = torch.device("cuda", device)
    y = np.empty((n1, n2), dtype=x.dtype)  # host intermediate Y[k1][n2]
    res = out if out is not None else np.empty(n, dtype=x.dtype)
    x2 = x.reshape(n1, n2)
    xr = res.reshape(n2, n1)  # X[k1 + N1 k2] viewed as [k2][k1]
    with torch.cuda.device(device):
        s = torch.cuda.current_stream().cuda_stream
        a = torch.empty(max(n1 * cblk, n2 * rblk), dtype=tdt, device=dev)
        b = torch.empty_like(a)
        pin = torch.empty(a.numel(), dtype=tdt, pin_memory=True)
        pin_np = pin.numpy()
        # step 1: column DFTs of length N1 over blocks of C columns
        p1 = _native.NativePlan(n1, ndt, direction, device, flags, columns=(cblk, 0, 0))
        for c0 in range(0, n2, cblk):
            blk = pin_np[: n1 * cblk].reshape(n1, cblk)
            np.copyto(blk, x2[:, c0:c0 + cblk])
            a[: n1 * cblk].copy_(pin[: n1 * cblk], non_blocking=True)
            p1.execute(a.data_ptr(), a.data_ptr(), s)
            pin[: n1 * cblk].copy_(a[: n1 * cblk], non_blocking=True)
            torch.cuda.current_stream().synchronize()
            y[:, c0:c0 + cblk] = blk
        p1.close()
        # step 2: twiddle W_N^(n2 k1) + DFTs of length N2 over blocks of Rr rows k1
        for r0 in range(0, n1, rblk):
            p2 = _native.NativePlan(n2, ndt, direction, device, flags, columns=(rblk, n, r0))
            m = n2 * rblk
            np.copyto(pin_np[:m].reshape(rblk, n2), y[r0:r0 + rblk])
            a[:m].copy_(pin[:m], non_blocking=True)
            _native.permute_swap01(a.data_ptr(), b.data_ptr(), rblk, n2, 1, ELEM[dtype], s)  # -> [n2][r]
            p2.execute(b.data_ptr(), b.data_ptr(), s)  # -> [k2][r]
            pin[:m].copy_(b[:m], non_blocking=True)
            torch.cuda.current_stream().synchronize()
            xr[:, r0:r0 + rblk] = pin_np[:m].reshape(n2, rblk)
            p2.close()
    return res


def flops(n: int) -> float:
    return 5.0 * n * math.log2(n)
