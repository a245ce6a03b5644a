"""Out-of-core transform (outofcore.py) on a B200: host-streamed four-step vs the oracle."""
import math

import numpy as np
import pytest

import oracle
from conftest import random_c

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1409_5757_b200 import outofcore  # noqa: E402


def tol(n, dtype):
    return (1e-12 if dtype == np.complex128 else 1e-5) * math.log2(n)


@pytest.mark.parametrize("n,dtype,budget", [(1 << 22, np.complex128, 1 << 20), (3 << 20, np.complex64, 1 << 19),
                                            (1 << 23, np.complex64, 1 << 21)])
def test_out_of_core_vs_oracle_and_roundtrip(n, dtype, budget):
    x = random_c(n, seed=n % 997).astype(dtype)
    n1, n2, cb, rb = outofcore.plan_blocks(n, "complex64" if dtype == np.complex64 else "complex128", budget)
    assert cb < n2 and rb < n1  # really streamed in several blocks per step
    y = outofcore.transform(x, device_bytes=budget)
    assert oracle.rel_l2(y, oracle.transform(x.astype(np.complex128))) <= tol(n, dtype)
    z = outofcore.transform(y, direction=1, device_bytes=budget)
    assert oracle.rel_l2(z, x) <= 2 * tol(n, dtype)


def test_out_of_core_matches_in_hbm_transform_at_2p28():
    """Same result as the in-HBM (lean) transform at a size whose blocks are 32x smaller than the array."""
    from paper_1409_5757_b200 import _native

    n = 1 << 28
    g = torch.Generator(device="cuda").manual_seed(28)
    xd = torch.randn(n, dtype=torch.complex64, device="cuda", generator=g)
    yd = torch.empty_like(xd)
    p = _native.NativePlan(n, _native.EFFT_C64, -1, 0)
    p.execute(xd.data_ptr(), yd.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    x = xd.cpu().numpy()
    ref = yd.cpu().numpy()
    del xd, yd
    torch.cuda.empty_cache()
    y = outofcore.transform(x, device_bytes=n * 8 // 16)
    err = float(np.linalg.norm(y.astype(np.complex128) - ref) / np.linalg.norm(ref.astype(np.complex128)))
    assert err <= 2 * tol(n, np.complex64)


def test_out_of_core_caller_pinned_buffers_and_out_argument():
    """Buffers the caller already page-locked (cudaHostRegister reports them as
    registered) are used as they are and stay pinned; `out` is written in place."""
    n = 3 << 20
    x = torch.from_numpy(random_c(n, seed=5).astype(np.complex64)).pin_memory()
    o = torch.empty(n, dtype=torch.complex64).pin_memory()
    y = outofcore.transform(x.numpy(), device_bytes=1 << 20, out=o.numpy())
    assert y.ctypes.data == o.data_ptr()
    assert oracle.rel_l2(y, oracle.transform(x.numpy().astype(np.complex128))) <= tol(n, np.complex64)
    assert x.is_pinned() and o.is_pinned()


def test_out_of_core_rejects_overlap():
    x = random_c(1 << 20, seed=1).astype(np.complex64)
    with pytest.raises(ValueError, match="overlap"):  # EFFT_ERR_INVALID_ARG
        outofcore.transform(x, out=x)


def test_out_of_core_read_only_mapped_input(tmp_path):
    """The input may be a read-only file mapping (the reference reads binary arrays from disk)."""
    n = 1 << 20
    x = random_c(n, seed=9).astype(np.complex64)
    f = tmp_path / "x.c64"
    x.tofile(f)
    xm = np.memmap(f, dtype=np.complex64, mode="r", shape=(n,))
    y = outofcore.transform(xm, device_bytes=1 << 20)
    assert oracle.rel_l2(y, oracle.transform(x.astype(np.complex128))) <= tol(n, np.complex64)
