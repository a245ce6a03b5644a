"""efft_execute_sharded (single-process six-step over G devices, C ABI) on ONE
B200 with G emulated ranks: the same device id G times, distinct buffers and
streams, the exchanges as pitched device copies.  Checked against the oracle
(the CPU restatement of the reference algorithm) on natural-order block
shards; a real multi-GPU box runs the same code with peer copies over NVLink."""
import math

import numpy as np
import pytest

import oracle
from conftest import random_c

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1409_5757_b200 import _native  # noqa: E402

NP = {"complex64": np.complex64, "complex128": np.complex128}
NDT = {"complex64": _native.EFFT_C64, "complex128": _native.EFFT_C128}


def tol(n, dtype):
    return (1e-12 if dtype == "complex128" else 1e-5) * math.log2(n)


def sharded(x, dtype, direction, G, devices=None):
    n = x.shape[0]
    plan = _native.ShardedPlan(n, NDT[dtype], direction, devices or [0] * G)
    shards = np.split(np.ascontiguousarray(x, dtype=NP[dtype]), G)
    d_in = [torch.from_numpy(s.copy()).cuda() for s in shards]
    d_out = [torch.empty_like(t) for t in d_in]
    streams = [torch.cuda.Stream() for _ in range(G)]
    plan.execute([t.data_ptr() for t in d_in], [t.data_ptr() for t in d_out], [s.cuda_stream for s in streams])
    torch.cuda.synchronize()
    # the input shards are preserved
    for s, t in zip(shards, d_in):
        assert np.array_equal(t.cpu().numpy(), s)
    return np.concatenate([t.cpu().numpy() for t in d_out]), plan


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_sharded_vs_oracle(dtype, G):
    n = 1 << 26 if dtype == "complex64" else 1 << 26
    x = random_c(n, seed=G + 7)
    y, plan = sharded(x, dtype, -1, G)
    exact = oracle.transform(x)
    assert oracle.rel_l2(y, exact) <= tol(n, dtype)
    z, _ = sharded(y, dtype, 1, G)
    assert oracle.rel_l2(z, x.astype(NP[dtype])) <= 2 * tol(n, dtype)
    n1, n2 = plan.split()
    assert n1 * n2 == n and n1 % G == 0 and n2 % G == 0


def test_sharded_radix3_family():
    n = 3 << 24
    x = random_c(n, seed=5)
    y, _ = sharded(x, "complex128", -1, 4)
    assert oracle.rel_l2(y, oracle.transform(x)) <= tol(n, "complex128")


def test_sharded_size_errors():
    with pytest.raises(Exception):
        _native.ShardedPlan(1 << 20, _native.EFFT_C64, -1, [0] * 3)  # G not a power of two
    with pytest.raises(Exception):
        _native.ShardedPlan(1 << 16, _native.EFFT_C64, -1, [0] * 8)  # too small to shard


@pytest.mark.parametrize("chunks", [1, 2, 4])
@pytest.mark.parametrize("dtype,G", [("complex64", 2), ("complex64", 4), ("complex128", 8)])
def test_sharded_overlapped_schedule_matches_sequential(dtype, G, chunks, monkeypatch):
    """EFFT_SHARD_CHUNKS: the local passes in column chunks with the exchanges of the
    neighbouring chunks on copy streams (the overlapped schedule) -- same result as the
    sequential schedule (chunks = 1) bit for bit, also when a plan is executed repeatedly
    (the next call's exchanges must not overtake the previous call's)."""
    n = 1 << 26
    x = random_c(n, seed=3 * G + chunks)
    monkeypatch.setenv("EFFT_SHARD_CHUNKS", "1")
    ref, _ = sharded(x, dtype, -1, G)
    assert oracle.rel_l2(ref, oracle.transform(x)) <= tol(n, dtype)
    monkeypatch.setenv("EFFT_SHARD_CHUNKS", str(chunks))
    plan = _native.ShardedPlan(n, NDT[dtype], -1, [0] * G)
    shards = np.split(np.ascontiguousarray(x, dtype=NP[dtype]), G)
    d_in = [torch.from_numpy(s.copy()).cuda() for s in shards]
    d_out = [torch.empty_like(t) for t in d_in]
    streams = [torch.cuda.Stream() for _ in range(G)]
    for rep in range(3):
        plan.execute([t.data_ptr() for t in d_in], [t.data_ptr() for t in d_out], [s.cuda_stream for s in streams])
    torch.cuda.synchronize()
    y = np.concatenate([t.cpu().numpy() for t in d_out])
    assert np.array_equal(y, ref)
    for s, t in zip(shards, d_in):
        assert np.array_equal(t.cpu().numpy(), s)
