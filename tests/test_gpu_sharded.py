"""Sharded six-step on ONE B200: G emulated ranks as host threads, each with its
own CUDA stream; the all-to-all is a host-barrier-synchronised copy between
the ranks' device buffers (no kernel ever waits on another kernel).  Exercises
the product's local steps -- column plans (staged/direct passes) and the
permutation kernels -- for G = 2, 4, 8; the NCCL exchange itself is covered by
tests/test_sharded.py over gloo."""
import threading

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1409_5757_b200 import sharded  # noqa: E402


class EmulatedExchange:
    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.src = [None] * world

    def a2a(self, rank, src, dst):
        torch.cuda.current_stream().synchronize()
        self.src[rank] = src
        self.bar.wait()
        c = src.numel() // self.world
        for q in range(self.world):
            dst[q * c:(q + 1) * c].copy_(self.src[q][rank * c:(rank + 1) * c])
        torch.cuda.current_stream().synchronize()
        self.bar.wait()


class EmulatedBackend(sharded.GpuBackend):
    def __init__(self, dtype, rank, exchange):
        super().__init__(dtype, 0)
        self.rank, self.exchange = rank, exchange

    def all_to_all(self, src, dst):
        self.exchange.a2a(self.rank, src, dst)


def run_emulated(x, world, dtype, direction):
    n = x.shape[0]
    shard = n // world
    tdt = torch.complex64 if dtype == "complex64" else torch.complex128
    xd = torch.from_numpy(x.astype(np.complex64 if dtype == "complex64" else np.complex128)).cuda()
    ex = EmulatedExchange(world)
    outs, errs = [None] * world, []

    def worker(rank):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                b = EmulatedBackend(dtype, rank, ex)
                t = sharded.ShardedTransform(n, world, rank, direction, b)
                xl = xd[rank * shard:(rank + 1) * shard].clone()
                yl = torch.empty(shard, dtype=tdt, device="cuda")
                w = torch.empty_like(yl)
                t.execute(xl, yl, w)
                s.synchronize()
                outs[rank] = yl.cpu().numpy()
        except Exception as exc:  # surfaced below
            errs.append(exc)
            ex.bar.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return np.concatenate(outs)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
@pytest.mark.parametrize("n", [1 << 20, 3 << 20, 1 << 24])
def test_sharded_emulated_matches_oracle(world, dtype, n):
    rng = np.random.default_rng(world + n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y = run_emulated(x, world, dtype, -1)
    lg = np.log2(n)
    tol = (1e-12 if dtype == "complex128" else 1e-5) * lg
    assert oracle.rel_l2(y, oracle.transform(x)) <= tol
    z = run_emulated(y, world, dtype, 1)
    assert oracle.rel_l2(z, x) <= 2 * tol
