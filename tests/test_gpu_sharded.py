"""Sharded six-step (one process per GPU path, sharded.py) on ONE B200: G
emulated ranks as host threads, each with its own CUDA stream; the all-to-all
is a host-barrier-synchronised copy between the ranks' device buffers (no
kernel ever waits on another kernel).  Exercises the product's local steps --
the shard-rank lean passes (efft_plan_create_shard_rank: pass 0 with the
blocked transposing store, pass 1 in place) and the pack / unpack kernels --
for G = 2, 4, 8; the NCCL exchange itself is covered by tests/test_sharded.py
over gloo and by test_nccl_two_gpus below when two GPUs are present."""
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
@pytest.mark.parametrize("dtype,n", [("complex64", 1 << 24), ("complex64", 3 << 24), ("complex128", 1 << 26),
                                     ("complex128", 3 << 24)])
def test_sharded_emulated_matches_oracle(world, dtype, n):
    rng = np.random.default_rng(world + n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y = run_emulated(x, world, dtype, -1)
    lg = np.log2(n)
    tol = (1e-12 if dtype == "complex128" else 1e-5) * lg
    assert oracle.rel_l2(y, oracle.transform(x)) <= tol
    z = run_emulated(y, world, dtype, 1)
    assert oracle.rel_l2(z, x) <= 2 * tol


def _nccl_worker(rank, world, port, n, q):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        rng = np.random.default_rng(11)
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        shard = n // world
        xl = torch.from_numpy(x[rank * shard:(rank + 1) * shard].astype(np.complex64)).cuda()
        yl, w = torch.empty_like(xl), torch.empty_like(xl)
        t = sharded.ShardedTransform(n, world, rank, -1, sharded.GpuBackend("complex64", rank))
        t.execute(xl, yl, w)
        torch.cuda.synchronize()
        q.put((rank, yl.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_nccl_two_gpus():
    """The NCCL data plane on 2 real GPUs against the oracle (skipped on 1-GPU boxes)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    n, world = 1 << 24, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_nccl_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    parts = dict(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    y = np.concatenate([parts[r] for r in range(world)])
    rng = np.random.default_rng(11)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    assert oracle.rel_l2(y, oracle.transform(x)) <= 1e-5 * 24
