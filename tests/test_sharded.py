"""Host logic of the six-step sharded transform (paper_1409_5757_b200/sharded.py)
on CPU: world_size 2 and 4 over gloo, local steps through the oracle's pass
primitive (test backend), checked against the oracle transform."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1409_5757_b200 import sharded


class CpuBackend:
    """Test stand-in for GpuBackend: numpy passes with the same contract as the
    shard-rank plan (efft_execute_shard_pass), numpy permutations, gloo all-to-all."""

    def split(self, n, world):
        # any N1 x N2 works for the numpy passes; small test sizes use a balanced split
        m, t = sharded._factor(n)
        t1 = t // 2
        return m << t1, 1 << (t - t1)

    def shard_plan(self, n, world, rank, direction, n1, n2):
        return dict(n=n, world=world, rank=rank, direction=direction, n1=n1, n2=n2)

    def pass0(self, plan, src, dst):
        n, G, p, d, n1, n2 = (plan[k] for k in ("n", "world", "rank", "direction", "n1", "n2"))
        l1, l2 = n1 // G, n2 // G
        b = src.numpy().reshape(n1, l2)
        y = np.fft.fft(b, axis=0) if d == -1 else np.fft.ifft(b, axis=0) * n1
        k1 = np.arange(n1)[:, None]
        c = (p * l2 + np.arange(l2))[None, :]
        y = y * np.exp(d * 2j * np.pi * ((c * k1) % n) / n)  # W_N^(n2 k1)
        # blocked by destination rank: [q][c][k1']
        dst.numpy()[:] = y.reshape(G, l1, l2).transpose(0, 2, 1).reshape(-1)

    def pass1(self, plan, buf):
        n, G, d, n1, n2 = (plan[k] for k in ("n", "world", "direction", "n1", "n2"))
        t = buf.numpy().reshape(n2, n1 // G)
        x = np.fft.fft(t, axis=0) if d == -1 else np.fft.ifft(t, axis=0) / n1
        buf.numpy()[:] = x.reshape(-1)

    def swap01(self, src, dst, n0, n1, n2):
        dst.numpy()[:] = src.numpy().reshape(n0, n1, n2).transpose(1, 0, 2).reshape(-1)

    def all_to_all(self, src, dst):
        # gloo has no complex all_to_all: exchange the float64 view
        dist.all_to_all_single(torch.view_as_real(dst), torch.view_as_real(src))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, direction, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(99)
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        shard = n // world
        xl = torch.from_numpy(x[rank * shard:(rank + 1) * shard].copy())
        yl = torch.zeros_like(xl)
        work = torch.zeros_like(xl)
        t = sharded.ShardedTransform(n, world, rank, direction, CpuBackend())
        t.execute(xl, yl, work)
        assert np.array_equal(xl.numpy(), x[rank * shard:(rank + 1) * shard])  # input preserved
        q.put((rank, yl.numpy().copy()))
    finally:
        dist.destroy_process_group()


def _run(world, n, direction):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, direction, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return np.concatenate([parts[r] for r in range(world)])


@pytest.mark.parametrize("world,n", [(2, 1024), (2, 3 * 1024), (4, 4096)])
@pytest.mark.parametrize("direction", [-1, 1])
def test_sharded_matches_oracle(world, n, direction):
    rng = np.random.default_rng(99)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y = _run(world, n, direction)
    assert oracle.rel_l2(y, oracle.transform(x, direction=direction)) < 1e-13


def test_split_sizes():
    """the Python mirror of lean.cu split_sharded (the GPU test checks the two agree)"""
    assert sharded.split_sizes(1 << 30, 8) == (1 << 15, 1 << 15)
    assert sharded.split_sizes(1 << 32, 8, "complex128") == (1 << 16, 1 << 16)
    assert sharded.split_sizes(3 << 28, 8, "complex128") == (1 << 15, 3 << 13)
    assert sharded.split_sizes(1 << 27, 4, "complex128") == (1 << 14, 1 << 13)
    assert sharded.split_sizes(5 << 24, 2) == (1 << 14, 5 << 10)
    with pytest.raises(ValueError):
        sharded.split_sizes(9 << 20, 2)
    with pytest.raises(ValueError):
        sharded.split_sizes(1 << 30, 3)
    with pytest.raises(ValueError):
        sharded.split_sizes(1 << 20, 2)  # below the pass range


def test_exchange_bytes_model():
    # C3 on 8 GPUs: 3 exchanges of 7/8 of a 1 GiB shard
    assert sharded.ShardedTransform.exchanged_bytes(1 << 30, 8, 8) == 3 * 7 * (1 << 27) * 8 // 8
