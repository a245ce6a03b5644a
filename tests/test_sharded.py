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
    """Test stand-in for GpuBackend: numpy permutations, oracle pass, gloo all-to-all."""

    def column_plan(self, length, cols, direction, tw_mod, tw_offset, scale):
        return dict(length=length, cols=cols, direction=direction, tw_mod=tw_mod, tw_offset=tw_offset,
                    scale=scale)

    def run(self, plan, src, dst):
        a = src.numpy().copy()
        out = np.empty_like(a)
        oracle.pass_c128(a, out, length=plan["length"], cols=plan["cols"], batch=1, in_col=1,
                         in_stride=plan["cols"], in_batch=0, out_col=1, out_stride=plan["cols"],
                         out_batch=0, tw_mod=plan["tw_mod"], tw_base=plan["tw_offset"], tw_col=1,
                         direction=plan["direction"], threads=1)
        if plan["scale"]:
            out /= plan["length"]
        dst.numpy()[:] = out

    def swap01(self, src, dst, n0, n1, n2):
        dst.numpy()[:] = src.numpy().reshape(n0, n1, n2).transpose(1, 0, 2).reshape(-1)

    def swap12(self, src, dst, n0, n1, n2):
        dst.numpy()[:] = src.numpy().reshape(n0, n1, n2).transpose(0, 2, 1).reshape(-1)

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
    assert sharded.split_sizes(1 << 30, 8) == (1 << 15, 1 << 15)
    assert sharded.split_sizes(3 << 28, 8) == (3 << 14, 1 << 14)
    n1, n2 = sharded.split_sizes(1 << 32, 4)
    assert n1 * n2 == 1 << 32 and n1 % 4 == 0 and n2 % 4 == 0
    assert sharded.split_sizes(5 << 20, 2) == (5 << 10, 1 << 10)
    assert sharded.split_sizes(7 << 20, 2) == (7 << 10, 1 << 10)
    with pytest.raises(ValueError):
        sharded.split_sizes(9 << 20, 2)
    with pytest.raises(ValueError):
        sharded.split_sizes(1 << 20, 3)


def test_exchange_bytes_model():
    # C3 on 8 GPUs: 3 exchanges of 7/8 of a 1 GiB shard
    assert sharded.ShardedTransform.exchanged_bytes(1 << 30, 8, 8) == 3 * 7 * (1 << 27) * 8 // 8
