"""Six-step sharded transform, one process per GPU: one N-point DFT
block-distributed over G ranks, the exchanges as NCCL all-to-alls.

Layout contract (natural-order block shards): rank p holds input elements
x[p*N/G, (p+1)*N/G) and receives output coefficients X[p*N/G, (p+1)*N/G).
The reference has no distributed path (it is one shared-memory process whose
only parallelism is the fork-join of parallel.py:34-98 / recombine.py:263-295);
this is the B200 extension BASELINE.json asks for.

With N = N1*N2, n = n1*N2 + n2 and k = k1 + N1*k2,

    X[k1 + N1 k2] = sum_n2 W_N2^(n2 k2) W_N^(n2 k1) sum_n1 x[n1 N2 + n2] W_N1^(n1 k1)

Per rank p (L1 = N1/G, L2 = N2/G), buffers x (input, preserved), y, w:
  1. pack   w[q][r][c] = x_p[r][q*L2 + c]                 (swap01, local)
  2. a2a    y = B[n1 = p'*L1 + r][c], the rank's L2 columns, all n1
  3. pass 0 w = Y[q][c][k1'] = DFT_N1(B[:, c])[q*L1 + k1'] * W_N^((p*L2 + c) k1)
            -- the lean transposing pass (lean.cu) with the four-step twiddle
            fused and its store blocked by destination rank: the send buffer
  4. a2a    y = T[n2 = q*L2 + c][k1']                     (N2 x L1)
  5. pass 1 y = X[k2][k1'] = DFT_N2(T[:, k1']) in place    (the lean in-place pass)
  6. a2a    w = V[q][k2'][k1'] = X_q[p*L2 + k2'][k1']
  7. unpack y_p[k2'][q][k1'] = V[q][k2'][k1']               (swap01) -> natural order
Three all-to-all exchanges (k = 3 in SURVEY section 8e) and four local HBM
passes: two FFT passes plus the pack and unpack the contiguous-chunk NCCL
all-to-all needs (the transposes between the passes are fused into pass 0's
store).  The single-process C entry efft_execute_sharded does the same with
pitched peer copies instead and needs only the two FFT passes.

The compute steps go through a backend: `GpuBackend` (libefft_b200.so
shard-rank plan + permutation kernels, NCCL all-to-all via torch.distributed)
is the product path; tests substitute a CPU backend (numpy) and run the
exchange over gloo (tests/test_sharded.py).
"""

import math

from .errors import BinsizeNotPowerOfTwo

F_LANES = {"complex64": 16, "complex128": 8}


def _factor(n):
    m, t = n, 0
    while m > 0 and m % 2 == 0:
        m //= 2
        t += 1
    return m, t


def split_sizes(n: int, world: int, dtype: str = "complex64"):
    """N = N1 * N2 of the lean passes (lean.cu split_sharded, mirrored): N1 = 256 RB1,
    N2 = RA2 RB2 (RA2 = 256 / 192 / 160 / 224 for M = 1 / 3 / 5 / 7), G*F | N1, N2."""
    m, t = _factor(n)
    if m not in (1, 3, 5, 7) or world < 1 or world & (world - 1):
        raise BinsizeNotPowerOfTwo(f"n={n} / world={world} not shardable (need n = M*2^t with M in {{1, 3, 5, 7}}, "
                                   f"G = 2^g)")
    ra2 = {1: 256, 3: 192, 5: 160, 7: 224}[m]
    lbs = t - 16 if m == 1 else t - 14 if m == 3 else t - 13
    lb1 = (lbs + 1) // 2
    lb2 = lbs - lb1
    lbmin = 4 if (dtype == "complex64" and m == 1) else 5
    if not (lbmin <= lb1 <= 8 and lbmin <= lb2 <= 8):
        raise BinsizeNotPowerOfTwo(f"n={n} is outside the sharded pass range")
    n1, n2 = 256 << lb1, ra2 << lb2
    f = F_LANES[dtype]
    if n1 % (world * f) or n2 % (world * f):
        raise BinsizeNotPowerOfTwo(f"n={n} too small for {world} shards")
    return n1, n2


class ShardedTransform:
    """Forward (-1) or inverse (+1, scaled 1/N) DFT of a block-sharded array."""

    def __init__(self, n: int, world: int, rank: int, direction: int, backend):
        self.n, self.world, self.rank, self.direction = n, world, rank, direction
        self.backend = backend
        self.n1, self.n2 = backend.split(n, world)
        self.l1, self.l2 = self.n1 // world, self.n2 // world
        self.plan = backend.shard_plan(n, world, rank, direction, self.n1, self.n2)

    def execute(self, x_local, y_local, work):
        """x_local, y_local, work: N/G-element device (or host) buffers; x_local preserved."""
        b, G, L1, L2 = self.backend, self.world, self.l1, self.l2
        b.swap01(x_local, work, L1, G, L2)   # [q][r][c]
        b.all_to_all(work, y_local)          # B[n1][c]
        b.pass0(self.plan, y_local, work)    # Y[q][c][k1'] (send buffer)
        b.all_to_all(work, y_local)          # T[n2][k1']
        b.pass1(self.plan, y_local)          # X[k2][k1'], in place
        b.all_to_all(y_local, work)          # V[q][k2'][k1']
        b.swap01(work, y_local, G, L2, L1)   # y[k2'][q][k1']
        return y_local

    @staticmethod
    def exchanged_bytes(n: int, world: int, elem: int) -> int:
        """Bytes one rank sends per transform: 3 exchanges of (G-1)/G of its N/G elements."""
        return 3 * (world - 1) * (n // world) * elem // world

    @staticmethod
    def local_passes() -> int:
        """HBM passes per rank per transform: pack, two FFT passes, unpack."""
        return 4


class GpuBackend:
    """Product path: libefft_b200.so shard-rank plan (the lean pass kernels) +
    permutation kernels, NCCL all-to-all."""

    def __init__(self, dtype: str, device: int, group=None):
        import torch

        from . import _native

        self.torch = torch
        self.native = _native
        self.dtype = dtype
        self.device = device
        self.elem = 8 if dtype == "complex64" else 16
        self.ndt = _native.EFFT_C64 if dtype == "complex64" else _native.EFFT_C128
        self.group = group

    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def split(self, n, world):
        return split_sizes(n, world, self.dtype)

    def shard_plan(self, n, world, rank, direction, n1, n2):
        p = self.native.ShardRankPlan(n, self.ndt, direction, world, rank, self.device)
        if p.split() != (n1, n2):  # the Python mirror and the library must agree
            raise RuntimeError(f"split mismatch: library {p.split()} vs {(n1, n2)}")
        return p

    def pass0(self, plan, src, dst):
        plan.execute_pass(0, src.data_ptr(), dst.data_ptr(), self._stream())

    def pass1(self, plan, buf):
        plan.execute_pass(1, buf.data_ptr(), buf.data_ptr(), self._stream())

    def swap01(self, src, dst, n0, n1, n2):
        self.native.permute_swap01(src.data_ptr(), dst.data_ptr(), n0, n1, n2, self.elem, self._stream())

    def all_to_all(self, src, dst):
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            # real views: every NCCL build handles float all-to-all
            dist.all_to_all_single(self.torch.view_as_real(dst), self.torch.view_as_real(src),
                                   group=self.group)
        else:
            dst.copy_(src)


def flops(n: int) -> float:
    return 5.0 * n * math.log2(n)
