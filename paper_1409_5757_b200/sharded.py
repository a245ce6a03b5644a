"""Six-step sharded transform: one N-point DFT block-distributed over G ranks.

Layout contract (natural-order block shards): rank p holds input elements
x[p*N/G, (p+1)*N/G) and receives output coefficients X[p*N/G, (p+1)*N/G).
The reference has no distributed path (it is one shared-memory process,
reference parallel.py); this is the B200 extension BASELINE.json asks for.

With N = N1*N2, n = n1*N2 + n2 and k = k1 + N1*k2,

    X[k1 + N1 k2] = sum_n2 W_N2^(n2 k2) W_N^(n2 k1) sum_n1 x[n1 N2 + n2] W_N1^(n1 k1)

Per rank p (L1 = N1/G, L2 = N2/G):
  1. pack   S[q][r][c] = x_p[r][q*L2 + c]                    (swap01, local)
  2. a2a    B[n1][c]   = column block p of x, all n1         (all-to-all #1)
  3. FFT    Y[k1][c]   = sum_n1 B[n1][c] W_N1^(n1 k1)          (column plan, len N1)
  4. a2a    Z[q][k1'][c] = Y_q[p*L1 + k1'][c]                 (all-to-all #2)
  5. unpack T[n2][k1'] = Z[q][k1'][c], n2 = q*L2 + c          (swap12, local)
  6. FFT    X[k2][k1'] = sum_n2 T[n2][k1'] W_N^(n2 (p L1 + k1')) W_N2^(n2 k2)
                                                              (column plan, len N2, twiddle offset p*L1)
  7. a2a    V[q][k2'][k1'] = X_q[p*L2 + k2'][k1']             (all-to-all #3)
  8. unpack y_p[k2'][q][k1'] = V[q][k2'][k1']                 (swap01) -> natural order
Three all-to-all exchanges (k = 3 in SURVEY section 8e), two local FFT passes
(each one HBM pass through the staged kernels), three local permutations.

The compute steps go through a backend: `GpuBackend` (libefft_b200.so column
plans + permutation kernels, NCCL all-to-all via torch.distributed) is the
product path; tests substitute a CPU backend built on the oracle's pass
primitive and run the exchange over gloo (tests/test_sharded.py).
"""

import math

from .errors import BinsizeNotPowerOfTwo


def split_sizes(n: int, world: int):
    """N = N1 * N2 with G | N1, G | N2, both as balanced as possible (N1 gets the factor 3)."""
    m, t = n, 0
    while m % 2 == 0:
        m //= 2
        t += 1
    if m not in (1, 3, 5, 7) or world < 1 or world & (world - 1):
        raise BinsizeNotPowerOfTwo(f"n={n} / world={world} not shardable (need n = M*2^t with M in {1, 3, 5, 7}, G = 2^g)")
    g = world.bit_length() - 1
    t1 = t // 2
    n1, n2 = m << t1, 1 << (t - t1)
    if (n1 % world) or (n2 % world) or n1 // world < 1 or n2 // world < 1:
        raise BinsizeNotPowerOfTwo(f"n={n} too small for {world} shards")
    del g
    return n1, n2


class ShardedTransform:
    """Forward (-1) or inverse (+1, scaled 1/N) DFT of a block-sharded array."""

    def __init__(self, n: int, world: int, rank: int, direction: int, backend):
        self.n, self.world, self.rank, self.direction = n, world, rank, direction
        self.n1, self.n2 = split_sizes(n, world)
        self.l1, self.l2 = self.n1 // world, self.n2 // world
        self.backend = backend
        # inverse: each column plan scales by 1/len, together 1/(N1*N2) = 1/N
        self.fft1 = backend.column_plan(self.n1, self.l2, direction, tw_mod=0, tw_offset=0,
                                        scale=direction == 1)
        self.fft2 = backend.column_plan(self.n2, self.l1, direction, tw_mod=n,
                                        tw_offset=rank * self.l1, scale=direction == 1)

    def execute(self, x_local, y_local, work):
        """x_local, y_local, work: N/G-element device (or host) buffers; x_local preserved."""
        b, G, L1, L2, N1, N2 = self.backend, self.world, self.l1, self.l2, self.n1, self.n2
        b.swap01(x_local, work, L1, G, L2)            # S[q][r][c]
        b.all_to_all(work, y_local)                   # B[n1][c]   (N1 x L2)
        b.run(self.fft1, y_local, y_local)            # Y[k1][c], in place
        b.all_to_all(y_local, work)                   # Z[q][k1'][c]
        b.swap12(work, y_local, G, L1, L2)            # T[q][c][k1'] = T[n2][k1']
        b.run(self.fft2, y_local, y_local)            # X[k2][k1'], in place
        b.all_to_all(y_local, work)                   # V[q][k2'][k1']
        b.swap01(work, y_local, G, L2, L1)            # y[k2'][q][k1']
        return y_local

    @staticmethod
    def exchanged_bytes(n: int, world: int, elem: int) -> int:
        """Bytes one rank sends per transform: 3 exchanges of (G-1)/G of its N/G elements."""
        return 3 * (world - 1) * (n // world) * elem // world


class GpuBackend:
    """Product path: libefft_b200.so column plans + permutation kernels, NCCL all-to-all."""

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

    def column_plan(self, length, cols, direction, tw_mod, tw_offset, scale):
        flags = self.native.EFFT_FLAG_SCALE_INVERSE if scale else 0
        return self.native.NativePlan(length, self.ndt, direction, self.device, flags,
                                      columns=(cols, tw_mod, tw_offset))

    def run(self, plan, src, dst):
        plan.execute(src.data_ptr(), dst.data_ptr(), self._stream())

    def swap01(self, src, dst, n0, n1, n2):
        self.native.permute_swap01(src.data_ptr(), dst.data_ptr(), n0, n1, n2, self.elem, self._stream())

    def swap12(self, src, dst, n0, n1, n2):
        self.native.permute_swap12(src.data_ptr(), dst.data_ptr(), n0, n1, n2, self.elem, self._stream())

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
