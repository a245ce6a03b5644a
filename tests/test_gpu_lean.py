"""The lean staged passes (paper_1409_5757_b200/csrc/lean.cu) vs the oracle -- needs a B200.

The planner routes complex64 / complex128 transforms with 2^26 <= N <= 2^32
and 3*2^24 <= N <= 3*2^30 to the lean kernels; these tests pin them at sizes
the fp64 oracle (oracle/efft_oracle.c) finishes in seconds, for both
directions, both pass shapes (R1 = R2 and R1 = 2 R2), the radix-3 family, the
non-finite input flag and the agreement with the generic staged kernels
(EFFT_LEAN=0).
Tolerances as in test_gpu_parity.py: rel-L2 <= 1e-12 log2N (c128), 1e-5 log2N (c64).
"""
import math
import os

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
TT = {"complex64": torch.complex64, "complex128": torch.complex128}
NDT = {"complex64": _native.EFFT_C64, "complex128": _native.EFFT_C128}


def tol(n, dtype):
    return (1e-12 if dtype == "complex128" else 1e-5) * math.log2(n)


def run(x_dev, dtype, direction=-1, flags=0):
    p = _native.NativePlan(x_dev.shape[0], NDT[dtype], direction, 0, flags)
    y = torch.empty_like(x_dev)
    p.execute(x_dev.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return p, y


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
@pytest.mark.parametrize("lg", [26, 27])
def test_lean_forward_inverse_vs_oracle(lg, dtype):
    n = 1 << lg
    x = random_c(n, seed=lg)
    xd = torch.from_numpy(x.astype(NP[dtype])).cuda()
    p, y = run(xd, dtype)
    assert "lean" in p.describe()
    assert oracle.rel_l2(y.cpu().numpy(), oracle.transform(x)) <= tol(n, dtype)
    _, z = run(y, dtype, direction=1)  # inverse, scaled by 1/N
    assert oracle.rel_l2(z.cpu().numpy(), x) <= 2 * tol(n, dtype)
    _, w = run(xd, dtype, direction=1)
    assert oracle.rel_l2(w.cpu().numpy(), oracle.transform(x, direction=1)) <= tol(n, dtype)


@pytest.mark.parametrize("lg", [24, 25])
def test_lean_complex64_rho_b_16_vs_oracle(lg):
    """complex64 from 2^24: rho_b = 16 (the B stage is one 16-point DFT)."""
    n = 1 << lg
    x = random_c(n, seed=lg + 100)
    xd = torch.from_numpy(x.astype(np.complex64)).cuda()
    p, y = run(xd, "complex64")
    assert "rho_b=16" in p.describe()
    assert oracle.rel_l2(y.cpu().numpy(), oracle.transform(x)) <= tol(n, "complex64")
    _, z = run(y, "complex64", direction=1)
    assert oracle.rel_l2(z.cpu().numpy(), x) <= 2 * tol(n, "complex64")


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
@pytest.mark.parametrize("n", [3 << 24, 3 << 25])
def test_lean_radix3_family_vs_oracle(n, dtype):
    """N = 3 * 2^k: pass 1 runs rho_a = 192 = 16 x 12 tiles."""
    x = random_c(n, seed=n % 1000)
    xd = torch.from_numpy(x.astype(NP[dtype])).cuda()
    p, y = run(xd, dtype)
    assert "rho_a=192" in p.describe()
    assert oracle.rel_l2(y.cpu().numpy(), oracle.transform(x)) <= tol(n, dtype)
    _, z = run(y, dtype, direction=1)
    assert oracle.rel_l2(z.cpu().numpy(), x) <= 2 * tol(n, dtype)


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
@pytest.mark.parametrize("m,ra", [(5, 160), (7, 224)])
def test_lean_radix5_radix7_families_vs_oracle(m, ra, dtype):
    """N = 5 * 2^23, 7 * 2^23: the in-place pass runs rho_a = 10 x 16 / 14 x 16 tiles."""
    n = m << 23
    x = random_c(n, seed=m)
    xd = torch.from_numpy(x.astype(NP[dtype])).cuda()
    p, y = run(xd, dtype)
    assert f"rho_a={ra}" in p.describe()
    assert oracle.rel_l2(y.cpu().numpy(), oracle.transform(x)) <= tol(n, dtype)
    _, z = run(y, dtype, direction=1)
    assert oracle.rel_l2(z.cpu().numpy(), x) <= 2 * tol(n, dtype)


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
def test_lean_agrees_with_generic_staged_path(dtype, monkeypatch):
    n = 1 << 26
    x = torch.from_numpy(random_c(n, seed=7).astype(NP[dtype])).cuda()
    p, y = run(x, dtype)
    assert "lean" in p.describe()
    monkeypatch.setenv("EFFT_LEAN", "0")
    q, z = run(x, dtype)
    assert "lean" not in q.describe()
    d = (torch.linalg.vector_norm((y - z).to(torch.complex128)) /
         torch.linalg.vector_norm(z.to(torch.complex128))).item()
    assert d <= 2 * tol(n, dtype)


def test_lean_structured_inputs_exact_bins():
    """Impulse -> flat spectrum, pure tone -> one bin (c128, exact up to rounding)."""
    n = 1 << 26
    x = torch.zeros(n, dtype=torch.complex128, device="cuda")
    x[0] = 1
    _, y = run(x, "complex128")
    assert torch.max(torch.abs(y - 1)).item() < 1e-13
    k0 = 123457
    t = torch.arange(n, device="cuda", dtype=torch.float64)
    x = torch.polar(torch.ones_like(t), 2 * math.pi * ((k0 * t) % n) / n)
    _, y = run(x, "complex128")
    mag = torch.abs(y)
    assert int(torch.argmax(mag)) == k0
    assert abs(mag[k0].item() / n - 1) < 1e-12
    mag[k0] = 0
    assert mag.max().item() / n < 1e-11


@pytest.mark.parametrize("n,dtype", [(1 << 26, "complex64"), (1 << 26, "complex128"), (3 << 24, "complex128")])
def test_lean_nonfinite_flag(n, dtype):
    x = torch.zeros(n, dtype=TT[dtype], device="cuda")
    x[12345] = float("inf")
    p, _ = run(x, dtype, flags=1)  # EFFT_FLAG_CHECK_FINITE
    assert p.nonfinite_seen(torch.cuda.current_stream().cuda_stream)
    x[12345] = 0
    p.execute(x.data_ptr(), torch.empty_like(x).data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert not p.nonfinite_seen(torch.cuda.current_stream().cuda_stream)
    assert "lean" in p.describe()


@pytest.mark.slow
@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
def test_lean_2p29_vs_oracle_spots_and_parseval(dtype):
    """R1 = 2 R2 at a size the full oracle is too slow for: spot values against
    the fp64 direct sum, Parseval and the round trip."""
    n = 1 << 29
    g = torch.Generator(device="cuda").manual_seed(29)
    x = torch.randn(n, dtype=TT[dtype], device="cuda", generator=g)
    p, y = run(x, dtype)
    assert "lean" in p.describe()
    ks = np.array([0, 1, 2, n // 2, n - 1] + list(np.random.default_rng(29).integers(0, n, 11)))
    xh = x.cpu().numpy().astype(np.complex128)
    exact = oracle.dft_at(xh, ks)
    yk = y[torch.from_numpy(ks).cuda()].cpu().numpy().astype(np.complex128)
    scale = np.sqrt(np.mean(np.abs(exact) ** 2))
    assert float(np.max(np.abs(yk - exact) / np.maximum(np.abs(exact), scale))) < tol(n, dtype)
    ex = torch.sum(torch.abs(x.to(torch.complex128)) ** 2).item()
    ey = torch.sum(torch.abs(y.to(torch.complex128)) ** 2).item()
    assert abs(ey / (n * ex) - 1) < (1e-12 if dtype == "complex128" else 1e-5)
    _, z = run(y, dtype, direction=1)
    rt = (torch.linalg.vector_norm((z - x).to(torch.complex128)) /
          torch.linalg.vector_norm(x.to(torch.complex128))).item()
    assert rt <= 2 * tol(n, dtype)


def test_lean_env_restored():
    assert os.environ.get("EFFT_LEAN") in (None, "1")


@pytest.mark.parametrize("lag,slots", [(1, 2), (2, 3), (3, 5)])
@pytest.mark.parametrize("n,dtype", [(1 << 24, "complex64"), (1 << 26, "complex128"), (3 << 24, "complex128")])
def test_lean_minimal_ring_is_deadlock_free_and_exact(n, dtype, lag, slots, monkeypatch):
    """Maximal dependency pressure: B tiles claimed right behind their A tiles and
    a ring of only lag + 1 slots -- every wait is exercised, results unchanged."""
    x = torch.from_numpy(random_c(n, seed=11).astype(NP[dtype])).cuda()
    _, ref = run(x, dtype)
    monkeypatch.setenv("EFFT_LEAN_LAG", str(lag))
    monkeypatch.setenv("EFFT_LEAN_SLOTS", str(slots))
    p, y = run(x, dtype)
    assert f"lag={lag} slots={slots}" in p.describe()
    assert torch.equal(y, ref)  # deterministic: same arithmetic, any schedule


@pytest.mark.parametrize("lg", [24, 26, 27])
def test_pipelined_kernel_vs_oracle_and_default_path(lg, monkeypatch):
    """EFFT_LEAN_PIPE=3: the TMA-fed pipelined pair kernel (one CTA per SM, three
    compute groups, issue warps + a release lane, static schedule) in both passes:
    same arithmetic as the default kernels, so bit-identical output, both directions."""
    n = 1 << lg
    x = random_c(n, seed=lg + 7)
    xd = torch.from_numpy(x.astype(np.complex64)).cuda()
    _, ref = run(xd, "complex64")
    _, iref = run(ref, "complex64", direction=1)
    monkeypatch.setenv("EFFT_LEAN_PIPE", "3")
    p, y = run(xd, "complex64", flags=_native.EFFT_FLAG_CHECK_FINITE)
    assert "x 512" in p.describe()  # 3 x 128 compute threads + 4 service warps
    assert not p.nonfinite_seen(torch.cuda.current_stream().cuda_stream)
    assert oracle.rel_l2(y.cpu().numpy(), oracle.transform(x)) <= tol(n, "complex64")
    assert torch.equal(y, ref)
    _, z = run(y, "complex64", direction=1)
    assert torch.equal(z, iref)
    assert oracle.rel_l2(z.cpu().numpy(), x) <= 2 * tol(n, "complex64")


@pytest.mark.parametrize("lag,slots", [(1, 2), (2, 3), (4, 6)])
def test_pipelined_kernel_minimal_ring_and_repeats(lag, slots, monkeypatch):
    """The pipelined kernel under maximal dependency pressure, run repeatedly (its
    mbarrier rings must never be overrun whatever the timing), and its non-finite flag."""
    n = 1 << 25
    x = torch.from_numpy(random_c(n, seed=5).astype(np.complex64)).cuda()
    _, ref = run(x, "complex64")
    monkeypatch.setenv("EFFT_LEAN_PIPE", "3")
    monkeypatch.setenv("EFFT_LEAN_LAG", str(lag))
    monkeypatch.setenv("EFFT_LEAN_SLOTS", str(slots))
    p = _native.NativePlan(n, _native.EFFT_C64, -1, 0, _native.EFFT_FLAG_CHECK_FINITE)
    assert f"lag={lag} slots={slots}" in p.describe()
    s = torch.cuda.current_stream().cuda_stream
    y = torch.empty_like(x)
    for _ in range(8):
        y.zero_()
        p.execute(x.data_ptr(), y.data_ptr(), s)
    torch.cuda.synchronize()
    assert torch.equal(y, ref)
    assert not p.nonfinite_seen(s)
    xb = x.clone()
    xb[12345] = complex(float("inf"), 0.0)
    p.execute(xb.data_ptr(), y.data_ptr(), s)
    torch.cuda.synchronize()
    assert p.nonfinite_seen(s)
