"""CUDA path vs the oracle (oracle/efft_oracle.c) through the C ABI -- needs a B200.

Tolerances (north star, BASELINE.json): relative L2 <= 1e-12*log2(N) for
complex128 and <= 1e-5*log2(N) for complex64; the reference's own real-input
criterion (L2 <= 1e-6, test_acceptance.py:33-51) for the float32 PERM path.
"""
import math

import numpy as np
import pytest

import oracle
from conftest import golden, random_c, random_f32

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1409_5757_b200 as efft  # noqa: E402
from paper_1409_5757_b200 import _native  # noqa: E402

NP = {"complex64": np.complex64, "complex128": np.complex128}
NDT = {"complex64": _native.EFFT_C64, "complex128": _native.EFFT_C128}


def tol(n, dtype):
    lg = max(1.0, math.log2(n))
    return (1e-12 if dtype == "complex128" else 1e-5) * lg


def gpu_transform(x, dtype, direction=-1):
    """Device transform through the C ABI (efft_execute)."""
    p = _native.NativePlan(x.shape[0], NDT[dtype], direction, 0)
    xi = torch.from_numpy(np.ascontiguousarray(x, dtype=NP[dtype])).cuda()
    yo = torch.empty_like(xi)
    p.execute(xi.data_ptr(), yo.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return yo.cpu().numpy()


SIZES = [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 3, 6, 12, 24, 48, 96, 192, 384, 768, 3 * 1024,
         4096, 2 ** 14, 3 * 2 ** 14, 2 ** 16, 2 ** 18, 2 ** 19, 2 ** 20, 3 * 2 ** 19, 2 ** 21,
         # radix-5 / radix-7 families: direct tiles, two direct
         # passes, staged rho_a = 320 / 448
         5, 10, 40, 160, 320, 640, 5 * 2 ** 10, 5 * 2 ** 14, 5 * 2 ** 16, 5 * 2 ** 19,
         7, 28, 112, 448, 896, 7 * 2 ** 10, 7 * 2 ** 15, 7 * 2 ** 17, 7 * 2 ** 19,
         # generic two-pass plans above dmax^2 (direct M*2^k pass 1 + staged pass 2,
         # c128 rho_b up to 512 at 2^25) and the radix-M families in that range
         2 ** 22, 2 ** 23, 2 ** 24, 2 ** 25, 3 * 2 ** 21, 3 * 2 ** 23, 5 * 2 ** 21, 7 * 2 ** 21]


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
@pytest.mark.parametrize("n", SIZES)
def test_forward_and_roundtrip_vs_oracle(n, dtype):
    x = random_c(n, seed=n + 17)
    exact = oracle.transform(x)  # fp64 restatement
    y = gpu_transform(x, dtype)
    assert oracle.rel_l2(y, exact) <= tol(n, dtype), n
    z = gpu_transform(y, dtype, direction=1)
    assert oracle.rel_l2(z, x.astype(NP[dtype])) <= 2 * tol(n, dtype)
    # inverse alone against the oracle's inverse
    assert oracle.rel_l2(gpu_transform(x, dtype, 1), oracle.transform(x, direction=1)) <= tol(n, dtype)


@pytest.mark.parametrize("n", [1024, 3072, 4096])
@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
def test_golden_fixtures_from_reference(n, dtype):
    g = golden(f"complex_{n}.npz")
    y = gpu_transform(g["x"], dtype)
    assert oracle.rel_l2(y, g["exact"]) <= tol(n, dtype)


def test_c1_full_parity_and_reference_spot_checks():
    """Config 1: N=2^21 complex128 through the public API vs oracle + reference naive_dft_at."""
    g = golden("spot_c1.npz")
    n = 1 << 21
    rng = np.random.default_rng(int(g["seed"]))
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    plan = efft.plan_create(n, 3, dtype="complex128")
    with efft.handle_create(plan) as h:
        h.data[:] = x
        y = np.array(efft.run_transform(h))
        assert np.array_equal(h.data, x)  # input preserved (core.py:146-149)
    assert oracle.rel_l2(y, oracle.transform(x)) <= tol(n, "complex128")
    exact = g["vals"]
    scale = np.maximum(np.abs(exact), np.sqrt(np.mean(np.abs(exact) ** 2)))
    assert np.max(np.abs(y[g["ks"]] - exact) / scale) < 1e-12


class TestRealPermPath:
    """The reference's own real float32 PERM contract on the GPU."""

    @pytest.mark.parametrize("n", [256, 1024, 4096])
    def test_reference_fixtures(self, n):
        g = golden(f"real_{n}.npz")
        with efft.handle_create(efft.plan_create(n, 2, test_mode=True)) as h:
            h.data[:] = g["x"]
            out = np.asarray(h.run(), dtype=np.float64)
        assert oracle.rel_l2(out, g["naive"]) <= 1e-6
        assert oracle.rel_l2(out, g["ref_s2"].astype(np.float64)) <= 1e-6

    @pytest.mark.parametrize("exp", [3, 8, 10, 12, 14, 20, 22])
    def test_oracle_grid(self, exp):
        n = 1 << exp
        x = random_f32(n, seed=exp)
        exact = np.fft.fft(x.astype(np.float64))
        packed = np.empty(n)
        packed[0], packed[1] = exact[0].real, exact[n // 2].real
        packed[2::2], packed[3::2] = exact[1:n // 2].real, exact[1:n // 2].imag
        with efft.handle_create(efft.plan_create(n, 0, test_mode=True)) as h:
            h.data[:] = x
            out = np.asarray(h.run(), dtype=np.float64)
        assert oracle.rel_l2(out, packed) <= 1e-6

    def test_kats(self):  # reference test_leaf_dft.py:22-38 via the full transform
        with efft.handle_create(efft.plan_create(8, 0, test_mode=True)) as h:
            h.data[:] = [1, 0, 0, 0, 0, 0, 0, 0]
            assert np.allclose(h.run(), [1, 1, 1, 0, 1, 0, 1, 0], atol=1e-6)
            h.data[:] = np.arange(1, 9)
            assert np.allclose(h.run(), [36, -4, -4, 9.6569, -4, 4, -4, 1.6569], atol=1e-3)


class TestHandle:
    """reference pkg/tests/test_core.py::TestHandle against the GPU handle."""

    def test_buffers_aligned_and_distinct(self):
        with efft.handle_create(efft.plan_create(2 ** 12, 2, dtype="complex64")) as h:
            d, r = efft.data_view(h), efft.result_view(h)
            assert d.shape == (2 ** 12,) and r.shape == (2 ** 12,)
            assert d.ctypes.data % 64 == 0
            assert not np.shares_memory(d, r)

    def test_result_view_is_read_only(self):
        with efft.handle_create(efft.plan_create(2 ** 12, 2)) as h:
            with pytest.raises(ValueError):
                efft.result_view(h)[0] = 1.0

    def test_reuse_is_bitwise_deterministic(self):
        n = 2 ** 20
        with efft.handle_create(efft.plan_create(n, 3, dtype="complex64")) as h:
            h.data[:] = random_c(n, seed=1, dtype=np.complex64)
            first = np.array(h.run())
            for _ in range(5):
                assert np.array_equal(np.array(h.run()), first)

    def test_two_handles_are_independent(self):
        p = efft.plan_create(2 ** 10, 1, test_mode=True, dtype="complex128")
        with efft.handle_create(p) as h1, efft.handle_create(p) as h2:
            h1.data[:] = 1.0
            h2.data[:] = 2.0
            h1.run()
            assert np.all(h2.data == 2.0)
            assert np.allclose(h1.result[0], 1024.0)

    def test_close_is_idempotent(self):
        h = efft.handle_create(efft.plan_create(2 ** 10, 0, test_mode=True))
        h.close()
        h.close()

    def test_non_finite_input_rejected(self):  # scatter.py:38-39
        with efft.handle_create(efft.plan_create(2 ** 12, 0, dtype="complex64")) as h:
            h.data[:] = 0
            h.data[5] = np.nan
            with pytest.raises(ValueError):
                h.run()
            h.data[5] = 0
            h.run()  # flag cleared

    def test_host_batch_entry_matches_single_calls(self):
        """efft_execute_host_batch (pipelined H2D / passes / D2H) == one call per input."""
        from paper_1409_5757_b200 import _native

        n = 1 << 22
        xs = [random_c(n, seed=s).astype(np.complex64) for s in (1, 2, 3)]
        p = _native.NativePlan(n, _native.EFFT_C64, -1, 0)
        ins = [torch.from_numpy(x).pin_memory() for x in xs]
        outs = [torch.empty_like(t).pin_memory() for t in ins]
        p.execute_host_batch([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], 0)
        for x, o in zip(xs, outs):
            one = np.empty_like(x)
            p.execute_host(x.ctypes.data, one.ctypes.data, 0)
            assert np.array_equal(o.numpy(), one)

    def test_host_buffer_entry_matches_device_entry(self):
        n = 2 ** 18
        x = random_c(n, seed=3)
        with efft.handle_create(efft.plan_create(n, 2, dtype="complex128")) as h:
            out = np.empty_like(x)
            h.execute_host(x, out)
            h.data[:] = x
            assert np.array_equal(out, h.run())


# ---- full BASELINE sizes: size-independent properties ------------------------
def _spot(x_host, y, ks):
    exact = oracle.dft_at(x_host, ks)
    scale = np.sqrt(np.mean(np.abs(exact) ** 2))
    return float(np.max(np.abs(y - exact) / np.maximum(np.abs(exact), scale)))


@pytest.mark.slow
def test_c2_2p27_complex128_vs_oracle_and_roundtrip():
    from paper_1409_5757_b200 import workloads

    n = 1 << 27
    x = workloads.make_input(n, "complex128", "normal", workloads.seed_for("c2"))
    fwd = _native.NativePlan(n, _native.EFFT_C128, -1, 0)
    inv = _native.NativePlan(n, _native.EFFT_C128, 1, 0)
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    s = torch.cuda.current_stream().cuda_stream
    fwd.execute(x.data_ptr(), y.data_ptr(), s)
    inv.execute(y.data_ptr(), z.data_ptr(), s)
    torch.cuda.synchronize()
    xh, yh = x.cpu().numpy(), y.cpu().numpy()
    assert oracle.rel_l2(yh, oracle.transform(xh)) <= tol(n, "complex128")
    assert oracle.rel_l2(z.cpu().numpy(), xh) <= 2 * tol(n, "complex128")


@pytest.mark.slow
def test_c3_2p30_complex64_properties():
    from paper_1409_5757_b200 import workloads

    n = 1 << 30
    x = workloads.make_input(n, "complex64", "normal", workloads.seed_for("c3"))
    fwd = _native.NativePlan(n, _native.EFFT_C64, -1, 0)
    inv = _native.NativePlan(n, _native.EFFT_C64, 1, 0)
    y = torch.empty_like(x)
    s = torch.cuda.current_stream().cuda_stream
    fwd.execute(x.data_ptr(), y.data_ptr(), s)
    torch.cuda.synchronize()
    # Parseval: sum|X|^2 = N sum|x|^2
    ex = torch.sum(torch.abs(x.to(torch.complex128)) ** 2).item()
    ey = torch.sum(torch.abs(y.to(torch.complex128)) ** 2).item()
    assert abs(ey / (n * ex) - 1) < 1e-5
    # round trip
    z = torch.empty_like(x)
    inv.execute(y.data_ptr(), z.data_ptr(), s)
    torch.cuda.synchronize()
    rt = (torch.linalg.vector_norm((z - x).to(torch.complex128)) /
          torch.linalg.vector_norm(x.to(torch.complex128))).item()
    assert rt <= 2 * tol(n, "complex64")
    # spot checks against the fp64 direct sum (oracle.py:79-89 restated)
    ks = np.array([0, 1, 12345, n // 2, n - 1] + list(np.random.default_rng(3).integers(0, n, 11)))
    xh = x.cpu().numpy().astype(np.complex128)
    yk = y[torch.from_numpy(ks).cuda()].cpu().numpy().astype(np.complex128)
    assert _spot(xh, yk, ks) < 1e-4


@pytest.mark.slow
def test_c4_3x2p28_complex128_tones():
    from paper_1409_5757_b200 import workloads

    n = 3 << 28
    seed = workloads.seed_for("c4")
    x = workloads.make_input(n, "complex128", "tones", seed)
    fwd = _native.NativePlan(n, _native.EFFT_C128, -1, 0)
    y = torch.empty_like(x)
    fwd.execute(x.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    mag = torch.abs(y)
    top = torch.topk(mag, workloads.N_TONES).indices.cpu().numpy()
    freqs = workloads.tone_frequencies(n, seed)
    assert sorted(top.tolist()) == freqs
    peaks = mag[torch.tensor(freqs, device="cuda")].cpu().numpy()
    assert np.all(np.abs(peaks / n - 1) < 1e-3)
    ks = np.array(freqs[:4] + [1, n // 3, n - 1] + list(np.random.default_rng(4).integers(0, n, 9)))
    xh = x.cpu().numpy()
    yk = y[torch.from_numpy(ks).cuda()].cpu().numpy()
    assert _spot(xh, yk, ks) < tol(n, "complex128")


@pytest.mark.slow
def test_c5_2p32_complex128_roundtrip_and_spots():
    """Config 5: N = 2^32 complex128 (64 GiB) forward + inverse on ONE B200
    (in + out + staging ring = 128 GiB + ~90 MB); the input is regenerated from
    its seed for the round-trip check, so no third array is needed."""
    from paper_1409_5757_b200 import workloads

    n = 1 << 32
    import gc

    gc.collect()
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    if free < 2 * n * 16 + (1 << 30):
        pytest.skip("needs ~130 GiB of device memory")
    import psutil

    if psutil.virtual_memory().available < n * 16 + (16 << 30):
        pytest.skip("needs ~80 GB of host memory for the host-side checks")
    seed = workloads.seed_for("c5")
    x = workloads.make_input(n, "complex128", "uniform", seed)
    xh = x.cpu().numpy()
    y = torch.empty_like(x)
    s = torch.cuda.current_stream().cuda_stream
    fwd = _native.NativePlan(n, _native.EFFT_C128, -1, 0)
    fwd.execute(x.data_ptr(), y.data_ptr(), s)
    torch.cuda.synchronize()
    ks = np.array([0, 1, n // 2, n - 1] + list(np.random.default_rng(5).integers(0, n, 12)))
    yk = y[torch.from_numpy(ks).cuda()].cpu().numpy()
    assert _spot(xh, yk, ks) < tol(n, "complex128")
    # Parseval on the device (chunked: a full |x|^2 temporary would not fit)
    def energy(t):
        return sum(torch.view_as_real(t[i:i + (1 << 28)]).pow(2).sum().item() for i in range(0, n, 1 << 28))

    ex, ey = energy(x), energy(y)
    assert abs(ey / (n * ex) - 1) < 1e-12
    fwd.close()
    inv = _native.NativePlan(n, _native.EFFT_C128, 1, 0)
    inv.execute(y.data_ptr(), x.data_ptr(), s)  # overwrite x; xh holds the original
    torch.cuda.synchronize()
    del y
    # round-trip error chunk by chunk on the device (no second 64 GiB host copy)
    num = den = 0.0
    for i in range(0, n, 1 << 28):
        xc = torch.from_numpy(xh[i:i + (1 << 28)]).cuda()
        num += torch.view_as_real(x[i:i + (1 << 28)] - xc).pow(2).sum().item()
        den += torch.view_as_real(xc).pow(2).sum().item()
    rt = math.sqrt(num / den)
    assert rt <= 2 * tol(n, "complex128")
