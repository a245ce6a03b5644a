"""The reference's own acceptance and pipeline suites, restated against the GPU
backend behind the same entry points (the drop-in proof).

The reference package is not on the GPU box, so its test files cannot run
there unchanged; each test below restates one reference test -- same sizes,
seeds, split grids, worker counts, tolerances and comparators -- through
``paper_1409_5757_b200.plan_create / handle_create / run_transform`` (the
reference's names and argument validation).  The fp64 comparator of the
reference (``naive_dft`` / ``naive_dft_at``) is replaced by the oracle's fp64
restatement (``oracle.transform`` / ``oracle.dft_at``), which tests/test_oracle.py
pins to the reference's own ``naive_dft`` fixtures.  Not restated: the CPU
scaling test (test_acceptance.py:118-; the GPU ignores `workers`) and
bit-equality with the reference's CPU leaf kernel (test_recombine.py:136-144).
"""
import math

import numpy as np
import pytest

import oracle
from conftest import random_f32

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1409_5757_b200 as efft  # noqa: E402
from paper_1409_5757_b200 import PermSpectrum, data_view, handle_create, plan_create, result_view  # noqa: E402


def random_signal(n, seed):
    """reference bench.py:109-112"""
    rng = np.random.default_rng(seed)
    return rng.random(n, dtype=np.float32) - np.float32(0.5)


def packed_exact(x):
    """pack_perm(naive_dft(x)) (reference oracle.py:92-112) via the fp64 restatement."""
    n = x.shape[0]
    f = oracle.transform(x.astype(np.complex128))
    out = np.empty(n)
    out[0], out[1] = f[0].real, f[n // 2].real
    out[2::2], out[3::2] = f[1:n // 2].real, f[1:n // 2].imag
    return out


def l2_norm(computed, exact):
    """reference oracle.py:115-127"""
    a = np.asarray(computed, dtype=np.float64)
    b = np.asarray(exact, dtype=np.float64)
    return float(np.sqrt(np.sum((a - b) ** 2)) / np.sqrt(np.sum(b * b)))


def exact_coefficients(x, ks):
    """naive_dft_at (oracle.py:79-89) for real x at any k via conjugate symmetry."""
    n = x.shape[0]
    ks = np.asarray(ks, dtype=np.int64)
    lo = np.where(ks <= n // 2, ks, n - ks)
    v = oracle.dft_at(x.astype(np.complex128), lo)
    return np.where(ks <= n // 2, v, np.conj(v))


# ---- reference pkg/tests/test_acceptance.py --------------------------------
def test_oracle_equivalence_suite():
    """test_acceptance.py:33-51: L2 <= 1e-6 over n in {2^8..2^14}, every valid
    split, 20 seeded signals each, workers=2, test_mode."""
    worst = 0.0
    for exp in (8, 10, 12, 14):
        n = 1 << exp
        signals = [random_f32(n, seed=exp * 1000 + t) for t in range(20)]
        refs = [packed_exact(x) for x in signals]
        for s in range(exp - 1):
            with handle_create(plan_create(n, s, workers=2, test_mode=True)) as h:
                for x, ref in zip(signals, refs):
                    h.data[:] = x
                    err = l2_norm(np.asarray(h.run(), dtype=np.float64), ref)
                    worst = max(worst, err)
                    assert err <= 1e-6, (n, s, err)
    print(f"oracle equivalence: worst L2 {worst:.3e}")


def test_large_size_spot_checks():
    """test_acceptance.py:54-71: n = 2^24, 64 spot coefficients in [0, n/2],
    s in {2, 4}, relative error <= 1e-5 against the exact direct sums."""
    n = 1 << 24
    x = random_signal(n, seed=2024)
    idx = np.random.default_rng(77).integers(0, n // 2 + 1, size=64)
    exact = exact_coefficients(x, idx)
    scale = np.maximum(np.abs(exact), np.sqrt(np.mean(np.abs(exact) ** 2)))
    for s in (2, 4):
        with handle_create(plan_create(n, s, workers=2)) as h:
            h.data[:] = x
            spec = PermSpectrum(np.array(h.run(), dtype=np.float64))
        got = np.array([spec.coefficient(int(k)) for k in idx])
        err = float(np.max(np.abs(got - exact) / scale))
        assert err <= 1e-5, (s, err)


def test_determinism_across_workers_and_runs():
    """test_acceptance.py:100-115: n = 2^20, s = 3, bitwise identical for
    T in {1, 2, 4, 8} and across reruns."""
    n, s = 1 << 20, 3
    x = random_signal(n, seed=555)
    reference = None
    for workers in (1, 2, 4, 8):
        with handle_create(plan_create(n, s, workers=workers)) as h:
            h.data[:] = x
            first = np.array(h.run())
            h.run()
            again = np.array(h.result)
        assert np.array_equal(first, again)
        if reference is None:
            reference = first
        assert np.array_equal(first, reference)


# ---- reference pkg/tests/test_core.py::TestHandle ---------------------------
class TestHandle:
    def test_buffers_aligned_and_distinct(self):  # test_core.py:66-73
        with handle_create(plan_create(2 ** 12, 2, workers=2)) as h:
            d, r = data_view(h), result_view(h)
            assert d.shape == (2 ** 12,) and r.shape == (2 ** 12,)
            assert d.ctypes.data % 64 == 0 and r.ctypes.data % 64 == 0
            assert not np.shares_memory(d, r)
            assert np.all(np.isfinite(d)) and np.all(np.isfinite(r))

    def test_result_view_is_read_only(self):  # test_core.py:75-78
        with handle_create(plan_create(2 ** 12, 2, workers=1)) as h:
            with pytest.raises(ValueError):
                result_view(h)[0] = 1.0

    def test_buffers_do_not_alias(self):  # test_core.py:80-84
        with handle_create(plan_create(2 ** 12, 2, workers=1)) as h:
            before = np.array(h.result)
            h.data[:] = 7.0
            assert np.array_equal(np.array(h.result), before)

    def test_input_preserved_and_result_correct(self):  # test_core.py:86-94
        n = 2 ** 12
        x = random_f32(n, seed=42)
        with handle_create(plan_create(n, 2, workers=2)) as h:
            h.data[:] = x
            out = h.run()
            assert np.array_equal(h.data, x)
            assert l2_norm(np.asarray(out, dtype=np.float64), packed_exact(x)) < 1e-6

    def test_reuse_without_reallocation(self):  # test_core.py:96-110
        n = 2 ** 10
        with handle_create(plan_create(n, 1, workers=2, test_mode=True)) as h:
            buf = h.data.ctypes.data
            first = None
            for _ in range(25):
                h.data[:] = random_f32(n, seed=1)
                h.run()
                if first is None:
                    first = np.array(h.result)
                assert np.array_equal(np.array(h.result), first)
            assert h.data.ctypes.data == buf

    def test_two_handles_are_independent(self):  # test_core.py:112-119
        p = plan_create(2 ** 10, 1, workers=1, test_mode=True)
        with handle_create(p) as h1, handle_create(p) as h2:
            h1.data[:] = 1.0
            h2.data[:] = 2.0
            assert not np.shares_memory(h1.data, h2.data)
            h1.run()
            assert np.all(h2.data == 2.0)

    def test_close_is_idempotent(self):  # test_core.py:121-124
        h = handle_create(plan_create(2 ** 10, 0, workers=2, test_mode=True))
        h.close()
        h.close()


# ---- reference pkg/tests/test_recombine.py::TestFullPipeline ----------------
class TestFullPipeline:
    @pytest.mark.parametrize("s", [0, 1, 2])
    def test_impulse_n16(self, s):  # test_recombine.py:146-155
        with handle_create(plan_create(16, s, workers=1, test_mode=True)) as h:
            h.data[:] = 0.0
            h.data[0] = 1.0
            out = np.array(h.run())
        expected = np.zeros(16, dtype=np.float32)
        expected[0] = expected[1] = 1.0
        expected[2::2] = 1.0
        assert np.allclose(out, expected, atol=1e-6)

    def test_ramp_n8_s1(self):  # test_recombine.py:157-161
        with handle_create(plan_create(8, 1, workers=1, test_mode=True)) as h:
            h.data[:] = np.arange(1, 9, dtype=np.float32)
            out = np.array(h.run())
        assert np.allclose(out, [36, -4, -4, 9.6569, -4, 4, -4, 1.6569], atol=1e-3)

    def test_split_invariance(self):  # test_recombine.py:163-172
        n = 4096
        x = random_f32(n, seed=11)
        outs = []
        for s in range(int(math.log2(n)) - 1):
            with handle_create(plan_create(n, s, workers=2, test_mode=True)) as h:
                h.data[:] = x
                outs.append(np.array(h.run(), dtype=np.float64))
        for out in outs[1:]:
            assert l2_norm(out, outs[0]) <= 1e-6

    @pytest.mark.parametrize("workers", [1, 2, 4, 8])
    def test_bitwise_across_worker_counts(self, workers):  # test_recombine.py:174-183
        n, s = 1 << 14, 3
        x = random_f32(n, seed=12)
        with handle_create(plan_create(n, s, workers=1)) as h:
            h.data[:] = x
            reference = np.array(h.run())
        with handle_create(plan_create(n, s, workers=workers)) as h:
            h.data[:] = x
            assert np.array_equal(np.array(h.run()), reference)

    def test_hermitian_consistency(self):  # test_recombine.py:185-199
        n = 1 << 12
        x = random_f32(n, seed=13)
        with handle_create(plan_create(n, 3, workers=2)) as h:
            h.data[:] = x
            full = PermSpectrum(np.array(h.run(), dtype=np.float64)).to_full_complex()
        ks = np.random.default_rng(99).integers(0, n, size=64)
        exact = exact_coefficients(x, ks)
        scale = np.maximum(np.abs(exact), np.sqrt(np.mean(np.abs(exact) ** 2)))
        assert np.max(np.abs(full[ks] - exact) / scale) <= 1e-5


def test_entry_points_are_the_reference_names():
    """reference __init__.py: the transform-path names and the error module"""
    for name in ("plan_create", "handle_create", "run_transform", "data_view", "result_view", "PermSpectrum",
                 "TransformHandle", "TransformPlan", "build_scatter_index", "RunMetrics", "efficiency",
                 "flops_model", "pack_perm", "l2_norm", "errors"):
        assert hasattr(efft, name), name
    for name in ("EfftError", "SizeConstraintViolation", "BinsizeNotPowerOfTwo", "SplitsTooLarge", "SizeMismatch",
                 "AllocationFailure"):
        assert hasattr(efft.errors, name), name
    x = random_f32(64, seed=8)
    f = np.fft.fft(x.astype(np.float64))[:33]
    assert efft.l2_norm(efft.pack_perm(f), packed_exact(x)) < 1e-12
