"""Host-side plan validation: mirrors reference pkg/tests/test_core.py::TestPlanCreate
and the PermSpectrum contract (no GPU needed)."""
import numpy as np
import pytest

import paper_1409_5757_b200 as efft
from paper_1409_5757_b200 import errors
from paper_1409_5757_b200.core import PermSpectrum, plan_create
from paper_1409_5757_b200.metrics import RunMetrics, algorithmic_bytes, efficiency, flops_model


class TestPlanCreate:
    def test_derived_fields(self):
        plan = plan_create(2 ** 20, 4, workers=8)
        assert plan.bins == 16
        assert plan.binsize == 65536
        assert plan.i_tile == 16 and plan.k_tile == 64
        assert plan.dtype == "float32" and plan.direction == -1

    def test_size_constraint_enforced(self):
        with pytest.raises(errors.SizeConstraintViolation):
            plan_create(2 ** 10, 4, workers=1)

    def test_test_mode_relaxes_size_constraint(self):
        assert plan_create(2 ** 10, 4, workers=1, test_mode=True).binsize == 64

    def test_binsize_must_be_power_of_two_for_real_path(self):
        with pytest.raises(errors.BinsizeNotPowerOfTwo):
            plan_create(1536, 1, workers=1)

    def test_complex_accepts_three_times_power_of_two(self):
        # the paper's N = M x 2^s sizes; BASELINE config 4
        plan = plan_create(3 * 2 ** 28, 4, dtype="complex128")
        assert plan.binsize == 3 * 2 ** 24
        # radix 5 and 7
        assert plan_create(5 * 2 ** 20, 3, dtype="complex64").binsize == 5 * 2 ** 17
        assert plan_create(7 * 2 ** 20, 3, dtype="complex128").binsize == 7 * 2 ** 17
        with pytest.raises(errors.BinsizeNotPowerOfTwo):
            plan_create(9 * 2 ** 10, 1, dtype="complex64", test_mode=True)

    def test_binsize_minimum_holds_even_in_test_mode(self):
        assert plan_create(8, 1, workers=1, test_mode=True).binsize == 4
        with pytest.raises(errors.BinsizeNotPowerOfTwo):
            plan_create(8, 2, workers=1, test_mode=True)

    def test_splits_too_large(self):
        with pytest.raises(errors.SplitsTooLarge):
            plan_create(16, 5, workers=1, test_mode=True)

    def test_argument_validation(self):
        for bad in [dict(n=0, splits=0), dict(n=256, splits=-1), dict(n=256, splits=0, workers=0),
                    dict(n=256, splits=0, i_tile=0), dict(n=256, splits=0, dtype="int8"),
                    dict(n=256, splits=0, direction=2), dict(n=256, splits=0, dtype="float32",
                                                             direction=1)]:
            with pytest.raises(ValueError):
                plan_create(**bad)

    def test_deterministic_and_involution(self):
        a = plan_create(2 ** 12, 3, workers=2, test_mode=True)
        b = plan_create(2 ** 12, 3, workers=2, test_mode=True)
        assert np.array_equal(a.scatter_index, b.scatter_index)
        t = plan_create(2 ** 12, 5, workers=1, test_mode=True).scatter_index
        assert np.array_equal(t[t], np.arange(32))
        assert efft.build_scatter_index(3).tolist() == [0, 4, 2, 6, 1, 5, 3, 7]


class TestPermSpectrum:
    def test_layout_contract(self):
        x = np.random.default_rng(8).random(64) - 0.5
        f = np.fft.fft(x)[:33]
        packed = np.empty(64)
        packed[0], packed[1] = f[0].real, f[32].real
        packed[2::2], packed[3::2] = f[1:32].real, f[1:32].imag
        sp = PermSpectrum(packed)
        assert sp.dc == pytest.approx(f[0].real)
        assert sp.nyquist == pytest.approx(f[32].real)
        for k in range(64):
            exp = f[k] if k <= 32 else np.conj(f[64 - k])
            assert sp.coefficient(k) == pytest.approx(complex(exp), abs=1e-12)
        assert np.allclose(sp.to_full_complex(), np.fft.fft(x), atol=1e-12)

    def test_index_errors(self):
        sp = PermSpectrum(np.zeros(8, dtype=np.float32))
        with pytest.raises(errors.IndexOutOfRange):
            sp.coefficient(8)
        with pytest.raises(ValueError):
            PermSpectrum(np.zeros(7, dtype=np.float32))


class TestMetrics:
    def test_flop_models(self):
        assert flops_model(8) == 2.5 * 8 * 3
        assert flops_model(8, complex_input=True) == 5 * 8 * 3
        with pytest.raises(errors.NonPositiveSize):
            flops_model(0)

    def test_bytes_and_rows(self):
        assert algorithmic_bytes(2 ** 30, 8, 2) == 2 * 2 * 2 ** 30 * 8
        m = RunMetrics.from_timing(2 ** 20, 0, 1, 0.5)
        assert m.gflops == pytest.approx(5 * 2 ** 20 * 20 / 0.5 / 1e9)
        assert len(m.csv_row().split(",")) == 13
        assert efficiency({1: 2.0, 2: 3.0})[2] == pytest.approx(0.75)
        with pytest.raises(errors.MissingBaseline):
            efficiency({2: 1.0})
