"""Pins the CPU oracle (oracle/efft_oracle.c) to the reference.

* known-answer vectors copied from the reference's own tests
  (pkg/tests/test_leaf_dft.py:22-38, test_recombine.py:40-63,
  test_oracle.py:12-24, test_scatter.py:16-48);
* golden fixtures produced by importing the reference package
  (tests/golden/make_golden.py): the reference fast path and its fp64
  naive_dft / naive_dft_at on seeded inputs.
"""
import numpy as np
import pytest

import oracle
from conftest import golden, random_c


def perm_pack(full):
    """Complex spectrum of a real input -> reference PERM layout (core.py:10-15)."""
    m = full.shape[0]
    out = np.empty(m)
    out[0] = full[0].real
    out[1] = full[m // 2].real
    out[2::2] = full[1:m // 2].real
    out[3::2] = full[1:m // 2].imag
    return out


def real_fft(x, **kw):
    return oracle.transform(np.asarray(x, dtype=np.float64).astype(np.complex128), **kw)


# ---- reference known-answer tests ------------------------------------------
def test_leaf_impulse_m8():  # test_leaf_dft.py:22-24
    assert np.allclose(perm_pack(real_fft([1, 0, 0, 0, 0, 0, 0, 0])), [1, 1, 1, 0, 1, 0, 1, 0])


def test_leaf_constant_m8():  # test_leaf_dft.py:27-29
    assert np.allclose(perm_pack(real_fft(np.ones(8))), [8, 0, 0, 0, 0, 0, 0, 0], atol=1e-12)


def test_leaf_ramp_m8():  # test_leaf_dft.py:32-38
    out = perm_pack(real_fft(np.arange(1.0, 9.0)))
    assert np.allclose(out, [36, -4, -4, 9.6569, -4, 4, -4, 1.6569], atol=1e-3)


def test_merge_m2_example():  # test_recombine.py:40-52: packed DFT of [1,2,3,4]
    assert np.allclose(perm_pack(real_fft([1.0, 2.0, 3.0, 4.0])), [10, -2, -2, 2], atol=1e-12)


def test_merge_halves_of_ramp():  # test_recombine.py:54-63
    assert np.allclose(perm_pack(real_fft([1.0, 3.0, 5.0, 7.0])), [16, -4, -4, 4], atol=1e-12)
    assert np.allclose(perm_pack(real_fft([2.0, 4.0, 6.0, 8.0])), [20, -4, -4, 4], atol=1e-12)


def test_naive_ramp():  # test_oracle.py:20-24
    f = real_fft([1.0, 2.0, 3.0, 4.0])
    assert np.allclose(f[:3], [10, -2 + 2j, -2], atol=1e-12)


def test_scatter_index_examples():  # test_scatter.py:16-19
    assert [oracle.bitrev(j, 2) for j in range(4)] == [0, 2, 1, 3]
    assert [oracle.bitrev(j, 3) for j in range(8)] == [0, 4, 2, 6, 1, 5, 3, 7]


@pytest.mark.parametrize("n,s", [(16, 0), (16, 1), (16, 2)])
def test_impulse_pipeline(n, s):  # test_recombine.py:136-146
    x = np.zeros(n)
    x[0] = 1
    assert np.allclose(real_fft(x, splits=s), np.ones(n), atol=1e-15)


# ---- golden fixtures from the reference package ------------------------------
@pytest.mark.parametrize("n", [256, 1024, 4096])
def test_real_fixture_vs_reference(n):
    g = golden(f"real_{n}.npz")
    for s in range(3):
        ours = perm_pack(real_fft(g["x"], splits=s))
        # the exact fp64 direct sum of the reference (oracle.py:65-76)
        assert oracle.rel_l2(ours, g["naive"]) < 1e-13
        # the reference's own float32 fast path agrees to its 1e-6 criterion
        assert oracle.rel_l2(ours, g[f"ref_s{s}"].astype(np.float64)) < 1e-6


@pytest.mark.parametrize("n", [1024, 3072, 4096])
@pytest.mark.parametrize("splits", [0, 2, 5])
def test_complex_fixture_vs_reference_linearity(n, splits):
    g = golden(f"complex_{n}.npz")
    ours = oracle.transform(g["x"], splits=splits)
    assert oracle.rel_l2(ours, g["exact"]) < 1e-13
    if "ref_two_real" in g:
        # the reference's float32 two-real composition
        assert oracle.rel_l2(ours, g["ref_two_real"]) < 1e-6


def test_c1_spot_checks_vs_reference_naive_dft_at():
    g = golden("spot_c1.npz")
    n = 1 << 21
    rng = np.random.default_rng(int(g["seed"]))
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y = oracle.transform(x)
    exact = g["vals"]
    scale = np.maximum(np.abs(exact), np.sqrt(np.mean(np.abs(exact) ** 2)))
    err = np.max(np.abs(y[g["ks"]] - exact) / scale)
    assert err < 1e-12
    # and the oracle's own O(N) direct sum agrees with the reference's
    d = oracle.dft_at(x, g["ks"][:4])
    assert np.max(np.abs(d - exact[:4]) / scale[:4]) < 1e-12


# ---- self-consistency -------------------------------------------------------
@pytest.mark.parametrize("n", [8, 96, 1024, 3 * 2 ** 12, 2 ** 16, 5, 40, 5 * 2 ** 12, 7 * 2 ** 10])
def test_roundtrip_and_numpy(n):
    x = random_c(n, seed=n)
    y = oracle.transform(x)
    assert oracle.rel_l2(y, np.fft.fft(x)) < 1e-14
    assert oracle.rel_l2(oracle.transform(y, direction=1), x) < 1e-14


def test_split_invariance():  # test_recombine.py:154-163
    x = random_c(2 ** 12, seed=3)
    outs = [oracle.transform(x, splits=s) for s in range(0, 8)]
    for o in outs[1:]:
        assert oracle.rel_l2(o, outs[0]) < 1e-14


def test_c64_reference_precision_path():
    x = random_c(2 ** 14, seed=5)
    y = oracle.transform(x, precision="c64")
    assert oracle.rel_l2(y, np.fft.fft(x)) < 1e-6


def test_pass_primitive_matches_transform():
    # one column pass + one row pass with the four-step twiddle = the full DFT
    n1, n2 = 16, 32
    n = n1 * n2
    x = random_c(n, seed=11)
    tmp = np.empty(n, dtype=np.complex128)
    out = np.empty(n, dtype=np.complex128)
    # pass 1: for column j < n2: DFT_n1 over r of x[j + r*n2], twiddle W_N^(j*k) after
    # expressed as DIT on pass 2: out[j + k*n1]...
    oracle.pass_c128(x, tmp, length=n1, cols=n2, batch=1, in_col=1, in_stride=n2, in_batch=0,
                     out_col=n1, out_stride=1, out_batch=0)
    oracle.pass_c128(tmp, out, length=n2, cols=n1, batch=1, in_col=1, in_stride=n1, in_batch=0,
                     out_col=1, out_stride=n1, out_batch=0, tw_mod=n, tw_col=1)
    assert oracle.rel_l2(out, np.fft.fft(x)) < 1e-14
