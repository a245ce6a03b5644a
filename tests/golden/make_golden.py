"""Generate the golden fixtures that pin the oracle (run in the build container).

Imports the reference package read-only from /root/reference/pkg/src and
records, for seeded inputs:
  real_<n>.npz      : x (float32), the reference fast path output
                      (efft.run_transform, PERM float32) for splits 0..2, and
                      pack_perm(naive_dft(x)) (fp64 direct sum, oracle.py:65-76)
  complex_<n>.npz   : complex x (re/im float64) and the exact complex spectrum by
                      linearity, to_full_complex(pack_perm(naive_dft(re))) +
                      1j*to_full_complex(pack_perm(naive_dft(im))) (core.py:242-249);
                      for power-of-two n also the reference fast-path composition
                      of two real float32 transforms
  spot_c1.npz       : 16 spot coefficients of a 2^21 complex input, each from the
                      reference naive_dft_at (oracle.py:79-89) on re and im
The fixtures are committed; /root/reference is never read by the tests.
Usage: python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import efft  # noqa: E402  (the reference package)
from efft.core import PermSpectrum  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def random_f32(n, seed):  # pkg/tests/conftest.py:7-9
    rng = np.random.default_rng(seed)
    return rng.random(n, dtype=np.float32) - np.float32(0.5)


def ref_fast(x, splits):
    plan = efft.plan_create(x.shape[0], splits, workers=1, test_mode=True)
    with efft.handle_create(plan) as h:
        h.data[:] = x
        return np.array(efft.run_transform(h))


def full_exact(re):
    return PermSpectrum(efft.pack_perm(efft.naive_dft(re))).to_full_complex()


def main():
    for n in (256, 1024, 4096):
        x = random_f32(n, seed=7000 + n)
        outs = {f"ref_s{s}": ref_fast(x, s) for s in range(3)}
        np.savez_compressed(os.path.join(HERE, f"real_{n}.npz"), x=x,
                            naive=efft.pack_perm(efft.naive_dft(x)), **outs)
    for n in (1024, 3072, 4096):
        rng = np.random.default_rng(9000 + n)
        re = rng.standard_normal(n)
        im = rng.standard_normal(n)
        exact = full_exact(re) + 1j * full_exact(im)
        extra = {}
        if n & (n - 1) == 0:
            fr = PermSpectrum(ref_fast(re.astype(np.float32), 2).astype(np.float64)).to_full_complex()
            fi = PermSpectrum(ref_fast(im.astype(np.float32), 2).astype(np.float64)).to_full_complex()
            extra["ref_two_real"] = fr + 1j * fi
        np.savez_compressed(os.path.join(HERE, f"complex_{n}.npz"), x=re + 1j * im,
                            exact=exact, **extra)
    n = 1 << 21
    rng = np.random.default_rng(2021)
    re = rng.standard_normal(n)
    im = rng.standard_normal(n)
    ks = np.concatenate([[0, 1, n // 2, n - 1], np.random.default_rng(5).integers(0, n, 12)])
    vals = []
    for k in ks:
        k = int(k)
        if k <= n // 2:
            a, b = efft.naive_dft_at(re, k), efft.naive_dft_at(im, k)
        else:
            a = np.conj(efft.naive_dft_at(re, n - k))
            b = np.conj(efft.naive_dft_at(im, n - k))
        vals.append(a + 1j * b)
    np.savez_compressed(os.path.join(HERE, "spot_c1.npz"), seed=2021, ks=ks,
                        vals=np.array(vals))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
