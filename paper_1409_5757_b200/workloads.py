"""Seeded synthetic inputs for BASELINE.json's five configurations.

No public dataset is involved.  Inputs are generated with
torch generators on the target device (fast for 8-64 GiB arrays) from a
recorded seed; the oracle checks the very array the device transformed (copied
to the host), so parity never depends on two generators agreeing.

  C1  N = 2^21      complex128  re/im iid N(0,1)
  C2  N = 2^27      complex128  re/im iid N(0,1), forward then inverse
  C3  N = 2^30      complex64   re/im iid N(0,1)
  C4  N = 3*2^28    complex128  16 unit tones at distinct seeded integer
                                frequencies + complex noise with VARIANCE 0.01
                                per real component (std 0.1)
  C5  N = 2^32      complex128  re/im iid U(-1, 1), forward then inverse
  R24, R27, R30     float32     the reference's own workload (bench.py:109-136):
                                real input U[-0.5, 0.5), packed PERM output,
                                N = 2^24, 2^27, 2^30
"""

import math

DEFAULT_SEED = 12345  # reference bench.py:23

CONFIGS = {
    "c1": dict(n=1 << 21, dtype="complex128", kind="normal", roundtrip=False),
    "c2": dict(n=1 << 27, dtype="complex128", kind="normal", roundtrip=True),
    "c3": dict(n=1 << 30, dtype="complex64", kind="normal", roundtrip=False),
    "c4": dict(n=3 << 28, dtype="complex128", kind="tones", roundtrip=False),
    "c5": dict(n=1 << 32, dtype="complex128", kind="uniform", roundtrip=True),
    "r24": dict(n=1 << 24, dtype="float32", kind="uniform_half", roundtrip=False),
    "r27": dict(n=1 << 27, dtype="float32", kind="uniform_half", roundtrip=False),
    "r30": dict(n=1 << 30, dtype="float32", kind="uniform_half", roundtrip=False),
}

N_TONES = 16
NOISE_STD = 0.1  # variance 0.01 per real component


def seed_for(config: str) -> int:
    return DEFAULT_SEED + list(CONFIGS).index(config) + 1


def tone_frequencies(n: int, seed: int):
    """16 distinct integer frequencies in [0, n), drawn without replacement."""
    import numpy as np

    rng = np.random.default_rng(seed)
    freqs = set()
    while len(freqs) < N_TONES:
        freqs.add(int(rng.integers(0, n)))
    return sorted(freqs)


def make_input(n: int, dtype: str, kind: str, seed: int, device="cuda"):
    """Complex (or, for dtype float32, real) tensor of length n on `device` (torch)."""
    import torch

    if dtype == "float32":  # the reference's signal: U[-0.5, 0.5) float32 (bench.py:109-112)
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        return torch.rand(n, generator=g, device=device, dtype=torch.float32) - 0.5

    tdt = {"complex64": torch.complex64, "complex128": torch.complex128}[dtype]
    rdt = torch.float32 if dtype == "complex64" else torch.float64
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = torch.empty(n, dtype=tdt, device=device)
    ri = torch.view_as_real(out)
    chunk = 1 << 26
    for lo in range(0, n, chunk):
        hi = min(lo + chunk, n)
        part = ri[lo:hi]
        if kind == "normal":
            part.copy_(torch.randn(hi - lo, 2, generator=g, device=device, dtype=rdt))
        elif kind == "uniform":
            part.copy_(torch.rand(hi - lo, 2, generator=g, device=device, dtype=rdt) * 2 - 1)
        elif kind == "tones":
            part.copy_(torch.randn(hi - lo, 2, generator=g, device=device, dtype=rdt) * NOISE_STD)
        else:
            raise ValueError(kind)
    if kind == "tones":
        freqs = tone_frequencies(n, seed)
        for lo in range(0, n, chunk):
            hi = min(lo + chunk, n)
            idx = torch.arange(lo, hi, device=device, dtype=torch.int64)
            acc = torch.zeros(hi - lo, dtype=torch.complex128, device=device)
            for f in freqs:
                ph = (idx * f) % n  # exact integer phase
                ang = ph.to(torch.float64) * (2.0 * math.pi / n)
                acc += torch.polar(torch.ones_like(ang), ang)
            out[lo:hi] += acc.to(tdt)
    return out
