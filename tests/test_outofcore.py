"""Out-of-core (host-streamed) transform: block planning on CPU (no GPU needed)."""
import pytest

from paper_1409_5757_b200 import outofcore
from paper_1409_5757_b200.errors import BinsizeNotPowerOfTwo


def test_split_balanced_and_factor3_first():
    assert outofcore.split(1 << 30) == (1 << 15, 1 << 15)
    assert outofcore.split(1 << 31) == (1 << 15, 1 << 16)
    assert outofcore.split(3 << 28) == (3 << 14, 1 << 14)
    assert outofcore.split(5 << 20) == (5 << 10, 1 << 10)
    assert outofcore.split(7 << 20) == (7 << 10, 1 << 10)
    with pytest.raises(BinsizeNotPowerOfTwo):
        outofcore.split(9 << 20)
    with pytest.raises(BinsizeNotPowerOfTwo):
        outofcore.split(1 << 36)


@pytest.mark.parametrize("n,dtype,budget", [(1 << 30, "complex64", 1 << 30), (1 << 24, "complex128", 1 << 20),
                                            (3 << 20, "complex64", 1 << 18)])
def test_blocks_fit_budget_and_tile_the_array(n, dtype, budget):
    n1, n2, cb, rb = outofcore.plan_blocks(n, dtype, budget)
    e, f = outofcore.ELEM[dtype], outofcore.LANES[dtype]
    assert n1 * n2 == n
    assert n2 % cb == 0 and n1 % rb == 0 and cb % f == 0 and rb % f == 0
    assert 4 * n1 * cb * e <= max(budget, 4 * n1 * f * e)
    assert 4 * n2 * rb * e <= max(budget, 4 * n2 * f * e)


@pytest.mark.parametrize("n", [1 << 8, 1 << 20, 3 << 20, 5 << 21, 7 << 19, 1 << 30, 1 << 34])
@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
@pytest.mark.parametrize("budget", [1 << 16, 1 << 22, 1 << 30])
def test_python_mirror_matches_library_block_rule(n, dtype, budget):
    """outofcore.plan_blocks restates efft_outofcore_blocks (host-only query, no GPU)."""
    from paper_1409_5757_b200 import _native

    ndt = _native.EFFT_C64 if dtype == "complex64" else _native.EFFT_C128
    try:
        want = outofcore.plan_blocks(n, dtype, budget)
    except BinsizeNotPowerOfTwo:
        with pytest.raises(BinsizeNotPowerOfTwo):
            _native.outofcore_blocks(n, ndt, budget)
        return
    assert _native.outofcore_blocks(n, ndt, budget) == want
