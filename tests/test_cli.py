"""CLI front end (paper_1409_5757_b200/cli.py) -- host-side logic, no GPU needed.

Mirrors the reference CLI tests (pkg/tests/test_cli.py): size parsing, the
stable CSV header, failure rows, raw-file validation and the independent
fp64 checker the `check` subcommand uses.
"""
import numpy as np
import pytest

from paper_1409_5757_b200 import cli
from paper_1409_5757_b200.metrics import CSV_HEADER


def test_parse_size_forms():
    assert cli.parse_size("4096") == 4096
    assert cli.parse_size("2^22") == 1 << 22
    assert cli.parse_size("3x2^28") == 3 << 28
    assert cli.parse_size("3*2^4") == 48
    with pytest.raises(ValueError):
        cli.parse_size("0")


def test_parse_int_list():
    assert cli.parse_int_list("2,3, 4") == [2, 3, 4]


def test_csv_header_extends_reference_schema():
    ref = "size,splits,workers,runtime_s,gflops,l2,mem_bytes,status"  # reference bench.py:21
    assert CSV_HEADER.startswith(ref)
    assert CSV_HEADER.split(",")[len(ref.split(",")):] == ["gbps", "roofline_frac", "ngpus", "dtype", "rt_err"]
    assert len(cli._failed(16, 2, 1, "complex64").split(",")) == len(CSV_HEADER.split(","))


def test_parser_subcommands():
    p = cli.build_parser()
    a = p.parse_args(["bench", "--size", "2^20", "--splits", "3", "--dtype", "complex64"])
    assert (a.cmd, a.size, a.splits, a.dtype, a.repeats) == ("bench", "2^20", 3, "complex64", cli.DEFAULT_REPEATS)
    a = p.parse_args(["scan", "--size", "4096", "--splits", "2,3"])
    assert a.splits == "2,3" and a.dtype == "float32"
    a = p.parse_args(["check", "--size", "4096", "--splits", "2", "--spot-checks", "8"])
    assert a.spot_checks == 8


def test_exact_dft_at_matches_numpy():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(3 * 512) + 1j * rng.standard_normal(3 * 512)
    ks = np.array([0, 1, 7, 1000, 1535])
    np.testing.assert_allclose(cli._exact_dft_at(x, ks, chunk=256), np.fft.fft(x)[ks], rtol=1e-12, atol=1e-10)


def test_raw_file_length_is_validated(tmp_path):
    p = tmp_path / "sig.bin"
    np.zeros(10, dtype="<f4").tofile(p)
    with pytest.raises(ValueError, match="short read"):
        cli._read_raw(str(p), 16, "float32")
    with pytest.raises(ValueError, match="trailing data"):
        cli._read_raw(str(p), 4, "float32")
    np.zeros(8, dtype="<c8").tofile(p)
    assert cli._read_raw(str(p), 8, "complex64").dtype == np.complex64


def test_bad_size_exits_nonzero(capsys):
    assert cli.main(["bench", "--size", "-5", "--splits", "2"]) == 1
    assert "error" in capsys.readouterr().err
