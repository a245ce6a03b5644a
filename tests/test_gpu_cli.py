"""CLI subcommands on the B200 (bench / check / scan / transform rows)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1409_5757_b200 import cli  # noqa: E402
from paper_1409_5757_b200.metrics import CSV_HEADER  # noqa: E402


def rows(out):
    lines = [l for l in out.strip().splitlines() if not l.startswith("#")]
    assert lines[0] == CSV_HEADER
    hdr = CSV_HEADER.split(",")
    return [dict(zip(hdr, l.split(","))) for l in lines[1:]]


@pytest.mark.parametrize("dtype", ["float32", "complex64", "complex128"])
def test_check_ok(dtype, capsys):
    assert cli.main(["check", "--size", "2^16", "--splits", "3", "--dtype", dtype]) == 0
    (r,) = rows(capsys.readouterr().out)
    assert r["status"] == "ok" and float(r["l2"]) < 1e-4


def test_check_spot_mode_on_a_lean_size(capsys):
    assert cli.main(["check", "--size", "2^26", "--splits", "3", "--dtype", "complex128", "--spot-checks", "6"]) == 0
    (r,) = rows(capsys.readouterr().out)
    assert r["status"] == "ok"


def test_bench_and_scan_rows(capsys):
    assert cli.main(["bench", "--size", "2^22", "--splits", "3", "--dtype", "complex64", "--repeats", "2"]) == 0
    (r,) = rows(capsys.readouterr().out)
    assert float(r["gflops"]) > 0 and float(r["gbps"]) > 0 and r["dtype"] == "complex64"
    assert cli.main(["scan", "--size", "2^20", "--splits", "2,3,30", "--repeats", "1"]) == 1  # 30 splits invalid
    rs = rows(capsys.readouterr().out)
    assert [x["status"] for x in rs] == ["ok", "ok", "failed"]


def test_transform_file_roundtrip(tmp_path, capsys):
    n = 4096
    x = (np.random.default_rng(5).standard_normal(n) + 1j * np.random.default_rng(6).standard_normal(n))
    x = x.astype(np.complex128)
    src, dst = tmp_path / "in.bin", tmp_path / "out.bin"
    x.tofile(src)
    assert cli.main(["transform", "--size", str(n), "--splits", "2", "--dtype", "complex128",
                     "--input", str(src), "--output", str(dst)]) == 0
    y = np.fromfile(dst, dtype=np.complex128)
    assert np.linalg.norm(y - np.fft.fft(x)) / np.linalg.norm(np.fft.fft(x)) < 1e-12


def test_transform_out_of_core_option(tmp_path, capsys):
    n = 1 << 20
    x = (np.random.default_rng(7).standard_normal(n) + 1j * np.random.default_rng(8).standard_normal(n))
    src, dst = tmp_path / "in.bin", tmp_path / "out.bin"
    x.astype(np.complex128).tofile(src)
    assert cli.main(["transform", "--size", "2^20", "--splits", "2", "--dtype", "complex128",
                     "--input", str(src), "--output", str(dst), "--device-bytes", str(1 << 20)]) == 0
    y = np.fromfile(dst, dtype=np.complex128)
    ref = np.fft.fft(x)
    assert np.linalg.norm(y - ref) / np.linalg.norm(ref) < 1e-12


@pytest.mark.parametrize("dtype", ["float32", "complex64"])
def test_check_corrupt_fails_like_the_reference(dtype, capsys):
    """reference cli.py:125-150: --corrupt perturbs the result; status failed, exit 1"""
    assert cli.main(["check", "--size", "2^12", "--splits", "2", "--dtype", dtype, "--corrupt"]) == 1
    (r,) = rows(capsys.readouterr().out)
    assert r["status"] == "failed"


def test_check_reports_roundtrip_error(capsys):
    assert cli.main(["check", "--size", "2^20", "--splits", "3", "--dtype", "complex128"]) == 0
    (r,) = rows(capsys.readouterr().out)
    assert 0 <= float(r["rt_err"]) < 1e-13
