"""The C-ABI library loads and exports every symbol include/efft_b200.h declares
(no compute calls without a GPU), and argument errors come back as status codes."""
import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_1409_5757_b200 import _native, errors

HEADER = os.path.join(ROOT, "include", "efft_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(efft_\w+)\s*\(", text, re.M)))


def test_header_declares_the_abi():
    names = declared_functions()
    assert "efft_plan_create" in names and "efft_execute" in names
    assert set(names) == set(_native.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.efft_version() == 1


def test_argument_errors_are_status_codes():
    lib = _native.load()
    h = ctypes.c_void_p()
    assert lib.efft_plan_create(None, 16, 1, -1, 0, 0) == 1
    assert lib.efft_plan_create(ctypes.byref(h), 16, 7, -1, 0, 0) == 1  # bad dtype
    assert b"dtype" in lib.efft_last_error()
    assert lib.efft_plan_create(ctypes.byref(h), 16, 1, 5, 0, 0) == 1  # bad direction
    assert lib.efft_plan_create(ctypes.byref(h), 0, 1, -1, 0, 0) == 1
    assert lib.efft_plan_create(ctypes.byref(h), 7, 3, -1, 0, 0) == 4  # odd real length
    assert lib.efft_execute(None, None, None, None) == 1
    assert lib.efft_plan_destroy(None) == 0


def test_status_mapping():
    with pytest.raises(errors.BinsizeNotPowerOfTwo):
        _native.check(4)
    with pytest.raises(errors.AllocationFailure):
        _native.check(5)
    with pytest.raises(errors.DeviceError):
        _native.check(8)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1409_5757_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "efft_oracle" not in text, f
