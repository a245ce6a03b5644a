"""Build-output guards (CPU): the lean kernels keep their register arrays in
registers.  A digit-reversal map the optimiser fails to fold turns every
register array into local memory (a 272-byte stack frame) and makes the lean
passes ~5x slower -- that happened once; this catches it from
the ptxas report of the last build without a GPU."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LOG = os.path.join(ROOT, "build", "obj", "lean.o.ptxas.log")


def _entries():
    if not os.path.exists(LOG):
        pytest.skip("no ptxas report (run __graft_entry__.build() first)")
    text = open(LOG).read()
    out = []
    for block in text.split("Compiling entry function '")[1:]:
        name = block.split("'")[0]
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", block)
        if m:
            out.append((name, int(m.group(1)), int(m.group(2))))
    return out


def test_lean_kernels_have_no_local_arrays():
    entries = _entries()
    lean = [e for e in entries if "lean_pass" in e[0] or "lean_pair" in e[0]]
    assert lean, "no lean kernels in the ptxas report"
    bad = [(n[:60], st, sp) for n, st, sp in lean if st > 64 or sp > 64]
    assert not bad, f"lean kernels with local-memory arrays or heavy spills: {bad}"
