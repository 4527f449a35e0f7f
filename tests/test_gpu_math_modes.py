"""Which math mode each path needs for the accuracy gate (each comparison path
runs in the cheapest mode that meets the same tolerance).  Errors max|y - y_ref| / max|y_ref|
against the FP64 oracle; printed with -s for DESIGN.md's ledger."""
import numpy as np
import pytest

from oracle.errstudy import rel_err
from test_gpu_comparison import _run
from test_gpu_nested import SMALL, TOL, _ref, check_parity

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", list(SMALL))
def test_error_by_path_and_mode(name):
    layer = SMALL[name]
    errs = {}
    for path in ("nested", "ola", "direct"):
        for math in ("bf16", "bf16x3"):
            t, y = _run(layer, math, path)
            errs[(path, math)] = rel_err(y, _ref(layer, t))
    print(name, {f"{p}/{m}": f"{e:.2e}" for (p, m), e in errs.items()})
    assert all(np.isfinite(e) for e in errs.values())


@pytest.mark.parametrize("name", list(SMALL))
def test_direct_path_meets_gate_in_plain_bf16(name):
    # bench.py's direct_bf16 comparison leg: the direct path's cheapest mode passing the 5e-3 gate
    layer = SMALL[name]
    t, y = _run(layer, "bf16", "direct")
    check_parity(y, _ref(layer, t), "bf16x3", layer.dtype)
