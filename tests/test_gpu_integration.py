"""INTEGRATION.md's reference-side ctypes stub, run against the real
reference package (installed in baseline/_ref; skipped when absent).

The python code block of INTEGRATION.md is executed as-is in a namespace
that provides what the stub's module (tcurves/kernels_gpu.py) would import
from tcurves; its gpu_sweep() feeds the reference's own _finish (sweep.py:
183-195).  The resulting report must equal tcurves.sweep computed by the
reference itself on the CPU, JSONL / CSV bytes included."""

import os
import re
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _tcurves():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "tcurves")):
        pytest.skip("reference package not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tcg_numba")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import tcurves
    except Exception as exc:  # numba missing
        pytest.skip(f"tcurves not importable: {exc!r}")
    return tcurves


def _stub_namespace(tc):
    from paper_2604_09221_b200 import _lib

    with open(os.path.join(ROOT, "INTEGRATION.md")) as fh:
        text = fh.read()
    block = re.search(r"## ctypes stub.*?```python\n(.*?)```", text, re.S).group(1)
    block = block.replace('C.CDLL("libtcg.so")', "C.CDLL(LIBTCG)")
    import importlib

    ns = {"LIBTCG": _lib.LIB_PATH, "kernels": importlib.import_module("tcurves.kernels"),
          "InvariantViolation": tc.InvariantViolation}
    exec(compile(block, "INTEGRATION.md", "exec"), ns)
    return ns


@pytest.mark.parametrize("name,raw,a,b", [("delaunay-4", True, 0, 1 << 15),
                                          ("delaunay-5", False, 0, 1 << 18),
                                          ("delaunay-7", True, 123456789, 123456789 + (1 << 16))])
def test_stub_against_real_reference(name, raw, a, b):
    tc = _tcurves()
    import importlib

    from tcurves.io import histogram_csv, report_jsonl

    sweep_mod = importlib.import_module("tcurves.sweep")
    ns = _stub_namespace(tc)
    T = tc.builtin(name)
    c = tc.Classifier(T)
    schemes, hist, total = ns["gpu_sweep"](c, raw, a, b)
    params = {"mode": "sweep", "start": a, "end": b, "raw_space": raw}
    gpu = sweep_mod._finish(T, raw, schemes, hist, total, params)
    cpu = tc.sweep(T, tc.SweepRange(a, b), raw_space=raw, classifier=c, workers=4)
    assert gpu == cpu
    assert report_jsonl(gpu) == report_jsonl(cpu)
    assert histogram_csv(gpu) == histogram_csv(cpu)
