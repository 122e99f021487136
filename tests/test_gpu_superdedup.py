"""Super-tile deduplication (tiles.cuh k_super_dedup / k_super_prop): the
tiles of a super-tile whose super record equals an earlier one's are neither
built nor compared -- each joins its twin's tile group.  Reports (counts,
witnesses, histograms, statuses and failing indices) must equal the sweeps
without it (TCG_NO_SUPER_DEDUP=1), which tests/test_gpu_headline.py and
tests/test_gpu_parity.py pin to the oracle and the reference.
"""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

_SCRIPT = r'''
import json, sys
sys.path.insert(0, %r)
from paper_2604_09221_b200 import builtin, sweep, SweepRange, Classifier
from paper_2604_09221_b200.io import report_jsonl
from conftest import tri_from_fixture, triangulations
cases = [("delaunay-7", True, 3 << 30, (3 << 30) + (1 << 31) + 12345),   # ragged ends
         ("delaunay-7", True, 0, 1 << 33),
         ("c4-7-3", True, 1 << 33, (1 << 33) + (1 << 32)),
         ("random-7-1", True, 5 << 29, (5 << 29) + (1 << 31) - 777),
         ("bowtie8", False, 1 << 38, (1 << 38) + (1 << 33)),              # even degree, rep domain
         ("delaunay-6", True, 0, 1 << 28)]
out = []
for name, raw, a, b in cases:
    t = triangulations().get(name)
    T = tri_from_fixture(t) if t is not None else builtin(name)
    c = Classifier(T)
    r = sweep(T, SweepRange(a, b), raw_space=raw, classifier=c)
    out.append([name, report_jsonl(r), sorted(r.scheme_map.items()), list(r.oval_histogram),
                c.native.tile_stats()])
print(json.dumps(out))
''' % ROOT


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    env["PYTHONPATH"] = os.path.join(ROOT, "tests") + os.pathsep + env.get("PYTHONPATH", "")
    p = subprocess.run([sys.executable, "-c", _SCRIPT], env=env, capture_output=True, text=True,
                       timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("extra", [{}, {"TCG_TILE_MAXNODES": "44"}])
def test_super_dedup_reports_equal(extra):
    """With and without super-tile deduplication, on ragged ranges, random
    triangulations, even degree, and (TCG_TILE_MAXNODES=44) with many tiles
    whose contraction does not fit (never merged: their twins are copied)."""
    on = _run(dict(extra))
    off = _run(dict(extra, TCG_NO_SUPER_DEDUP="1"))
    for a, b in zip(on, off):
        assert a[0] == b[0]
        assert a[1] == b[1], a[0]  # report JSONL bytes
        assert a[2] == b[2] and a[3] == b[3], a[0]
        assert a[4][0] == b[4][0]  # tiles contracted


def test_super_dedup_failing_index():
    """Garbage degree-7 plans (rare classification failures inside deduplicated
    groups): the earliest failing index survives super-tile deduplication."""
    script = r'''
import json, sys
sys.path.insert(0, %r); sys.path.insert(0, %r)
from paper_2604_09221_b200 import _lib
from conftest import golden, plan_arrays_of, plan_dict
out = []
for e in golden("garbage_sweep.json"):
    plan = _lib.NativePlan(plan_arrays_of(plan_dict(e)), 0)
    rc, bad, _ = plan.sweep(e["raw"], e["start"], e["end"])
    out.append([rc, bad, e["status"], e["bad"]])
print(json.dumps(out))
''' % (ROOT, os.path.join(ROOT, "tests"))
    for extra in ({}, {"TCG_NO_SUPER_DEDUP": "1"}):
        env = dict(os.environ, **extra)
        p = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True,
                           text=True, timeout=900)
        assert p.returncode == 0, p.stderr[-3000:]
        for rc, bad, st, want in json.loads(p.stdout.strip().splitlines()[-1]):
            assert (rc, bad) == (st, want)
