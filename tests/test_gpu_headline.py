"""The bench's exact computation, pinned.

bench.py times config C3 as one sweep call over [0, 2^35) of delaunay-7's
raw space with the default pipeline (super-tiles, tile dedup, two-stage
level 2; one 2^35-index dedup window); N = 2 ranks sweep the 2^34-index
halves.  These tests check those very calls:

* against the per-patchwork full-diamond kernel (``TCG_NO_TILES=1``, the
  path the oracle pins pair by pair), in subprocesses, comparing the report
  JSONL bytes, histograms, counts and witnesses;
* against ``tests/golden/c3_full.json``, the complete C3 report computed by
  the pinned CPU oracle in 2^30-index pieces (make_c3_full.py), both piece
  by piece and merged per chunk (reference semantics: sweep.py:198-227,
  merge sweep.py:83-105).
"""

import json
import os
import subprocess
import sys

import pytest

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu

CHUNK = 1 << 34
C3_FULL = os.path.join(GOLDEN, "c3_full.json")

_SWEEP_CHUNKS = (
    "import json, sys; sys.path.insert(0, %r)\n"
    "from paper_2604_09221_b200 import builtin, sweep, SweepRange, Classifier, merge\n"
    "from paper_2604_09221_b200.io import report_jsonl, histogram_csv\n"
    "T = builtin('delaunay-7'); c = Classifier(T)\n"
    "halves = [sweep(T, SweepRange(a, a + (1 << 34)), raw_space=True, classifier=c)\n"
    "          for a in (0, 1 << 34)]\n"
    "out = [[report_jsonl(r), histogram_csv(r), sorted(r.scheme_map.items())] for r in halves]\n"
    "if len(sys.argv) > 1:  # the bench's call: the whole domain in one sweep\n"
    "    r = sweep(T, SweepRange(0, 1 << 35), raw_space=True, classifier=c)\n"
    "else:\n"
    "    r = merge(*halves)\n"
    "    r.params = {'mode': 'sweep', 'start': 0, 'end': 1 << 35, 'raw_space': True}\n"
    "out.append([report_jsonl(r), histogram_csv(r), sorted(r.scheme_map.items())])\n"
    "print(json.dumps(out))\n" % ROOT)


def _run(env_extra, whole=False, timeout=900):
    env = dict(os.environ, **env_extra)
    p = subprocess.run([sys.executable, "-c", _SWEEP_CHUNKS] + (["whole"] if whole else []),
                       env=env, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_bench_chunks_equal_per_patchwork_kernel():
    """The 2^34-index halves and the whole-domain sweep the bench times (one
    2^35-index dedup window) vs the per-patchwork kernel's halves, merged."""
    default = _run({}, whole=True)
    flat = _run({"TCG_NO_TILES": "1"})
    for k in range(3):
        assert default[k][0] == flat[k][0]  # report JSONL bytes (witness strings included)
        assert default[k][1] == flat[k][1]  # histogram CSV bytes
        assert default[k][2] == flat[k][2]  # scheme -> (count, witness index)


def _golden_pieces():
    if not os.path.exists(C3_FULL):
        pytest.skip("tests/golden/c3_full.json not generated")
    with open(C3_FULL) as fh:
        doc = json.load(fh)
    return {int(k): v for k, v in doc["pieces"].items()}, doc["piece_log2"]


def _merge(pieces):
    hist = [0] * len(pieces[0]["hist"])
    schemes = {}
    for p in pieces:
        hist = [a + b for a, b in zip(hist, p["hist"])]
        for s, (c, w) in p["schemes"].items():
            if s in schemes:
                schemes[s] = (schemes[s][0] + c, min(schemes[s][1], w))
            else:
                schemes[s] = (c, w)
    return hist, schemes


def test_c3_pieces_equal_oracle_golden():
    from paper_2604_09221_b200 import Classifier, SweepRange, builtin, sweep

    pieces, lg = _golden_pieces()
    T = builtin("delaunay-7")
    c = Classifier(T)
    for p, g in sorted(pieces.items()):
        r = sweep(T, SweepRange(g["start"], g["end"]), raw_space=True, classifier=c)
        assert list(r.oval_histogram) == g["hist"], p
        assert r.scheme_map == {s: tuple(v) for s, v in g["schemes"].items()}, p
        assert r.total_classified == g["end"] - g["start"] == 1 << lg


def test_c3_bench_chunks_equal_oracle_golden():
    from paper_2604_09221_b200 import Classifier, SweepRange, builtin, sweep

    pieces, lg = _golden_pieces()
    per = CHUNK >> lg
    T = builtin("delaunay-7")
    c = Classifier(T)
    done = 0
    for k in range(2):
        want = [pieces.get(k * per + i) for i in range(per)]
        if any(w is None for w in want):
            continue
        hist, schemes = _merge(want)
        r = sweep(T, SweepRange(k * CHUNK, (k + 1) * CHUNK), raw_space=True, classifier=c)
        assert list(r.oval_histogram) == hist
        assert r.scheme_map == schemes
        done += 1
    if done == 2:  # the bench's single whole-domain call
        hist, schemes = _merge([pieces[i] for i in range(2 * per)])
        r = sweep(T, SweepRange(0, 2 * CHUNK), raw_space=True, classifier=c)
        assert list(r.oval_histogram) == hist
        assert r.scheme_map == schemes
    if not done:
        pytest.skip("no complete 2^34 chunk in c3_full.json yet")
