"""Error-path and differential parity on the GPU, against reference fixtures.

* every classification status 1..8 (kernels.py:183-266) on bad plans,
  per patchwork, through the mask engine (`tcg_classify_batch`) or, for
  plans it rejects (an antipodal "pair" that is not (p, -p)), the generic
  engine (`tcg_large_classify`);
* the smallest failing index of sweeps over rare-failure degree-7 plans,
  through the default tile / level-2 pipeline (kernels.py:423-436);
* the reference's differential criterion (test_acceptance.py:144-160):
  25 random unimodular T x 10^4 signs for each degree 1..6.
"""

import numpy as np
import pytest

from conftest import diff_triangulation, golden, plan_arrays_of, plan_dict

pytestmark = pytest.mark.gpu


def test_every_status_matches_reference():
    from paper_2604_09221_b200 import _lib

    seen = set()
    for e in golden("status.json"):
        arr = plan_arrays_of(plan_dict(e))
        words = np.array([r[0] for r in e["rows"]], np.uint64)
        want = [r[1] for r in e["rows"]]
        if e["engine"] == "mask":
            _, _, _, st = _lib.NativePlan(arr, 0).classify_words(words)
        else:
            st, _, _ = _lib.NativeLarge(arr, 0).classify_rows(words.reshape(-1, 1))
        assert [int(s) for s in st] == want, e["name"]
        seen.update(want)
    assert seen == {1, 2, 3, 4, 5, 6, 7, 8}


def test_mask_engine_rejects_non_antipodal_pairs():
    from paper_2604_09221_b200 import _lib
    from paper_2604_09221_b200.errors import TcurvesError

    e = next(g for g in golden("status.json") if g["engine"] == "generic")
    with pytest.raises(TcurvesError):
        _lib.NativePlan(plan_arrays_of(plan_dict(e)), 0)


@pytest.mark.parametrize("idx", range(6))
def test_sweep_reports_smallest_failing_index(idx):
    """The first failure lies 4 K..760 K indices into a 2^20-index range, so
    it sits inside a deduplicated tile / level-2 group, not at its start."""
    from paper_2604_09221_b200 import _lib

    e = golden("garbage_sweep.json")[idx]
    plan = _lib.NativePlan(plan_arrays_of(plan_dict(e)), 0)
    rc, bad, _ = plan.sweep(e["raw"], e["start"], e["end"])
    assert (rc, bad) == (e["status"], e["bad"]), e["name"]
    # same answer from a sub-range that starts just before the failure
    rc2, bad2, _ = plan.sweep(e["raw"], e["bad"] - 1000, e["end"])
    assert (rc2, bad2) == (e["status"], e["bad"])
    # and a range that stops just before it is clean
    rc3, _, agg = plan.sweep(e["raw"], e["start"], e["bad"])
    assert rc3 == 0 and agg.result()[1] == e["bad"] - e["start"]


def test_differential_criterion_all_degrees():
    from paper_2604_09221_b200 import Classifier, scheme_from_key

    n = 0
    for g in golden("diff.json"):
        d = g["degree"]
        rows = np.array(g["rows"], dtype=np.int64)
        for k, edges in enumerate(g["triangulations"]):
            c = Classifier(diff_triangulation(d, edges), device=0)
            sel = rows[rows[:, 0] == k]
            keys, ov, nr, st = c.classify_words(sel[:, 1].astype(np.uint64))
            assert (st == 0).all()
            assert (ov.astype(np.int64) == sel[:, 3]).all() and (nr.astype(np.int64) == sel[:, 4]).all()
            names = [scheme_from_key(int(x), d % 2 == 1) for x in keys]
            assert names == [g["schemes"][i] for i in sel[:, 2]], (d, k)
            n += len(sel)
    assert n == 60_000
