"""Stage-1 F-space compression (level2.cuh l15_build): with the free nodes
numbered by tile bit (host_plan.cuh), the B, A1 and A2 nodes are contiguous
and the compression is a shift (TileTables::l15sh); TCG_L15_LUT=1 forces the
byte lookup tables instead.  Both must give the same stage-1 records, hence
equal reports and equal pipeline statistics, on the cases of
test_gpu_superdedup (ragged ranges, random triangulations, even degree).
"""

import pytest

from test_gpu_superdedup import _run

pytestmark = pytest.mark.gpu


def test_l15_shift_equals_lookup_tables():
    shift = _run({})
    lut = _run({"TCG_L15_LUT": "1"})
    assert len(shift) == len(lut) > 0
    for a, b in zip(shift, lut):
        assert a == b, a[0]
