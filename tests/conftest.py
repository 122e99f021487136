import json
import os
import sys
from functools import lru_cache

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


@lru_cache(maxsize=None)
def golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


@lru_cache(maxsize=None)
def triangulations():
    return {t["name"]: t for t in golden("triangulations.json")}


def tri_from_fixture(t):
    from paper_2604_09221_b200.lattice import Triangulation, validate_triangulation

    edges = [((a, b), (c, e)) for a, b, c, e in t["edges"]]
    if t.get("unimodular", True) is None:
        return Triangulation(t["degree"], tuple(sorted(edges)), ())
    try:
        return validate_triangulation(t["degree"], edges, require_unimodular=t.get("unimodular", True))
    except Exception:
        return Triangulation(t["degree"], tuple(sorted(edges)), ())


def plan_dict(t):
    P = dict(t["plan"])
    P["degree"] = t["degree"]
    return P


@pytest.fixture
def rng():
    import random

    return random.Random(0xC0FFEE)
