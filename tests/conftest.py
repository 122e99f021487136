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


def plan_arrays_of(P):
    """PlanArrays from a fixture plan dict (degree included)."""
    import numpy as np

    from paper_2604_09221_b200.diamond import PlanArrays

    return PlanArrays(P["degree"], P["nv"], P["npts"], np.array(P["edge_u"], np.int32),
                      np.array(P["edge_v"], np.int32), np.array(P["src"], np.int32),
                      np.array(P["par"], np.uint8), np.array(P["used"], np.uint8),
                      np.array(P["ap_u"], np.int32), np.array(P["ap_v"], np.int32),
                      P["maxreg"])


def diff_triangulation(d, edges):
    from paper_2604_09221_b200.lattice import validate_triangulation

    return validate_triangulation(d, [((a, b), (c, e)) for a, b, c, e in edges])
