"""Separator-split sampling (split.cuh) against the flat sampler and the reference.

The split sampler classifies a draw on the graph of a separator's vertices
plus the same-sign components of the two sides, read from per-plan tables;
draws whose graph is too large or whose status is not OK go to the flat
classifier.  Its aggregate must equal the flat sampler's bit for bit
(counts, witnesses = smallest drawn m, oval histogram, failing draw and
status) -- the flat sampler being the one pinned to the reference's
sample_kernel slices (kernels.py:447-462) in test_gpu_parity.py.
"""

import os

import numpy as np
import pytest

from conftest import golden, plan_arrays_of, plan_dict, tri_from_fixture, triangulations

pytestmark = pytest.mark.gpu

SEED = 20260810


def _agg(plan, split, seed, k0, k1, nbits):
    plan.set_split(split)
    rc, bad, agg = plan.sample(seed, k0, k1, nbits)
    stats = plan.split_stats()
    hist, total, keys, counts, wits = agg.result()
    return (rc, bad, tuple(hist), total, tuple(keys), tuple(counts), tuple(wits)), stats


def _check(T, n, k0=1 << 30, seed=SEED, expect_split=True, min_fallback=0):
    from paper_2604_09221_b200 import Classifier
    from paper_2604_09221_b200.sweep import _domain_bits

    c = Classifier(T, device=0)
    nb = _domain_bits(T.degree, raw_space=False)
    a, st = _agg(c.native, True, seed, k0, k0 + n, nb)
    b, st_flat = _agg(c.native, False, seed, k0, k0 + n, nb)
    if expect_split:
        assert st[0] == 1 and st[1] == n, st
        assert st[2] >= min_fallback, st
    assert st_flat[1] == 0
    assert a == b
    assert a[0] == 0 and a[3] == n
    return st


@pytest.mark.parametrize("name", ["bowtie8", "delaunay-8", "fig2-middle8", "fig2-right8",
                                  "delaunay-9", "delaunay-7", "delaunay-6"])
def test_split_equals_flat_named(name):
    from paper_2604_09221_b200 import builtin

    st = _check(builtin(name), 1 << 20)
    # the contracted graph fits for almost every draw
    assert st[2] < (1 << 20) // 20, st


@pytest.mark.parametrize("name", ["random-8-0", "random-8-1", "random-8-2", "random-7-0",
                                  "random-6-1", "c4-7-3", "c4-7-11"])
def test_split_equals_flat_random_triangulations(name):
    T = tri_from_fixture(triangulations()[name])
    _check(T, 1 << 18, k0=12345)


def test_split_fallback_path_exact(monkeypatch):
    """A 40-node cap sends a large share of the draws to the flat list kernel;
    the merged aggregate is still the flat sampler's."""
    from paper_2604_09221_b200 import builtin

    monkeypatch.setenv("TCG_SPLIT_MAXNODES", "40")
    st = _check(builtin("bowtie8"), 1 << 19, min_fallback=1 << 14)
    assert st[2] < (1 << 19)


def test_split_reference_sample_slices():
    """The reference's own sample_kernel slices (d = 8) through the split path."""
    from paper_2604_09221_b200 import builtin, Classifier
    from paper_2604_09221_b200.sweep import sample_slice

    for s in golden("c5_sample_slices.json")["slices"]:
        T = builtin(s["name"])
        c = Classifier(T, device=0)
        c.native.set_split(True)
        rep = sample_slice(T, s["seed"], s["k0"], s["k1"], classifier=c)
        assert c.native.split_stats()[0] == 1
        assert list(rep.oval_histogram) == s["hist"], (s["name"], s["k0"])
        assert rep.scheme_map == {k: tuple(v) for k, v in s["schemes"].items()}


@pytest.mark.parametrize("idx", range(6))
def test_split_failure_status_and_draw(idx):
    """Garbage degree-7 plans: failing draws reach the flat kernel, which
    reports the same status and earliest failing draw as the flat sampler."""
    from paper_2604_09221_b200 import _lib

    e = golden("garbage_sweep.json")[idx]
    plan = _lib.NativePlan(plan_arrays_of(plan_dict(e)), 0)
    a, st = _agg(plan, True, 7, 0, 1 << 18, 33)
    b, _ = _agg(plan, False, 7, 0, 1 << 18, 33)
    assert a[:2] == b[:2] and a[0] != 0
    assert st[0] == 1 and st[2] > 0


def test_split_multi_launch_and_slices():
    """Ranges over several launches (2^26 draws each) and arbitrary slice
    boundaries merge to the same aggregate."""
    from paper_2604_09221_b200 import builtin, Classifier
    from paper_2604_09221_b200.sweep import sample_slice

    T = builtin("delaunay-8")
    c = Classifier(T, device=0)
    k0, k1 = (1 << 39) - (1 << 25), (1 << 39) + (1 << 26) + 12345
    whole = sample_slice(T, SEED, k0, k1, classifier=c)
    a = sample_slice(T, SEED, k0, k0 + 999_999, classifier=c)
    b = sample_slice(T, SEED, k0 + 999_999, k1, classifier=c)
    from paper_2604_09221_b200.sweep import merge

    assert merge(a, b).scheme_map == whole.scheme_map
    assert merge(a, b).oval_histogram == whole.oval_histogram
    c.native.set_split(False)
    flat = sample_slice(T, SEED, k0, k1, classifier=c)
    assert flat.scheme_map == whole.scheme_map and flat.oval_histogram == whole.oval_histogram
