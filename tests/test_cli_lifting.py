"""CPU tests: CLI plumbing (exit codes, codecs) and the lifting generator."""

import json
import random

import pytest

from paper_2604_09221_b200 import builtin
from paper_2604_09221_b200.cli import main
from paper_2604_09221_b200.io import read_triangulation
from paper_2604_09221_b200.lifting import delaunay_lifting, from_lifting, random_unimodular


def run(capsys, *argv):
    code = main(list(argv))
    out = capsys.readouterr()
    return code, out.out, out.err


def test_export_builtin_roundtrip(capsys, tmp_path):
    path = tmp_path / "t.json"
    code, out, _ = run(capsys, "export-builtin", "bowtie8", str(path))
    assert code == 0 and out.strip() == str(path)
    assert read_triangulation(str(path)).edges == builtin("bowtie8").edges


def test_input_errors_exit_2(capsys, tmp_path):
    code, _, err = run(capsys, "classify", "000")  # neither file nor --builtin
    assert code == 2 and "error:" in err
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    code, _, err = run(capsys, "classify", str(bad), "000")
    assert code == 2


def test_budget_exit_4(capsys):
    code, _, err = run(capsys, "sweep", "--builtin", "delaunay-10")
    assert code in (2, 4)  # 4 with a GPU (budget); 2 when no device is visible


def test_lifting_generator():
    assert from_lifting(5, delaunay_lifting(5)).edges == builtin("delaunay-5").edges
    rng = random.Random(1)
    for d in (3, 5, 7):
        T = random_unimodular(d, rng)
        assert T.is_unimodular and T.degree == d
