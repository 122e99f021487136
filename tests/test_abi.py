"""The C-ABI library loads and exports every entry point include/tcg.h declares.

No compute calls: these run on the CPU-only build box too.  Without a GPU
the product path must fail loudly (no CPU fallback)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT


def _declared():
    with open(os.path.join(ROOT, "include", "tcg.h")) as fh:
        text = fh.read()
    decl = r"^(?:int|int64_t|double|const char \*)\s*\*?\s*(tcg_[a-z_0-9]+)\s*\("
    return sorted(set(re.findall(decl, text, flags=re.M)))


def test_library_exports_header_symbols():
    from paper_2604_09221_b200 import _lib

    L = _lib.load()
    names = _declared()
    assert len(names) >= 17
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_lib.EXPORTS)
    assert L.tcg_version().decode().startswith("tcg ")


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(ROOT, "paper_2604_09221_b200",
                                                                  "libtcg.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    from paper_2604_09221_b200 import Classifier, DeviceUnavailable, builtin, _lib

    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible; the loud-failure path is for GPU-less hosts")
    with pytest.raises(DeviceUnavailable):
        Classifier(builtin("delaunay-3"))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2604_09221_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                with open(os.path.join(dirpath, f)) as fh:
                    src = fh.read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src).replace("oracle_", ""), f


def test_kernel_kinds_match_header():
    """tcg_kernel_times fills TCG_NKINDS slots, named by the TCG_KT_* kinds."""
    from paper_2604_09221_b200 import _lib

    with open(os.path.join(ROOT, "include", "tcg.h")) as fh:
        text = fh.read()
    n = int(re.search(r"#define TCG_NKINDS (\d+)", text).group(1))
    kinds = dict((int(v), k.lower()) for k, v in re.findall(r"#define TCG_KT_([A-Z0-9_]+) (\d+)", text))
    assert len(_lib.KERNEL_KINDS) == n == len(kinds)
    for i, name in enumerate(_lib.KERNEL_KINDS):
        assert kinds[i] == name, (i, name, kinds[i])
