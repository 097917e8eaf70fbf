"""CPU checks of the C-ABI library: it builds for sm_100a, loads, and exports every symbol
include/octmg.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "octmg.h")


def _declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(octmg_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2604_18886_b200._build import build_library
    return build_library()


def test_header_declares_the_survey_calls():
    names = _declared()
    for n in ("octmg_build_tree", "octmg_setup_hierarchy", "octmg_apply", "octmg_vcycle", "octmg_pcg_solve"):
        assert n in names


def test_library_exports_every_declared_symbol(libpath):
    L = ctypes.CDLL(libpath)
    missing = [n for n in _declared() if not hasattr(L, n)]
    assert not missing, missing
    from paper_2604_18886_b200 import ABI_SYMBOLS
    assert sorted(ABI_SYMBOLS) == _declared()


def test_library_is_sm100a_only(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_version_and_error_without_gpu(libpath):
    from paper_2604_18886_b200 import lib
    assert b"sm_100a" in lib().octmg_version()
    assert isinstance(lib().octmg_last_error(), bytes)


def test_oracle_shares_no_code_with_cuda_path():
    orc = open(os.path.join(ROOT, "oracle", "octmg_oracle.cpp")).read()
    assert "octmg.h" not in orc and "octmg_internal" not in orc
    for f in os.listdir(os.path.join(ROOT, "paper_2604_18886_b200")):
        if f.endswith(".py"):
            src = open(os.path.join(ROOT, "paper_2604_18886_b200", f)).read()
            assert not re.search(r"^\s*(from|import)\s+oracle", src, flags=re.M), f
