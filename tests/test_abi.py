"""The C-ABI library loads and exports every symbol include/grace.h declares (CPU only).

No compute calls here: this box may have no GPU.  The binding's SIGNATURES
table must cover the header exactly, and the product package must not import
the oracle (the two share no code).
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "grace.h")


def _header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(grace_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1411_2565_b200 import LIB_PATH, build

    build.build()
    assert os.path.exists(LIB_PATH)
    return LIB_PATH


def test_header_declares_the_paper_call_list():
    fns = _header_functions()
    for name in ("grace_create", "grace_set_m", "grace_set_hext", "grace_heff", "grace_step", "grace_get_m",
                 "grace_destroy", "grace_last_error"):
        assert name in fns


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (grace_\w+)", out))
    missing = [f for f in _header_functions() if f not in exported]
    assert not missing, missing


def test_binding_loads_and_covers_header(lib_path):
    import paper_1411_2565_b200 as pb

    lib = pb.load()
    names = [s[0] for s in pb.SIGNATURES]
    assert sorted(names) == _header_functions()
    for n in names:
        assert hasattr(lib, n)
    assert pb.grace_last_error() == ""


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1411_2565_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, flags=re.M), f
                assert "oracle/" not in src.replace("oracle/ ", ""), f


def test_error_codes_match_header():
    import paper_1411_2565_b200 as pb

    text = open(HEADER).read()
    for name in ("GRACE_OK", "GRACE_EINVAL", "GRACE_ENOMEM", "GRACE_EZEROCELL", "GRACE_ENONFINITE", "GRACE_ECUDA",
                 "GRACE_EUNSUPPORTED"):
        v = int(re.search(name + r"\s*=\s*(-?\d+)", text).group(1))
        assert getattr(pb, name) == v
