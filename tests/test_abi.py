"""The C-ABI library builds for sm_100a, loads, and exports every symbol that
include/s3r.h declares (no compute calls: this runs without a GPU)."""
import os
import re
import subprocess

import pytest

from paper_2503_08217_b200 import build as B
from paper_2503_08217_b200 import s3r

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "s3r.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(s3r_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return s3r.lib()


def test_header_and_binding_agree():
    assert declared_functions() == sorted(s3r.EXPORTS)


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", B.OUT], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (s3r_[a-z_]+)$", out, flags=re.M))
    for name in declared_functions():
        assert name in exported, name
        assert getattr(lib, name) is not None


def test_sm100a_code_present(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", B.OUT], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_null_handling(lib):
    assert lib.s3r_version() == 10100
    assert lib.s3r_create(0, None) == s3r.S3R_EINVAL
    assert lib.s3r_render_batch(None, None, None, 0, None, None) == s3r.S3R_EINVAL
    assert lib.s3r_last_error(None) == b"null context"
    assert lib.s3r_set_debug(None, 1) == s3r.S3R_EINVAL
    assert lib.s3r_check(None, None) == s3r.S3R_EINVAL
    assert lib.s3r_set_capacity(None, None) == s3r.S3R_EINVAL
    assert lib.s3r_capacity_from_last(None, 1.0, None) == s3r.S3R_EINVAL


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2503_08217_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "s3r_oracle" not in txt, f
