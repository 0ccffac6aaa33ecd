"""The C-ABI library loads and exports every entry point include/hbk.h declares
(no GPU needed, no compute calls)."""
from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "hbk.h"
LIB = ROOT / "paper_1904_03329_b200" / "libhbk.so"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+char\*|int|void)\s+(hbk_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists():
        from paper_1904_03329_b200.build import build

        build()
    from paper_1904_03329_b200 import _native

    return _native.load_library()


def test_header_declares_entry_points():
    names = declared()
    assert len(names) >= 35
    for must in ("hbk_build_hbcsf", "hbk_split_fibers", "hbk_assign_slice_blocks", "hbk_plan_create",
                 "hbk_plan_execute", "hbk_coo_canonicalize", "hbk_coo_sort", "hbk_last_error"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (hbk_\w+)$", out, re.M))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    for n in declared():
        assert hasattr(lib, n)


def test_python_binding_covers_header(lib):
    from paper_1904_03329_b200 import _native

    assert sorted(_native.EXPORTED) == declared()


def test_abi_version_and_error_path(lib):
    from paper_1904_03329_b200 import _native

    assert lib.hbk_abi_version() == 1
    info = _native.CooInfo()
    st = lib.hbk_coo_info_get(None, C.byref(info))
    assert st == _native.HBK_EINVAL
    assert b"null" in lib.hbk_last_error()
    with pytest.raises(ValueError):
        _native.check(st)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
