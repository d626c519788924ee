"""The C-ABI library loads and exports every symbol include/pa_b200.h declares (no GPU calls)."""
import ctypes
import os
import re
import subprocess

from paper_1910_04429_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pa_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(pab_[a-z_0-9]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = _native.load()
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    # and the python binding types every one of them
    assert set(syms) == set(_native.SIGNATURES)


def test_dynamic_symbol_table():
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_sm100a_code_present():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_only_queries():
    lib = _native.load()
    assert lib.pab_version() == 100
    assert _native.max_bits() == 1 << 27
    assert _native.plan_info(10**6) == (16, 8, 8)
    assert _native.plan_info(10**7) == (20, 10, 10)
    assert _native.plan_info(10**8) == (23, 11, 12)
    assert _native.plan_info(4) == (6, 0, 6)
    assert lib.pab_hash_workspace_bytes(10**6, 1) > 6 * 4 * (1 << 16)
    assert lib.pab_hash_workspace_bytes(0, 1) == 0
    rc = lib.pab_plan_info(0, None, None, None)
    assert rc == _native.PAB_EINVAL
    assert b"block length" in lib.pab_last_error()
    assert lib.pab_plan_info((1 << 27) + 1, None, None, None) == _native.PAB_ERANGE
