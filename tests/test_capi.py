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
    assert lib.pab_version() == 102
    assert _native.max_bits() == 32 * ((5 * 2**22 + 1) // 2)
    # 64-bit coefficients over five primes (K' = ceil(n/64)), L = m * 2^lg >= 2K' - 1:
    # pow2 at 1e6 (32768), radix-5 at 1e7 (327680), radix-3 at 1e8 (3145728)
    assert _native.plan_info(10**6) == (1, 15, 7, 8)
    assert _native.plan_info(10**7) == (5, 16, 7, 9)
    assert _native.plan_info(10**8) == (3, 20, 8, 12)
    assert _native.plan_info(4) == (1, 6, 0, 6)
    # the five-prime CRT bound K' * (2^64-1)^2 < P ends at K' = 1,895,236; beyond it
    # 32-bit coefficients over three primes (2-adicity 22) reach 5 * 2^22
    for n in (1, 10**6, 10**8, 121_295_104):
        assert _native.plan_width(n) == (64, 5)
    for n in (121_295_105, _native.max_bits()):
        assert _native.plan_width(n) == (32, 3)
    for n in (1, 33, 2047, 2049, 65537, 131_072 * 32, 3 * 10**6, 5 * 10**7, 1 << 27,
              _native.max_bits()):
        m, lg, lr, lc = _native.plan_info(n)
        bits, primes = _native.plan_width(n)
        K = (n + bits - 1) // bits
        assert (m << lg) >= 2 * K - 1 and m in (1, 3, 5)
        assert lg <= (20 if primes == 5 else 22)
    _native.force_coef_words(1)
    try:
        assert _native.plan_width(10**6) == (32, 3)
        assert _native.plan_info(10**6) == (1, 16, 8, 8)
    finally:
        _native.force_coef_words(0)
    assert _native.plan_width(10**6) == (64, 5)
    assert lib.pab_hash_workspace_bytes(10**6, 1) > 10 * 4 * (1 << 15)
    assert lib.pab_hash_workspace_bytes(0, 1) == 0
    rc = lib.pab_plan_info(0, None, None, None, None)
    assert rc == _native.PAB_EINVAL
    assert b"block length" in lib.pab_last_error()
    assert lib.pab_plan_info(_native.max_bits() + 1, None, None, None, None) == _native.PAB_ERANGE
