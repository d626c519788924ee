"""The paper's CPU method (GMP), via ctypes -- TEST INFRASTRUCTURE / CPU CONTEXT ONLY.

arxiv 1910.04429 computes the hash with GMP calls:
mpz_import -> mpz_mul + mpz_add (mpz_addmul) -> mpz_fdiv_r_2exp (mod 2^n) ->
mpz_fdiv_q_2exp (>> n-r) -> mpz_export.  The paper's C source is not in the
reference, so this restates that call sequence against the system
libgmp.so.10 (GMP 6.3.0 in this image).  Used as an independent cross-check
of the oracle at large sizes and as the "paper's method" context row of
bench.py's CPU baseline; never on the product path.
"""
from __future__ import annotations

import ctypes
import ctypes.util
import os
from concurrent.futures import ThreadPoolExecutor


class _Mpz(ctypes.Structure):
    _fields_ = [("alloc", ctypes.c_int), ("size", ctypes.c_int), ("d", ctypes.c_void_p)]


_gmp = None


def _lib():
    global _gmp
    if _gmp is None:
        name = ctypes.util.find_library("gmp") or "libgmp.so.10"
        lib = ctypes.CDLL(name)
        P = ctypes.POINTER(_Mpz)
        sz, vp = ctypes.c_size_t, ctypes.c_void_p
        lib.__gmpz_init.argtypes = [P]
        lib.__gmpz_clear.argtypes = [P]
        lib.__gmpz_import.argtypes = [P, sz, ctypes.c_int, sz, ctypes.c_int, sz, vp]
        lib.__gmpz_export.argtypes = [vp, ctypes.POINTER(sz), ctypes.c_int, sz, ctypes.c_int, sz, P]
        lib.__gmpz_export.restype = vp
        lib.__gmpz_addmul.argtypes = [P, P, P]
        lib.__gmpz_fdiv_r_2exp.argtypes = [P, P, ctypes.c_ulong]
        lib.__gmpz_fdiv_q_2exp.argtypes = [P, P, ctypes.c_ulong]
        _gmp = lib
    return _gmp


def available() -> bool:
    try:
        _lib()
        return True
    except OSError:
        return False


def compress(x: bytes, c: bytes, d: bytes, n: int, r: int) -> bytes:
    """((c*x + d) mod 2^n) >> (n - r), LSF bytes in and out, the paper's GMP sequence."""
    lib = _lib()
    mx, mc, mt = _Mpz(), _Mpz(), _Mpz()
    for m in (mx, mc, mt):
        lib.__gmpz_init(ctypes.byref(m))
    try:
        lib.__gmpz_import(ctypes.byref(mx), len(x), -1, 1, 0, 0, x)
        lib.__gmpz_import(ctypes.byref(mc), len(c), -1, 1, 0, 0, c)
        lib.__gmpz_import(ctypes.byref(mt), len(d), -1, 1, 0, 0, d)
        lib.__gmpz_addmul(ctypes.byref(mt), ctypes.byref(mc), ctypes.byref(mx))  # t = d + c*x
        lib.__gmpz_fdiv_r_2exp(ctypes.byref(mt), ctypes.byref(mt), n)
        lib.__gmpz_fdiv_q_2exp(ctypes.byref(mt), ctypes.byref(mt), n - r)
        rb = (r + 7) // 8
        out = ctypes.create_string_buffer(rb + 8)
        cnt = ctypes.c_size_t(0)
        lib.__gmpz_export(out, ctypes.byref(cnt), -1, 1, 0, 0, ctypes.byref(mt))
        return out.raw[:rb]  # export writes cnt <= rb bytes, the rest stays zero
    finally:
        for m in (mx, mc, mt):
            lib.__gmpz_clear(ctypes.byref(m))


def compress_batch(xs, cs, ds, n: int, r: int, threads: int = 1) -> list[bytes]:
    """One block per task over `threads` threads (ctypes releases the GIL)."""
    with ThreadPoolExecutor(max(1, threads)) as ex:
        return list(ex.map(lambda t: compress(t[0], t[1], t[2], n, r), zip(xs, cs, ds)))
