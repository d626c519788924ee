"""ctypes front-end of the C oracle (test infrastructure only)."""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "_build", "libmodpa_oracle.so")
_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def available() -> bool:
    return os.path.exists(LIB)


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = ctypes.CDLL(LIB)
        vp, u64 = ctypes.c_void_p, ctypes.c_uint64
        lib.oracle_compress.argtypes = [vp, vp, vp, u64, u64, ctypes.c_int, vp]
        lib.oracle_compress_batch.argtypes = [vp, vp, vp, u64, u64, ctypes.c_int, u64, vp,
                                              ctypes.c_int]
        lib.oracle_mul.argtypes = [vp, u64, vp, u64, vp]
        lib.oracle_plan.argtypes = [u64, ctypes.POINTER(ctypes.c_int)] + [ctypes.POINTER(u64)] * 3
        _lib = lib
    return _lib


def compress(x: bytes, c: bytes, d: bytes, n: int, r: int, msf: bool = False) -> bytes:
    """y = ((c*x + d) mod 2^n) >> (n - r) on serialized blocks (pa.py:175-190)."""
    out = ctypes.create_string_buffer((r + 7) // 8)
    rc = _load().oracle_compress(x, c, d, n, r, int(msf), out)
    if rc:
        raise ValueError("invalid geometry")
    return out.raw


def compress_batch(x: bytes, c: bytes, d: bytes, n: int, r: int, batch: int,
                   threads: int = 1, msf: bool = False) -> bytes:
    out = ctypes.create_string_buffer(batch * ((r + 7) // 8))
    rc = _load().oracle_compress_batch(x, c, d, n, r, int(msf), batch, out, threads)
    if rc:
        raise ValueError("invalid geometry")
    return out.raw


def mul(a: int, b: int) -> int:
    la = max(1, (a.bit_length() + 7) // 8)
    lb = max(1, (b.bit_length() + 7) // 8)
    out = ctypes.create_string_buffer(la + lb)
    _load().oracle_mul(a.to_bytes(la, "little"), la, b.to_bytes(lb, "little"), lb, out)
    return int.from_bytes(out.raw, "little")


def plan(n_bits: int) -> tuple[int, int, int, int]:
    """(k, N, M, Nprime) of the reference's SSA plan (ntt.py:90-108)."""
    k = ctypes.c_int()
    N, M, Np = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    _load().oracle_plan(n_bits, ctypes.byref(k), ctypes.byref(N), ctypes.byref(M), ctypes.byref(Np))
    return k.value, N.value, M.value, Np.value
