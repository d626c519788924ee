"""Zero-conversion access to CPython int digits for the drop-in boundary.

The reference's data are Python ints (BitBlock.value, HashSeed.c/.d,
pkg/src/modpa/pa.py:44-83).  CPython stores an int's magnitude as 30-bit
digits in 32-bit slots, least significant first.  Instead of
int.to_bytes / int.from_bytes on the host (O(n) Python-level conversions
whose cost grows with r and dominates a GPU round at 10^6 bits), the drop-in
hands the digit arrays to the C ABI (pab_hash_digits), the GPU converts
digits <-> words, and the key is written into a freshly allocated int.

Layout (CPython 3.12, Include/cpython/longintrepr.h): PyObject header
(16 bytes), then `lv_tag` = ndigits << 3 | sign (0 positive, 1 zero, 2
negative), then the digits.  `supported()` is False on any other
interpreter layout, and callers then use the byte conversions instead.
"""
from __future__ import annotations

import ctypes
import platform
import sys

_TAG_OFF = 16
_DIGIT_OFF = 24
_SIGN_ZERO = 1

_ok = (platform.python_implementation() == "CPython" and sys.version_info[:2] == (3, 12)
       and sys.int_info.bits_per_digit == 30 and sys.int_info.sizeof_digit == 4
       and ctypes.sizeof(ctypes.c_void_p) == 8)
_new = None
if _ok:
    try:
        _new = ctypes.pythonapi._PyLong_New
        _new.restype = ctypes.py_object
        _new.argtypes = [ctypes.c_ssize_t]
    except AttributeError:  # pragma: no cover
        _ok = False


def _tag(v: int) -> int:
    return ctypes.c_size_t.from_address(id(v) + _TAG_OFF).value


def _check_layout() -> bool:
    probe = (1 << 95) | (5 << 30) | 7
    t = _tag(probe)
    if t != (4 << 3) or _tag(0) != _SIGN_ZERO:
        return False
    d = (ctypes.c_uint32 * 4).from_address(id(probe) + _DIGIT_OFF)
    return list(d) == [7, 5, 0, 1 << 5]


_ok = _ok and _check_layout()


def supported() -> bool:
    return _ok


def digits(v: int) -> tuple[int, int]:
    """(address of the digit array, digit count) of a nonnegative int.  The
    address is valid while the caller holds a reference to `v`."""
    t = _tag(v)
    if t & 3 == 2:
        raise ValueError("negative integer")
    return id(v) + _DIGIT_OFF, t >> 3


def new_uninit(nd: int) -> tuple[int, int]:
    """A new int with nd (>= 1) digit slots (contents undefined) and its digit address."""
    v = _new(nd)
    return v, id(v) + _DIGIT_OFF


def normalize(v: int, nd: int) -> int:
    """Finish an int filled by the GPU: drop zero high digits (CPython's
    invariant) and return it; 0 and 1-digit values come back as plain ints."""
    arr = (ctypes.c_uint32 * nd).from_address(id(v) + _DIGIT_OFF)
    k = nd
    while k and arr[k - 1] == 0:
        k -= 1
    if k <= 1:
        return int(arr[0]) if k else 0
    ctypes.c_size_t.from_address(id(v) + _TAG_OFF).value = k << 3
    return v


_BYTES_DATA_OFF = 32  # PyBytesObject: header (16) + ob_size (8) + ob_shash (8), then ob_sval
_bytes_new = None
if _ok:
    _bytes_new = ctypes.pythonapi.PyBytes_FromStringAndSize
    _bytes_new.restype = ctypes.py_object
    _bytes_new.argtypes = [ctypes.c_void_p, ctypes.c_ssize_t]


def to_bytes(v: int, nbytes: int, msf: bool = False) -> bytes:
    """int.to_bytes(nbytes, 'little' / 'big') for a value known to fit, written by
    pab_digits_to_bytes straight into a new bytes object."""
    from . import _native

    out = _bytes_new(None, nbytes)
    a, nd = digits(v)
    _native.check(_native.load().pab_digits_to_bytes(a, nd, id(out) + _BYTES_DATA_OFF, nbytes,
                                                    int(msf)))
    return out


def from_bytes(raw, msf: bool = False) -> int:
    """int.from_bytes(raw, 'little' / 'big') through pab_bytes_to_digits."""
    from . import _native

    nb = len(raw)
    nd = (8 * nb + 29) // 30
    if nd == 0:
        return 0
    if not isinstance(raw, bytes):
        raw = bytes(raw)
    v, a = new_uninit(nd)
    _native.check(_native.load().pab_bytes_to_digits(raw, nb, int(msf), a, nd))
    return normalize(v, nd)
