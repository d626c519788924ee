"""ctypes binding of the C ABI declared in include/pa_b200.h.

The library is built in-tree (``paper_1910_04429_b200/_lib/libpa_b200.so``,
see csrc/Makefile and ``__graft_entry__.build``).  There is no CPU fallback:
if the library is missing or CUDA is unavailable every entry point raises.
Error codes map onto the reference's Python conventions: PAB_EINVAL and
PAB_ERANGE -> ValueError, PAB_ENOMEM -> MemoryError (what
``bench.run_bench`` catches, pkg/src/modpa/bench.py:162-173), anything else
-> RuntimeError.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PAB_LIB") or os.path.join(_HERE, "_lib", "libpa_b200.so")  # PAB_LIB: dev builds

PAB_OK = 0
PAB_EINVAL = -1
PAB_ENOMEM = -2
PAB_ECUDA = -3
PAB_ERANGE = -4
ORDER_LSF = 0
ORDER_MSF = 1

# name -> (restype, argtypes); every symbol include/pa_b200.h declares
_u8p = ctypes.c_void_p
SIGNATURES = {
    "pab_version": (ctypes.c_int, []),
    "pab_last_error": (ctypes.c_char_p, []),
    "pab_max_bits": (ctypes.c_uint64, []),
    "pab_plan_info": (ctypes.c_int, [ctypes.c_uint64] + [ctypes.POINTER(ctypes.c_int)] * 4),
    "pab_plan_width": (ctypes.c_int, [ctypes.c_uint64] + [ctypes.POINTER(ctypes.c_int)] * 2),
    "pab_force_coef_words": (None, [ctypes.c_int]),
    "pab_hash_workspace_bytes": (ctypes.c_size_t, [ctypes.c_uint64, ctypes.c_uint32]),
    "pab_hash_batch": (ctypes.c_int, [_u8p, _u8p, _u8p, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, _u8p,
                                      ctypes.c_uint64, _u8p, ctypes.c_size_t, _u8p]),
    "pab_hash_host": (ctypes.c_int, [_u8p, _u8p, _u8p, ctypes.c_uint64, ctypes.c_uint64,
                                     ctypes.c_uint32, ctypes.c_int, _u8p, ctypes.c_int]),
    "pab_hash_digits": (ctypes.c_int, [_u8p, ctypes.c_uint64, _u8p, ctypes.c_uint64, _u8p,
                                       ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _u8p,
                                       ctypes.c_uint64, ctypes.c_int]),
    "pab_digits_to_bytes": (ctypes.c_int, [_u8p, ctypes.c_uint64, _u8p, ctypes.c_uint64,
                                           ctypes.c_int]),
    "pab_bytes_to_digits": (ctypes.c_int, [_u8p, ctypes.c_uint64, ctypes.c_int, _u8p,
                                           ctypes.c_uint64]),
    "pab_hash_host_split": (ctypes.c_int, [_u8p, _u8p, _u8p, ctypes.c_uint64, ctypes.c_uint64,
                                           ctypes.c_uint32, ctypes.c_int, _u8p,
                                           ctypes.POINTER(ctypes.c_int), ctypes.c_int]),
    "pab_seed_expand": (ctypes.c_int, [_u8p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                                       ctypes.c_uint64, ctypes.c_int, _u8p, _u8p,
                                       ctypes.c_uint64, _u8p]),
    "pab_seed_expand_bench": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                                             ctypes.c_uint64, ctypes.c_int, _u8p, _u8p,
                                             ctypes.c_uint64, _u8p]),
    "pab_hash_seeded_host": (ctypes.c_int, [_u8p, ctypes.c_uint64, ctypes.c_uint64,
                                            ctypes.c_uint32, ctypes.c_int, _u8p, ctypes.c_uint64,
                                            ctypes.c_uint64, _u8p, ctypes.c_int]),
    "pab_hash_seeded_host_bench": (ctypes.c_int, [_u8p, ctypes.c_uint64, ctypes.c_uint64,
                                                  ctypes.c_uint32, ctypes.c_int, ctypes.c_uint64,
                                                  ctypes.c_uint64, _u8p, ctypes.c_int]),
    "pab_mul_workspace_bytes": (ctypes.c_size_t, [ctypes.c_uint64, ctypes.c_uint64]),
    "pab_mul": (ctypes.c_int, [_u8p, ctypes.c_uint64, _u8p, ctypes.c_uint64, _u8p, _u8p,
                               ctypes.c_size_t, _u8p]),
    "pab_mul_host": (ctypes.c_int, [_u8p, ctypes.c_uint64, _u8p, ctypes.c_uint64, _u8p,
                                    ctypes.c_int]),
    "pab_mul_add_workspace_bytes": (ctypes.c_size_t, [ctypes.c_uint64] * 3),
    "pab_mul_add": (ctypes.c_int, [_u8p, ctypes.c_uint64, _u8p, ctypes.c_uint64, _u8p,
                                   ctypes.c_uint64, _u8p, ctypes.c_uint64, _u8p, ctypes.c_size_t,
                                   _u8p]),
    "pab_mul_add_host": (ctypes.c_int, [_u8p, ctypes.c_uint64, _u8p, ctypes.c_uint64, _u8p,
                                        ctypes.c_uint64, _u8p, ctypes.c_uint64, ctypes.c_int]),
    "pab_profile_enable": (None, [ctypes.c_int]),
    "pab_profile_collect": (ctypes.c_int, [ctypes.POINTER(ctypes.c_char_p),
                                           ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_double), ctypes.c_int]),
}

_lib = None
_lock = threading.Lock()


class NativeUnavailable(RuntimeError):
    """The CUDA extension is missing or cannot run here (no CPU fallback)."""


def load() -> ctypes.CDLL:
    """Load the in-tree library (raises NativeUnavailable if it is not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                    " (there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def check(rc: int) -> None:
    if rc == PAB_OK:
        return
    msg = load().pab_last_error().decode(errors="replace")
    if rc in (PAB_EINVAL, PAB_ERANGE):
        raise ValueError(msg)
    if rc == PAB_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"CUDA error in pa_b200: {msg}")


def _device() -> int:
    import torch  # plumbing only: device selection follows torch's current device

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible (there is no CPU fallback)")
    return torch.cuda.current_device()


def hash_host(x: bytes, c: bytes, d: bytes, n: int, r: int, batch: int = 1,
              order: int = ORDER_LSF, device: int | None = None) -> bytes:
    """Hash `batch` blocks given as contiguous host byte strings; returns output bytes."""
    lib = load()
    dev = _device() if device is None else device
    out = ctypes.create_string_buffer(batch * ((r + 7) // 8))
    check(lib.pab_hash_host(x, c, d, n, r, batch, order, out, dev))
    return out.raw


def hash_ints(x: int, c: int, d: int, n: int, r: int, device: int | None = None) -> int:
    """The key of one block given as Python ints: digits in, digits out (pab_hash_digits);
    no int <-> bytes conversion on the host."""
    from . import _pyint

    lib = load()
    dev = _device() if device is None else device
    xa, xn = _pyint.digits(x)
    ca, cn = _pyint.digits(c)
    da, dn = _pyint.digits(d)
    ond = (r + 29) // 30
    out, oa = _pyint.new_uninit(ond)
    check(lib.pab_hash_digits(xa, xn, ca, cn, da, dn, n, r, oa, ond, dev))
    return _pyint.normalize(out, ond)


def hash_host_split(x: bytes, c: bytes, d: bytes, n: int, r: int, batch: int = 1,
                    order: int = ORDER_LSF, devices: list[int] | None = None) -> bytes:
    """As hash_host, with the NTT primes of the convolution split over `devices`
    (devices[0] does the CRT + carry); a device may repeat."""
    lib = load()
    devs = [_device()] if not devices else list(devices)
    arr = (ctypes.c_int * len(devs))(*devs)
    out = ctypes.create_string_buffer(batch * ((r + 7) // 8))
    check(lib.pab_hash_host_split(x, c, d, n, r, batch, order, out, arr, len(devs)))
    return out.raw


MAX_SEED_MATERIAL = 1024  # bytes of master seed material the device expander takes


def seed_material(rng_seed) -> bytes:
    """Seed material bytes exactly as _expand reads them (pkg/src/modpa/pa.py:141-146)."""
    if isinstance(rng_seed, int):
        if rng_seed < 0:
            raise ValueError("integer seed material must be nonnegative")
        return rng_seed.to_bytes(max(1, (rng_seed.bit_length() + 7) // 8), "little")
    return bytes(rng_seed)


def seed_material_fits(rng_seed) -> bool:
    """The material fits the device expander's kernel parameter (MAX_SEED_MATERIAL bytes)."""
    try:
        return len(seed_material(rng_seed)) <= MAX_SEED_MATERIAL
    except (TypeError, ValueError):
        return False


def hash_seeded_host(x: bytes, n: int, r: int, batch: int, rng_seed, first_index: int = 0,
                     order: int = ORDER_LSF, device: int | None = None) -> bytes:
    """run_pa's per-block step for `batch` contiguous blocks: x from the host, each block's
    (c, d) = gen_seed(n, derive_block_seed(rng_seed, first_index + j)) derived on the GPU."""
    lib = load()
    dev = _device() if device is None else device
    m = seed_material(rng_seed)
    out = ctypes.create_string_buffer(batch * ((r + 7) // 8))
    check(lib.pab_hash_seeded_host(x, n, r, batch, order, m, len(m), first_index, out, dev))
    return out.raw


def mul_host(a: bytes, b: bytes, device: int | None = None) -> bytes:
    lib = load()
    dev = _device() if device is None else device
    out = ctypes.create_string_buffer(len(a) + len(b))
    check(lib.pab_mul_host(a, len(a), b, len(b), out, dev))
    return out.raw


def mul_add_host(acc: bytes, a: bytes, b: bytes, device: int | None = None) -> bytes:
    """acc + a*b over LSF byte strings, max(len(a) + len(b), len(acc)) + 1 bytes."""
    lib = load()
    dev = _device() if device is None else device
    ob = max(len(a) + len(b), len(acc)) + 1
    out = ctypes.create_string_buffer(ob)
    check(lib.pab_mul_add_host(acc, len(acc), a, len(a), b, len(b), out, ob, dev))
    return out.raw


def plan_info(n: int) -> tuple[int, int, int, int]:
    """(radix m, lg, lg_rows, lg_cols): L = m * 2^lg, R = m * 2^lg_rows, C = 2^lg_cols."""
    lib = load()
    m, lg, lr, lc = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    check(lib.pab_plan_info(n, ctypes.byref(m), ctypes.byref(lg), ctypes.byref(lr),
                            ctypes.byref(lc)))
    return m.value, lg.value, lr.value, lc.value


def profile_enable(on: bool = True) -> None:
    """Record CUDA events around every kernel launch (see pab_profile_enable)."""
    load().pab_profile_enable(1 if on else 0)


def profile_collect() -> dict[str, tuple[int, float]]:
    """{kernel: (launches, total_ms)} since the last collect (synchronizes)."""
    cap = 32
    names = (ctypes.c_char_p * cap)()
    counts = (ctypes.c_int * cap)()
    ms = (ctypes.c_double * cap)()
    k = load().pab_profile_collect(names, counts, ms, cap)
    return {names[i].decode(): (counts[i], ms[i]) for i in range(k)}


def plan_width(n: int) -> tuple[int, int]:
    """(coefficient bits, NTT primes) of the convolution used for an n-bit hash."""
    lib = load()
    cb, np_ = ctypes.c_int(), ctypes.c_int()
    check(lib.pab_plan_width(n, ctypes.byref(cb), ctypes.byref(np_)))
    return cb.value, np_.value


def force_coef_words(words: int) -> None:
    """Test hook: force 1- or 2-word coefficients where valid (0 = automatic)."""
    load().pab_force_coef_words(int(words))


def max_bits() -> int:
    return int(load().pab_max_bits())
