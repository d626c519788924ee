"""Natural-number surface of the reference's ``modpa.bignum`` backed by the GPU.

Mirrors the names, argument meaning and error behaviour of
pkg/src/modpa/bignum.py so that callers (and the reference's own tests) can
switch modules.  The product ``mul`` (bignum.py:194-231) and
``fused_mul_add`` (bignum.py:234-238) run on the B200 through the C ABI
(``pab_mul_host``); ``alg`` and ``thresholds`` are accepted and ignored
because every route returns the identical exact product by contract
(bignum.py:197-201) -- the GPU's multi-prime NTT replaces all four.
``mod_pow2`` / ``shift_right`` are single bit-mask / shift operations on the
host int, exactly as in the reference (bignum.py:161-172); on the hash path
they are fused into the GPU carry kernel instead.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import Iterable, Union

from . import _native

WORD_BITS = 64
_WORD_MASK = (1 << WORD_BITS) - 1


class WordOrder(enum.Enum):
    """Word (or byte) significance order for import/export (bignum.py:27-31)."""

    MOST_SIGNIFICANT_FIRST = "msf"
    LEAST_SIGNIFICANT_FIRST = "lsf"


class MulAlgorithm(enum.Enum):
    """Route selector kept for API compatibility (bignum.py:34-39)."""

    SCHOOLBOOK = "schoolbook"
    KARATSUBA = "karatsuba"
    TOOM3 = "toom3"
    SSA = "ssa"
    AUTO = "auto"


@dataclass(frozen=True)
class ThresholdTable:
    """Size bands in 64-bit limbs (bignum.py:42-66); validated, then unused on the GPU."""

    schoolbook_max_limbs: int = 32
    karatsuba_max_limbs: int = 256
    toom3_max_limbs: int = 2048

    def __post_init__(self) -> None:
        if not (0 < self.schoolbook_max_limbs < self.karatsuba_max_limbs
                < self.toom3_max_limbs):
            raise ValueError(
                "thresholds must satisfy 0 < schoolbook < karatsuba < toom3, "
                f"got ({self.schoolbook_max_limbs}, {self.karatsuba_max_limbs}, "
                f"{self.toom3_max_limbs})")


DEFAULT_THRESHOLDS = ThresholdTable()


@dataclass(frozen=True)
class BigNat:
    """A nonnegative integer (bignum.py:69-105)."""

    value: int

    def __post_init__(self) -> None:
        if not isinstance(self.value, int) or isinstance(self.value, bool):
            raise TypeError(f"BigNat value must be int, got {type(self.value).__name__}")
        if self.value < 0:
            raise ValueError(f"BigNat must be nonnegative, got {self.value}")

    @property
    def bit_len(self) -> int:
        return self.value.bit_length()

    @property
    def limbs(self) -> tuple[int, ...]:
        return to_words(self, WordOrder.LEAST_SIGNIFICANT_FIRST)

    @property
    def limb_count(self) -> int:
        return (self.value.bit_length() + WORD_BITS - 1) // WORD_BITS

    def __int__(self) -> int:
        return self.value

    def __index__(self) -> int:
        return self.value

    def __repr__(self) -> str:
        return f"BigNat({self.value:#x})" if self.value else "BigNat(0)"


BigNatLike = Union[BigNat, int]


def _as_int(x: BigNatLike) -> int:
    v = x.value if isinstance(x, BigNat) else x
    if v < 0:
        raise ValueError(f"expected a nonnegative integer, got {v}")
    return v


def from_words(words: Iterable[int],
               order: WordOrder = WordOrder.LEAST_SIGNIFICANT_FIRST,
               word_bits: int = WORD_BITS) -> BigNat:
    """Assemble from fixed-width words (bignum.py:122-138)."""
    limit = 1 << word_bits
    seq = list(words)
    if order is WordOrder.MOST_SIGNIFICANT_FIRST:
        seq.reverse()
    acc = 0
    for pos, w in enumerate(seq):
        if not 0 <= w < limit:
            raise ValueError(f"word {w:#x} at position {pos} exceeds {word_bits} bits")
        acc |= w << (pos * word_bits)
    return BigNat(acc)


def to_words(x: BigNatLike,
             order: WordOrder = WordOrder.LEAST_SIGNIFICANT_FIRST,
             word_bits: int = WORD_BITS) -> tuple[int, ...]:
    """Decompose into fixed-width words, zero -> () (bignum.py:141-158)."""
    v = _as_int(x)
    if v == 0:
        return ()
    nwords = (v.bit_length() + word_bits - 1) // word_bits
    mask = (1 << word_bits) - 1
    out = tuple((v >> (i * word_bits)) & mask for i in range(nwords))
    if order is WordOrder.MOST_SIGNIFICANT_FIRST:
        out = out[::-1]
    return out


def mod_pow2(x: BigNatLike, k: int) -> BigNat:
    """x mod 2^k by masking (bignum.py:161-165)."""
    if k < 0:
        raise ValueError(f"bit count must be nonnegative, got {k}")
    return BigNat(_as_int(x) & ((1 << k) - 1))


def shift_right(x: BigNatLike, k: int) -> BigNat:
    """Floor division by 2^k (bignum.py:168-172)."""
    if k < 0:
        raise ValueError(f"bit count must be nonnegative, got {k}")
    return BigNat(_as_int(x) >> k)


def select_algorithm(n_bits_a: int, n_bits_b: int,
                     thresholds: ThresholdTable = DEFAULT_THRESHOLDS) -> MulAlgorithm:
    """Size-band dispatch of the reference (bignum.py:175-191), kept for reporting."""
    if n_bits_a < 0 or n_bits_b < 0:
        raise ValueError("bit lengths must be nonnegative")
    limbs = (max(n_bits_a, n_bits_b) + WORD_BITS - 1) // WORD_BITS
    if limbs <= thresholds.schoolbook_max_limbs:
        return MulAlgorithm.SCHOOLBOOK
    if limbs <= thresholds.karatsuba_max_limbs:
        return MulAlgorithm.KARATSUBA
    if limbs <= thresholds.toom3_max_limbs:
        return MulAlgorithm.TOOM3
    return MulAlgorithm.SSA


def mul(a: BigNatLike, b: BigNatLike,
        alg: MulAlgorithm = MulAlgorithm.AUTO,
        thresholds: ThresholdTable = DEFAULT_THRESHOLDS) -> BigNat:
    """Exact product a*b, computed on the GPU (bignum.py:194-231)."""
    av, bv = _as_int(a), _as_int(b)
    if not isinstance(alg, MulAlgorithm):
        raise ValueError(f"unknown algorithm {alg!r}")
    if av == 0 or bv == 0:
        return BigNat(0)
    la = (av.bit_length() + 7) // 8
    lb = (bv.bit_length() + 7) // 8
    raw = _native.mul_host(av.to_bytes(la, "little"), bv.to_bytes(lb, "little"))
    return BigNat(int.from_bytes(raw, "little"))


def fused_mul_add(acc: BigNatLike, c: BigNatLike, x: BigNatLike,
                  alg: MulAlgorithm = MulAlgorithm.AUTO,
                  thresholds: ThresholdTable = DEFAULT_THRESHOLDS) -> BigNat:
    """acc + c*x on the GPU (bignum.py:234-238): one call, the addend carried in
    the product's carry kernel (the hash's +d) instead of a host add."""
    av, cv, xv = _as_int(acc), _as_int(c), _as_int(x)
    if not isinstance(alg, MulAlgorithm):
        raise ValueError(f"unknown algorithm {alg!r}")
    if cv == 0 or xv == 0:
        return BigNat(av)
    nb = lambda v: (v.bit_length() + 7) // 8  # noqa: E731
    raw = _native.mul_add_host(av.to_bytes(nb(av), "little"), cv.to_bytes(nb(cv), "little"),
                               xv.to_bytes(nb(xv), "little"))
    return BigNat(int.from_bytes(raw, "little"))
