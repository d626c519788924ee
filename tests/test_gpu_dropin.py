"""GPU parity of the drop-in's remaining entry points against the oracle:
pa_round (pkg/src/modpa/pa.py:193-217) and fused_mul_add
(pkg/src/modpa/bignum.py:234-238), at C1 (n = 10^6) and n = 10^7."""
import random

import pytest

import oracle
import paper_1910_04429_b200 as pab
from paper_1910_04429_b200 import workloads

pytestmark = pytest.mark.gpu

SIZES = [(1_000_000, 500_000, 0), (10_000_000, 2_000_000, 3)]


def _block(n, seed):
    x, c, d = workloads.block_inputs(n, seed)
    return x, c, d, pab.BitBlock(int.from_bytes(x, "little"), n), pab.HashSeed(
        c=pab.BigNat(int.from_bytes(c, "little")), d=pab.BigNat(int.from_bytes(d, "little")),
        alpha=n)


@pytest.mark.parametrize("n,r,seed", SIZES)
def test_pa_round_unenforced_matches_oracle(n, r, seed):
    x, c, d, blk, hs = _block(n, seed)
    out = pab.pa_round(blk, pab.PAParams(n=n, r=r), hs, enforce=False)
    assert out.n == r
    assert pab.export_block(out) == oracle.compress(x, c, d, n, r)


@pytest.mark.parametrize("n,r,seed", SIZES)
def test_pa_round_enforced_in_budget_matches_oracle(n, r, seed):
    # h_min = n, epsilon = 2^-64: r_max = n - 128 >= r, so the round runs
    x, c, d, blk, hs = _block(n, seed)
    params = pab.PAParams(n=n, r=r, epsilon=2.0**-64, h_min=float(n))
    out = pab.pa_round(blk, params, hs)
    assert pab.export_block(out) == oracle.compress(x, c, d, n, r)
    with pytest.raises(pab.SecurityBoundError) as exc:
        pab.pa_round(blk, pab.PAParams(n=n, r=n - 127, epsilon=2.0**-64, h_min=float(n)), hs)
    assert exc.value.r_max == n - 128


@pytest.mark.parametrize("n,r,seed", SIZES)
def test_fused_mul_add_matches_oracle(n, r, seed):
    _, _, _, blk, hs = _block(n, seed)
    got = pab.fused_mul_add(hs.d, hs.c, pab.BigNat(blk.value)).value
    assert got == oracle.mul(hs.c.value, blk.value) + hs.d.value
    # and the composition compress is defined by (pkg/src/modpa/pa.py:188-189)
    key = pab.shift_right(pab.mod_pow2(got, n), n - r).value
    assert key == pab.compress(blk, hs, r).value


def test_fused_mul_add_edges():
    rng = random.Random(17)
    w = (1 << 64) - 1
    assert pab.fused_mul_add(1, w, w).value == w * w + 1
    assert pab.fused_mul_add(0, 0, 12345).value == 0
    assert pab.fused_mul_add(77, 0, 12345).value == 77
    big = rng.getrandbits(3_000_000)
    assert pab.fused_mul_add(big, 3, 5).value == big + 15  # addend longer than the product
    for _ in range(20):
        acc = rng.getrandbits(rng.randrange(1, 200_000))
        a = rng.getrandbits(rng.randrange(1, 200_000))
        b = rng.getrandbits(rng.randrange(1, 200_000))
        assert pab.fused_mul_add(acc, a, b).value == acc + a * b
    # carry out of the top word of the product: (2^k - 1)^2 + 2^(2k) - 2^(k+1) + 1 = 2^(2k)
    k = 1 << 20
    m = (1 << k) - 1
    assert pab.fused_mul_add((1 << (2 * k)) - m * m, m, m).value == 1 << (2 * k)


def test_compress_over_int_digits_matches_oracle():
    # the drop-in compress hands CPython's 30-bit digits to the GPU (pab_hash_digits)
    # and gets the key back as digits: ragged n and r around digit and word edges,
    # operands with fewer digits than n needs (zero high digits), zero keys
    from paper_1910_04429_b200 import _native, _pyint

    if not _pyint.supported():
        pytest.skip("interpreter int layout not supported")
    rng = random.Random(23)
    cases = [(2049, 1), (2049, 2049), (2050, 30), (2100, 60), (4096, 31), (30_000, 29_999),
             (65_536, 32_768), (99_999, 12_345), (300_007, 150_001), (1_000_000, 900_000)]
    for n, r in cases:
        nb = (n + 7) // 8
        for kind in ("rand", "short", "zero_x", "identity"):
            x = rng.getrandbits(n)
            c = rng.getrandbits(n) | 1
            d = rng.getrandbits(n)
            if kind == "short":
                c, d = c & ((1 << 61) - 1) | 1, d & 0xFFFF
            elif kind == "zero_x":
                x, d = 0, 0
            elif kind == "identity":
                c, d = 1, 0
            got = _native.hash_ints(x, c, d, n, r)
            want = oracle.compress(x.to_bytes(nb, "little"), c.to_bytes(nb, "little"),
                                   d.to_bytes(nb, "little"), n, r)
            assert got == int.from_bytes(want, "little"), (n, r, kind)
            if kind == "identity" and r == n:
                assert got == x


def test_digit_path_in_the_three_prime_mode():
    # n beyond the five-prime bound (32-bit coefficients over three primes): the
    # Python-int digit path equals the byte path, itself pinned to the oracle in
    # test_gpu_configs (max sizes); ragged n and r around digit / word edges
    from paper_1910_04429_b200 import _native

    rng = random.Random(31)
    n = 121_295_104 + 1_000_003
    assert _native.plan_width(n) == (32, 3)
    x, c, d = rng.getrandbits(n), rng.getrandbits(n) | 1, rng.getrandbits(n)
    nb = (n + 7) // 8
    for r in (n, n - 29, 77_777_777):
        got = pab.compress(pab.BitBlock(x, n),
                           pab.HashSeed(c=pab.BigNat(c), d=pab.BigNat(d), alpha=n), r).value
        raw = _native.hash_host(x.to_bytes(nb, "little"), c.to_bytes(nb, "little"),
                                d.to_bytes(nb, "little"), n, r)
        assert got == int.from_bytes(raw, "little"), r
