"""Property-based GPU parity (hypothesis), in the style of the reference's own
property tests (pkg/tests/test_bignum.py:138-143, pkg/tests/test_pa.py round trips):
random block sizes, output lengths, operands and byte orders through the drop-in
API, checked against the direct formula y = ((c x + d) mod 2^n) >> (n - r) on
Python ints, and products / fused multiply-adds against a * b (+ acc)."""
import pytest
from hypothesis import HealthCheck, given, settings, strategies as st

import paper_1910_04429_b200 as pab
from paper_1910_04429_b200.bignum import WordOrder

pytestmark = pytest.mark.gpu

SETTINGS = dict(max_examples=150, deadline=None,
                suppress_health_check=[HealthCheck.too_slow, HealthCheck.data_too_large])


@st.composite
def hash_cases(draw):
    n = draw(st.one_of(st.integers(1, 70), st.integers(1, 5000), st.integers(2040, 2060),
                       st.integers(1, 300_000)))
    r = draw(st.integers(1, n))
    x = draw(st.integers(0, (1 << n) - 1))
    c = draw(st.integers(0, (1 << n) - 1)) | 1
    d = draw(st.integers(0, (1 << n) - 1))
    return n, r, x, c, d


@settings(**SETTINGS)
@given(hash_cases())
def test_compress_equals_direct_formula(case):
    n, r, x, c, d = case
    seed = pab.HashSeed(c=pab.BigNat(c), d=pab.BigNat(d), alpha=n)
    out = pab.compress(pab.BitBlock(x, n), seed, r)
    assert out.n == r and out.value == ((c * x + d) % (1 << n)) >> (n - r)


@settings(**SETTINGS)
@given(hash_cases(), st.sampled_from([WordOrder.LEAST_SIGNIFICANT_FIRST,
                                      WordOrder.MOST_SIGNIFICANT_FIRST]))
def test_serialized_round_equals_direct_formula(case, order):
    n, r, x, c, d = case
    raw = pab.export_block(pab.BitBlock(x, n), order)
    seed = pab.HashSeed(c=pab.BigNat(c), d=pab.BigNat(d), alpha=n)
    blk = pab.import_block(raw, n, order)
    key = pab.export_block(pab.pa_round(blk, pab.PAParams(n=n, r=r), seed, enforce=False), order)
    want = ((c * x + d) % (1 << n)) >> (n - r)
    assert key == pab.export_block(pab.BitBlock(want, r), order)


@settings(**SETTINGS)
@given(st.integers(0, (1 << 40_000) - 1), st.integers(0, (1 << 40_000) - 1),
       st.integers(0, (1 << 90_000) - 1))
def test_products_and_fused_mul_add(a, b, acc):
    assert pab.mul(a, b).value == a * b
    assert pab.fused_mul_add(acc, a, b).value == acc + a * b
