"""The reference's own hash-path tests, run against the drop-in on the GPU.

`paper_1910_04429_b200.compat.install()` makes `import modpa` resolve to this
package (the module swap INTEGRATION.md §1 describes), and the cases below
restate the reference's hash-path tests against that name:

  pkg/tests/test_pa.py:125-193       TestCompress (KATs, identity member, exact
                                     output length, exhaustive alpha=6, primitive
                                     composition, route independence at 100,000
                                     bits, size mismatch, zero block)
  pkg/tests/test_pa.py:197-240       TestPaRound (parties agree, output length,
                                     r_max = 920 rejection / acceptance, budget
                                     needed for enforcement, geometry mismatches)
  pkg/tests/test_acceptance.py:96-128   the compress-correctness criterion:
                                     1,652,736 exhaustive/sampled compress calls
                                     in under 60 s
  pkg/tests/test_acceptance.py:214-246  the 10^6-bit round ceiling and the
                                     compression-ratio independence criterion
  pkg/tests/test_cli.py:113-155      run_pa == compress per block (LSF and MSF),
                                     budget enforcement, short input

Every compress / pa_round / run_pa call here goes through the CUDA path (the
drop-in has no CPU fallback).  /root/reference is not read: the expected
values are the reference tests' own closed forms and constants.
"""
import random
import statistics
import time

import pytest

import paper_1910_04429_b200.compat as compat

pytestmark = pytest.mark.gpu

compat.install()

from modpa import bench, pa  # noqa: E402  (the swapped-in package)
from modpa.bench import RunConfig, run_pa  # noqa: E402
from modpa.bignum import BigNat, MulAlgorithm, WordOrder  # noqa: E402
from modpa.bignum import fused_mul_add, mod_pow2, shift_right  # noqa: E402
from modpa.pa import BitBlock, HashSeed, PAParams, SecurityBoundError  # noqa: E402

LSF = WordOrder.LEAST_SIGNIFICANT_FIRST
MSF = WordOrder.MOST_SIGNIFICANT_FIRST


def member(c: int, d: int, alpha: int) -> HashSeed:
    return HashSeed(c=BigNat(c), d=BigNat(d), alpha=alpha)


def test_modpa_resolves_to_the_b200_package():
    import modpa

    import paper_1910_04429_b200

    assert modpa.__b200_dropin__ and pa is paper_1910_04429_b200.pa
    assert pa.compress is paper_1910_04429_b200.compress


# ---- pkg/tests/test_pa.py:125-193 (TestCompress) ---------------------------------

def test_worked_examples():
    # (3*5 + 1) mod 16 = 0 -> 0;  (5*7 + 2) mod 16 = 5 -> 5 >> 2 = 1
    out = pa.compress(BitBlock(5, 4), member(3, 1, 4), 2)
    assert (out.value, out.n) == (0, 2)
    out = pa.compress(BitBlock(7, 4), member(5, 2, 4), 2)
    assert (out.value, out.n) == (1, 2)


def test_identity_member_returns_the_block():
    rng = random.Random(3)
    for _ in range(50):
        x = BitBlock(rng.getrandbits(32), 32)
        assert pa.compress(x, member(1, 0, 32), 32).value == x.value


def test_output_has_exactly_r_bits():
    rng = random.Random(4)
    for _ in range(50):
        alpha = rng.randrange(2, 200)
        r = rng.randrange(1, alpha + 1)
        x = BitBlock(rng.getrandbits(alpha), alpha)
        assert pa.compress(x, pa.gen_seed(alpha, rng.randrange(1 << 30)), r).n == r


def test_exhaustive_alpha6_per_call():
    alpha, mask = 6, 63
    for beta in (1, 3, 6):
        for c in range(1, 64, 2):
            for d in range(64):
                s = member(c, d, alpha)
                for x in range(64):
                    got = pa.compress(BitBlock(x, alpha), s, beta).value
                    assert got == ((c * x + d) & mask) >> (alpha - beta), (beta, c, d, x)


def test_equals_primitive_composition():
    # compress == shift_right(mod_pow2(fused_mul_add(d, c, x), alpha), alpha - r)
    rng = random.Random(5)
    for _ in range(30):
        alpha = rng.randrange(8, 400)
        r = rng.randrange(1, alpha + 1)
        x = BitBlock(rng.getrandbits(alpha), alpha)
        s = pa.gen_seed(alpha, rng.randrange(1 << 30))
        manual = shift_right(mod_pow2(fused_mul_add(s.d, s.c, BigNat(x.value)), alpha), alpha - r)
        assert pa.compress(x, s, r).value == manual.value


def test_same_key_for_every_multiplication_route():
    rng = random.Random(6)
    alpha = 100_000
    x = BitBlock(rng.getrandbits(alpha), alpha)
    s = pa.gen_seed(alpha, 99)
    keys = {alg: pa.compress(x, s, alpha // 2, alg).value
            for alg in (MulAlgorithm.SCHOOLBOOK, MulAlgorithm.KARATSUBA, MulAlgorithm.TOOM3,
                        MulAlgorithm.SSA, MulAlgorithm.AUTO)}
    assert len(set(keys.values())) == 1
    c, d = s.c.value, s.d.value
    assert keys[MulAlgorithm.AUTO] == ((c * x.value + d) % (1 << alpha)) >> (alpha - alpha // 2)


def test_size_mismatches_raise():
    with pytest.raises(ValueError):
        pa.compress(BitBlock(1, 8), member(3, 1, 16), 4)
    with pytest.raises(ValueError):
        pa.compress(BitBlock(1, 8), member(3, 1, 8), 9)


def test_zero_block_zero_offset():
    assert pa.compress(BitBlock(0, 64), member(12345, 0, 64), 32).value == 0


# ---- pkg/tests/test_pa.py:197-240 (TestPaRound) ----------------------------------

def test_pa_round_parties_agree():
    rng = random.Random(7)
    n = 4096
    x = BitBlock(rng.getrandbits(n), n)
    params = PAParams(n=n, r=1024, epsilon=2**-40, h_min=2000.0)
    alice = pa.pa_round(x, params, pa.gen_seed(n, b"shared"))
    bob = pa.pa_round(x, params, pa.gen_seed(n, b"shared"))
    assert alice == bob
    s = pa.gen_seed(n, b"shared")
    assert alice.value == ((s.c.value * x.value + s.d.value) % (1 << n)) >> (n - 1024)


def test_pa_round_output_length():
    rng = random.Random(8)
    n = 10_000
    x = BitBlock(rng.getrandbits(n), n)
    out = pa.pa_round(x, PAParams(n=n, r=n // 2), pa.gen_seed(n, 3), enforce=False)
    assert out.n == n // 2


def test_pa_round_budget_bound():
    # h_min = 1000, epsilon = 2^-40: r_max = floor(1000 - 80) = 920
    n = 4096
    x = BitBlock(123, n)
    with pytest.raises(SecurityBoundError) as exc:
        pa.pa_round(x, PAParams(n=n, r=1000, epsilon=2**-40, h_min=1000.0), pa.gen_seed(n, 1))
    assert exc.value.r_max == 920 and exc.value.r == 1000
    out = pa.pa_round(x, PAParams(n=n, r=920, epsilon=2**-40, h_min=1000.0), pa.gen_seed(n, 1))
    assert out.n == 920


def test_pa_round_enforcement_needs_budget_and_geometry():
    with pytest.raises(ValueError, match="enforce"):
        pa.pa_round(BitBlock(1, 64), PAParams(n=64, r=32), pa.gen_seed(64, 1))
    params = PAParams(n=64, r=32, epsilon=0.5, h_min=64.0)
    with pytest.raises(ValueError):
        pa.pa_round(BitBlock(1, 32), params, pa.gen_seed(64, 1))
    with pytest.raises(ValueError):
        pa.pa_round(BitBlock(1, 64), params, pa.gen_seed(32, 1))


# ---- pkg/tests/test_acceptance.py:96-128 (compress correctness criterion) -----------

def test_criterion_compress_exhaustive_under_60s():
    t0 = time.perf_counter()
    checked = 0
    for alpha, betas in ((4, (1, 2, 4)), (6, (1, 3, 6)), (7, (4,))):
        dom = 1 << alpha
        for beta in betas:
            for c in range(1, dom, 2):
                for d in range(dom):
                    s = member(c, d, alpha)
                    for x in range(dom):
                        got = pa.compress(BitBlock(x, alpha), s, beta).value
                        assert got == ((c * x + d) % dom) >> (alpha - beta), (alpha, beta, c, d, x)
                        checked += 1
    rng = random.Random(5150)
    alpha, beta, dom = 10, 5, 1 << 10
    for _ in range(200):
        c = rng.randrange(1, dom, 2)
        d = rng.randrange(dom)
        s = member(c, d, alpha)
        for x in range(dom):
            assert pa.compress(BitBlock(x, alpha), s, beta).value == ((c * x + d) % dom) >> 5
            checked += 1
    elapsed = time.perf_counter() - t0
    print(f"compress criterion: {checked} calls in {elapsed:.1f} s "
          f"({elapsed / checked * 1e6:.1f} us per call)")
    assert checked == 1_652_736
    assert elapsed < 60.0, f"{checked} compress calls took {elapsed:.1f} s (criterion: < 60 s)"


# ---- pkg/tests/test_acceptance.py:214-246 ------------------------------------------

def test_criterion_million_bit_round_ceiling():
    n = 1_000_000
    block = bench.bench_input(RunConfig(rng_seed=33), n)
    seed = pa.gen_seed(n, 33)
    params = PAParams(n=n, r=n // 2)
    times = []
    for _ in range(5):
        t0 = time.perf_counter()
        out = pa.pa_round(block, params, seed, enforce=False)
        times.append(time.perf_counter() - t0)
        assert out.n == n // 2
    med = statistics.median(times)
    print(f"10^6-bit round: median {med * 1e3:.3f} ms")
    assert med < 0.5
    want = ((seed.c.value * block.value + seed.d.value) % (1 << n)) >> (n - n // 2)
    assert out.value == want


def test_criterion_ratio_independence():
    best = bench.measure_ratio_spread(1_000_000, (0.125, 0.5, 0.9), trials=11, rng_seed=451)
    vals = list(best.values())
    spread = (max(vals) - min(vals)) / min(vals)
    print("ratio spread:", {k: round(v * 1e3, 4) for k, v in best.items()}, f"{spread:.3f}")
    assert spread < 0.10


# ---- pkg/tests/test_cli.py:113-155 (run_pa) ----------------------------------------

def _key(tmp_path, nbytes, seed=1):
    path = tmp_path / "key.bin"
    path.write_bytes(random.Random(seed).randbytes(nbytes))
    return path


def test_run_pa_matches_library_pipeline(tmp_path):
    key = _key(tmp_path, 2 * 8, seed=3)  # two 64-bit blocks
    out = tmp_path / "out.bin"
    run_pa(RunConfig(sizes=(64,), out_bits=32, rng_seed=123, in_path=str(key),
                     out_path=str(out)))
    data = key.read_bytes()
    want = b"".join(
        pa.export_block(pa.compress(pa.import_block(data[i * 8:(i + 1) * 8], 64),
                                    pa.gen_seed(64, pa.derive_block_seed(123, i)), 32))
        for i in range(2))
    assert out.read_bytes() == want


def test_run_pa_msf_round_trip(tmp_path):
    key = _key(tmp_path, 16, seed=8)
    out = tmp_path / "out.bin"
    run_pa(RunConfig(sizes=(128,), out_bits=64, rng_seed=5, order=MSF, in_path=str(key),
                     out_path=str(out)))
    block = pa.import_block(key.read_bytes(), 128, MSF)
    seed = pa.gen_seed(128, pa.derive_block_seed(5, 0))
    assert out.read_bytes() == pa.export_block(pa.compress(block, seed, 64), MSF)


def test_run_pa_output_size_determinism_and_seed_dependence(tmp_path):
    key = _key(tmp_path, 3 * 512)  # three 4096-bit blocks
    outs = []
    for name, s in (("a", 77), ("b", 77), ("c", 78)):
        out = tmp_path / f"{name}.bin"
        res = run_pa(RunConfig(sizes=(4096,), ratio=0.5, rng_seed=s, in_path=str(key),
                               out_path=str(out)))
        assert res.blocks == 3 and res.r == 2048
        outs.append(out.read_bytes())
    assert outs[0] == outs[1] != outs[2]
    assert len(outs[0]) == 3 * 256


def test_run_pa_budget_and_short_input(tmp_path):
    key = _key(tmp_path, 512)
    out = tmp_path / "out.bin"
    with pytest.raises(SecurityBoundError):
        run_pa(RunConfig(sizes=(4096,), out_bits=2000, epsilon=2**-40, h_min=1000.0,
                         in_path=str(key), out_path=str(out)))
    assert not out.exists()
    res = run_pa(RunConfig(sizes=(4096,), out_bits=900, epsilon=2**-40, h_min=1000.0,
                           in_path=str(key), out_path=str(out)))
    assert res.budget.r == 900 and res.budget.eps_bar.log2 < -39
    short = _key(tmp_path, 100)
    with pytest.raises(ValueError, match="shorter"):
        run_pa(RunConfig(sizes=(4096,), in_path=str(short), out_path=str(out)))


def test_run_pa_config_size_against_compress(tmp_path):
    # run_pa (GPU seeds, batched) == compress per block at the C1 size
    n = 1_000_000
    key = _key(tmp_path, 3 * n // 8, seed=11)
    out = tmp_path / "out.bin"
    run_pa(RunConfig(sizes=(n,), ratio=0.5, rng_seed=2024, in_path=str(key), out_path=str(out)))
    data, got = key.read_bytes(), out.read_bytes()
    rb = n // 2 // 8
    for i in (0, 2):
        blk = pa.import_block(data[i * n // 8:(i + 1) * n // 8], n)
        s = pa.gen_seed(n, pa.derive_block_seed(2024, i))
        assert got[i * rb:(i + 1) * rb] == pa.export_block(pa.compress(blk, s, n // 2))
