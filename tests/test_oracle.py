"""Pin the CPU oracle (oracle/modpa_ssa.c) to outputs of the reference itself.

Golden vectors come from the reference package (tests/golden/make_golden.py):
raw vectors for small/ragged/MSF/edge blocks and full products, plus SHA-256
digests of every output key of configs C1..C5.  The oracle must reproduce
them bit-for-bit before it is trusted as the checker of the CUDA path.
"""
import hashlib
import random

import pytest

import oracle
from paper_1910_04429_b200 import workloads


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def test_oracle_small_golden_hash(small_golden):
    for case in small_golden["hash"]:
        y = oracle.compress(bytes.fromhex(case["x"]), bytes.fromhex(case["c"]),
                            bytes.fromhex(case["d"]), case["n"], case["r"], case["order"] == "msf")
        assert y.hex() == case["y"], (case["tag"], case["n"], case["r"])


def test_oracle_small_golden_products(small_golden):
    for case in small_golden["mul"]:
        a, b, p = int(case["a"], 16), int(case["b"], 16), int(case["p"], 16)
        assert oracle.mul(a, b) == p


def test_oracle_kats():
    # the reference's worked examples, pkg/tests/test_pa.py:125-133
    assert oracle.compress(bytes([5]), bytes([3]), bytes([1]), 4, 2) == bytes([0])
    assert oracle.compress(bytes([7]), bytes([5]), bytes([2]), 4, 2) == bytes([1])


def test_oracle_exhaustive_alpha6():
    # pkg/tests/test_pa.py:151-161, subsampled over c to keep the CPU suite fast
    alpha = 6
    for beta in (1, 3, 6):
        for c in range(1, 64, 6):
            for d in range(0, 64, 5):
                for x in range(64):
                    want = ((c * x + d) % 64) >> (alpha - beta)
                    got = oracle.compress(bytes([x]), bytes([c]), bytes([d]), alpha, beta)
                    assert got[0] == want


def test_oracle_plan_matches_reference_geometry():
    # reference ntt.plan at the config sizes (measured with modpa)
    assert oracle.plan(10**6) == (10, 1_015_808, 1984, 4096)
    assert oracle.plan(10**7) == (11, 10_027_008, 9792, 20_480)
    assert oracle.plan(10**8) == (13, 100_139_008, 24_448, 49_152)


def test_oracle_product_vs_interpreter():
    rng = random.Random(63)
    for bits in (1, 64, 1000, 2**17, 10**6):
        a, b = rng.getrandbits(bits), rng.getrandbits(bits)
        assert oracle.mul(a, b) == a * b


def _check_blocks(config_golden, name, idxs, ratio_idx=None):
    g = config_golden[name]
    n = g["n"]
    for i in idxs:
        rec = g["blocks"][i]
        x, c, d = workloads.block_inputs(n, rec["seed"])
        assert sha(x) == rec["x"] and sha(c) == rec["c"] and sha(d) == rec["d"]
        for m in g["ms"]:
            y = oracle.compress(x, c, d, n, m)
            assert sha(y) == rec["out"][str(m)], (name, rec["seed"], m)


def test_oracle_config_C1(config_golden):
    _check_blocks(config_golden, "C1", [0])


def test_oracle_config_C2_sample(config_golden):
    _check_blocks(config_golden, "C2", [1, 2, 511, 1023])


def test_oracle_config_C3_sample(config_golden):
    _check_blocks(config_golden, "C3", [0, 63])


def test_oracle_config_C4(config_golden):
    _check_blocks(config_golden, "C4", [0])


def test_oracle_config_C5_one_block_three_ratios(config_golden):
    _check_blocks(config_golden, "C5", [5])


def test_gmp_context_matches_reference(small_golden, config_golden):
    # the paper's GMP call sequence (oracle/gmp_ref.py) against reference outputs
    from oracle import gmp_ref

    if not gmp_ref.available():
        pytest.skip("libgmp not present")
    for case in small_golden["hash"]:
        if case["order"] != "lsf":
            continue
        y = gmp_ref.compress(bytes.fromhex(case["x"]), bytes.fromhex(case["c"]),
                             bytes.fromhex(case["d"]), case["n"], case["r"])
        assert y.hex() == case["y"], (case["tag"], case["n"])
    rec = config_golden["C1"]["blocks"][0]
    x, c, d = workloads.block_inputs(10**6, rec["seed"])
    assert sha(gmp_ref.compress(x, c, d, 10**6, 500_000)) == rec["out"]["500000"]
