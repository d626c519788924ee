"""Host logic of the drop-in (no GPU): validation, layout, seeds, enforcement.

Mirrors the reference's own tests for these behaviours
(pkg/tests/test_pa.py:30-121, 196-254) with identical error types/messages.
"""
import hashlib

import pytest

import paper_1910_04429_b200 as pab
from paper_1910_04429_b200 import security, workloads
from paper_1910_04429_b200.bignum import BigNat, WordOrder

LSF = WordOrder.LEAST_SIGNIFICANT_FIRST
MSF = WordOrder.MOST_SIGNIFICANT_FIRST


def seed_of(c, d, alpha):
    return pab.HashSeed(c=BigNat(c), d=BigNat(d), alpha=alpha)


def test_bitblock_validation():
    with pytest.raises(ValueError):
        pab.BitBlock(0, 0)
    with pytest.raises(ValueError):
        pab.BitBlock(4, 2)
    b = pab.BitBlock(0b1010, 4)
    assert [b.bit(i) for i in range(4)] == [0, 1, 0, 1]
    with pytest.raises(IndexError):
        b.bit(4)


def test_import_export_layout():
    assert pab.import_block(b"\x01\x02", 16, LSF).value == 0x0201
    assert pab.import_block(b"\x01\x02", 16, MSF).value == 0x0102
    with pytest.raises(ValueError, match="truncated"):
        pab.import_block(b"\x01", 16)
    pab.import_block(b"\xff\x0f", 12, LSF)
    with pytest.raises(ValueError, match="beyond"):
        pab.import_block(b"\xff\x10", 12, LSF)
    with pytest.raises(ValueError, match="beyond"):
        pab.import_block(b"\x10\xff", 12, MSF)
    blk = pab.BitBlock(0b101, 12)
    assert pab.export_block(blk, LSF) == b"\x05\x00"
    assert pab.export_block(blk, MSF) == b"\x00\x05"


def test_seed_validation_and_determinism():
    with pytest.raises(ValueError):
        seed_of(2, 0, 4)
    with pytest.raises(ValueError):
        seed_of(17, 0, 4)
    with pytest.raises(ValueError):
        seed_of(1, 16, 4)
    assert pab.gen_seed(256, 12345) == pab.gen_seed(256, 12345)
    assert pab.gen_seed(256, 1) != pab.gen_seed(256, 2)
    for s in range(64):
        assert pab.gen_seed(64, s).c.value % 2 == 1
    seen = {(pab.gen_seed(4, s).c.value, pab.gen_seed(4, s).d.value) for s in range(4096)}
    assert seen == {(c, d) for c in range(1, 16, 2) for d in range(16)}


def test_input_derivation_matches_reference_digests(config_golden):
    # SHAKE-256 framing of pa._expand / gen_seed / derive_block_seed (pa.py:138-172)
    for name, idxs in (("C2", range(0, 1024, 97)), ("C3", [3]), ("C5", [0])):
        g = config_golden[name]
        for i in idxs:
            rec = g["blocks"][i]
            x, c, d = workloads.block_inputs(g["n"], rec["seed"])
            assert hashlib.sha256(x).hexdigest() == rec["x"]
            assert hashlib.sha256(c).hexdigest() == rec["c"]
            assert hashlib.sha256(d).hexdigest() == rec["d"]


def test_params_validation():
    with pytest.raises(ValueError):
        pab.PAParams(n=8, r=0)
    with pytest.raises(ValueError):
        pab.PAParams(n=8, r=9)
    with pytest.raises(ValueError):
        pab.PAParams(n=8, r=4, epsilon=0.0)


def test_compress_validation_happens_before_device():
    with pytest.raises(ValueError, match="does not match seed alpha"):
        pab.compress(pab.BitBlock(1, 8), seed_of(3, 1, 16), 4)
    with pytest.raises(ValueError, match="must satisfy"):
        pab.compress(pab.BitBlock(1, 8), seed_of(3, 1, 8), 9)


def test_pa_round_enforcement_host_side():
    n = 4096
    params = pab.PAParams(n=n, r=1000, epsilon=2**-40, h_min=1000.0)
    with pytest.raises(pab.SecurityBoundError) as exc:
        pab.pa_round(pab.BitBlock(123, n), params, pab.gen_seed(n, 1))
    assert exc.value.r_max == 920  # pkg/tests/test_pa.py:205-211
    with pytest.raises(ValueError, match="enforce"):
        pab.pa_round(pab.BitBlock(1, 64), pab.PAParams(n=64, r=32), pab.gen_seed(64, 1))
    with pytest.raises(ValueError):
        pab.pa_round(pab.BitBlock(1, 32), pab.PAParams(n=64, r=32, epsilon=0.5, h_min=64.0),
                     pab.gen_seed(64, 1))


def test_security_values():
    assert security.max_key_length(1000.0, 2**-40) == 920
    assert security.max_key_length(10.0, 1.0) == 10
    assert security.max_key_length(5.0, 0.0) == 0
    assert security.leftover_bound_log2(100.0, 100.0, 0.0) == -1.0


def test_product_path_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        pab.compress(pab.BitBlock(5, 4), seed_of(3, 1, 4), 2)
    with pytest.raises(RuntimeError):
        pab.mul(3, 5)


def test_words_round_trip():
    v = (1 << 200) + 12345
    for order in (LSF, MSF):
        assert pab.from_words(pab.to_words(v, order), order).value == v
    assert pab.mod_pow2(0b1111, 2).value == 3
    assert pab.shift_right(0b1100, 2).value == 3


def test_digit_level_int_byte_conversions():
    # import_block / export_block over CPython digits (pab_bytes_to_digits /
    # pab_digits_to_bytes, host code) equal int.from_bytes / int.to_bytes
    import random

    from paper_1910_04429_b200 import _pyint
    from paper_1910_04429_b200.bignum import WordOrder

    if not _pyint.supported():
        pytest.skip("interpreter int layout not supported (byte conversions used)")
    rng = random.Random(12)
    for nb in list(range(0, 80)) + [255, 256, 257, 4096, 125_000, 125_001]:
        raw = rng.randbytes(nb)
        for msf in (False, True):
            endian = "big" if msf else "little"
            v = int.from_bytes(raw, endian)
            assert _pyint.from_bytes(raw, msf) == v
            assert _pyint.to_bytes(v, nb, msf) == raw
            if nb:
                assert _pyint.to_bytes(v >> 13, nb, msf) == (v >> 13).to_bytes(nb, endian)
    for order in (WordOrder.LEAST_SIGNIFICANT_FIRST, WordOrder.MOST_SIGNIFICANT_FIRST):
        raw = rng.randbytes(5000)
        n = 5000 * 8 - 3
        endian = "big" if order is WordOrder.MOST_SIGNIFICANT_FIRST else "little"
        raw = (int.from_bytes(raw, endian) >> 3).to_bytes(5000, endian)
        blk = pab.import_block(raw, n, order)
        assert blk.value == int.from_bytes(raw, endian)
        assert pab.export_block(blk, order) == raw
    with pytest.raises(ValueError, match="beyond"):
        pab.import_block(b"\xff" * 5000, 5000 * 8 - 3)


def test_exclusive_seed_windows_cover_the_call():
    # hash_seeded_host's exclusive schedule: windows (in hashing chunks) cover the call
    # exactly, stay at or under the target (or the cap), and are as even as possible;
    # a call of up to 1.5 targets is one window
    from paper_1910_04429_b200.batch import exclusive_windows

    assert exclusive_windows(20, 4, 16) == [4, 4, 4, 4, 4]
    assert exclusive_windows(25, 4, 16) == [4, 4, 4, 4, 3, 3, 3]
    assert exclusive_windows(9, 8, 1000) == [9]
    assert exclusive_windows(13, 8, 1000) == [7, 6]
    assert exclusive_windows(6, 2, 2) == [2, 2, 2]
    for n in range(1, 200):
        for target, cap in ((4, 16), (8, 5), (3, 3), (16, 1000)):
            w = exclusive_windows(n, target, cap)
            assert sum(w) == n and min(w) >= 1 and max(w) - min(w) <= 1
            assert max(w) <= cap or n <= cap
            assert len(w) == 1 or max(w) <= min(target, cap)
