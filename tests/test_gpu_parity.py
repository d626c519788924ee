"""GPU parity: the CUDA path through the C ABI against golden vectors made by the reference.

Bit-exact (integer/byte work).  Golden vectors: tests/golden/small.json, produced by
tests/golden/make_golden.py from modpa itself (pkg/src/modpa/pa.py:175-190,
pkg/src/modpa/bignum.py:194-231).
"""
import random

import pytest

import paper_1910_04429_b200 as pab
from paper_1910_04429_b200 import _native

pytestmark = pytest.mark.gpu


def _case_bytes(case):
    order = _native.ORDER_MSF if case["order"] == "msf" else _native.ORDER_LSF
    return (bytes.fromhex(case["x"]), bytes.fromhex(case["c"]), bytes.fromhex(case["d"]), order)


def test_small_golden_hash_cases(small_golden):
    bad = []
    for case in small_golden["hash"]:
        x, c, d, order = _case_bytes(case)
        got = _native.hash_host(x, c, d, case["n"], case["r"], 1, order)
        if got.hex() != case["y"]:
            bad.append((case["tag"], case["n"], case["r"], case["order"]))
    assert not bad, f"{len(bad)} mismatches: {bad[:10]}"


def test_small_golden_device_path_both_modes(small_golden, coef_words):
    # every small golden case through the batched device path (no tiny kernel)
    import torch

    from paper_1910_04429_b200.batch import HashEngine

    bad = []
    for case in small_golden["hash"]:
        x, c, d, order = _case_bytes(case)
        dev = [torch.frombuffer(bytearray(v), dtype=torch.uint8).view(1, -1).cuda()
               for v in (x, c, d)]
        out = HashEngine(case["n"], case["r"], order=order, max_batch=1).hash_device(*dev)
        if out.cpu().numpy().tobytes() != bytes.fromhex(case["y"]):
            bad.append((case["tag"], case["n"], case["r"], case["order"]))
    assert not bad, f"{len(bad)} mismatches: {bad[:10]}"


def test_small_golden_products(small_golden, coef_words):
    for case in small_golden["mul"]:
        a, b, p = int(case["a"], 16), int(case["b"], 16), int(case["p"], 16)
        assert pab.mul(a, b).value == p, (a.bit_length(), b.bit_length())


def test_compress_matches_direct_formula_random():
    rng = random.Random(11)
    for _ in range(200):
        n = rng.randrange(1, 3000)
        r = rng.randrange(1, n + 1)
        x = pab.BitBlock(rng.getrandbits(n), n)
        s = pab.gen_seed(n, rng.randrange(1 << 30))
        want = ((s.c.value * x.value + s.d.value) % (1 << n)) >> (n - r)
        assert pab.compress(x, s, r).value == want, (n, r)


def test_hash_host_multi_matches_single_device():
    import numpy as np
    import torch

    import oracle
    from paper_1910_04429_b200.batch import hash_host_multi

    n, r, B = 200_000, 77_777, 9
    rng = np.random.default_rng(4)
    arr = rng.integers(0, 256, size=(3, B, (n + 7) // 8), dtype=np.uint8)
    arr[1, :, 0] |= 1
    px, pc, pd = (torch.from_numpy(a).pin_memory() for a in arr)
    devs = list(range(torch.cuda.device_count())) * 2  # a device may appear twice (two workers)
    out = hash_host_multi(px, pc, pd, n, r, devices=devs, max_batch=2).numpy()
    for i in range(B):
        want = oracle.compress(arr[0, i].tobytes(), arr[1, i].tobytes(), arr[2, i].tobytes(), n, r)
        assert out[i].tobytes() == want, i
