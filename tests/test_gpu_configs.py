"""GPU parity at the five BASELINE configs and size-independent properties at full size.

Every output key of C1..C5 is compared (SHA-256) with digests produced by the
reference itself (tests/golden/configs.json via tests/golden/make_golden.py);
bit-exact is the only acceptable result.
"""
import hashlib
import random

import numpy as np
import pytest
import torch

import oracle
import paper_1910_04429_b200 as pab
from paper_1910_04429_b200 import _native, workloads
from paper_1910_04429_b200.batch import HashEngine

pytestmark = pytest.mark.gpu


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def _run_config(config_golden, name, max_batch=64, blocks=None):
    g = config_golden[name]
    n = g["n"]
    recs = g["blocks"] if blocks is None else [g["blocks"][i] for i in blocks]
    seeds = [rec["seed"] for rec in recs]
    xs, cs, ds = workloads.batch_inputs(n, seeds)
    for rec, x in zip(recs, xs):
        assert sha(x.tobytes()) == rec["x"]
    dx, dc, dd = (torch.from_numpy(a).cuda() for a in (xs, cs, ds))
    bad = []
    for m in g["ms"]:
        eng = HashEngine(n, m, max_batch=max_batch)
        out = eng.hash_device(dx, dc, dd).cpu().numpy()
        for i, rec in enumerate(recs):
            if sha(out[i].tobytes()) != rec["out"][str(m)]:
                bad.append((rec["seed"], m))
    assert not bad, f"{name}: {len(bad)} blocks differ from the reference: {bad[:8]}"


def test_config_C1(config_golden):
    _run_config(config_golden, "C1")


def test_config_C2_all_1024_blocks(config_golden):
    _run_config(config_golden, "C2", max_batch=1024)


def test_config_C3_all_64_blocks(config_golden):
    _run_config(config_golden, "C3", max_batch=16)


def test_config_C4(config_golden):
    _run_config(config_golden, "C4", max_batch=1)


@pytest.mark.parametrize("part", range(4))
def test_config_C5_all_blocks_all_ratios(config_golden, part):
    _run_config(config_golden, "C5", max_batch=8, blocks=range(part * 16, part * 16 + 16))


def test_small_batch_chunking_matches_single(small_golden):
    # batch larger than the workspace chunk: results independent of chunking
    n, r, B = 100_003, 33_333, 13
    rng = np.random.default_rng(3)
    nb = (n + 7) // 8
    arr = rng.integers(0, 256, size=(3, B, nb), dtype=np.uint8)
    arr[:, :, -1] &= (1 << (n % 8)) - 1
    arr[1, :, 0] |= 1
    dx, dc, dd = (torch.from_numpy(a).cuda() for a in arr)
    one = HashEngine(n, r, max_batch=B).hash_device(dx, dc, dd).cpu()
    few = HashEngine(n, r, max_batch=3).hash_device(dx, dc, dd).cpu()
    assert torch.equal(one, few)
    for i in (0, 7, 12):
        want = oracle.compress(arr[0, i].tobytes(), arr[1, i].tobytes(), arr[2, i].tobytes(), n, r)
        assert one[i].numpy().tobytes() == want


def test_identity_member_full_size():
    # c = 1, d = 0, r = n returns x (pkg/tests/test_pa.py:135-140) at n = 1e8
    n = 100_000_000
    x = workloads.block_inputs(n, 11)[0]
    one = (1).to_bytes((n + 7) // 8, "little")
    zero = bytes((n + 7) // 8)
    assert _native.hash_host(x, one, zero, n, n) == x


def test_full_length_carry_full_size():
    # x = 1, c = 2^n - 1, d = 1: c*x + d = 2^n -> 0 after mod 2^n (carry through every word)
    for n in (1_000_000, 100_000_000, 1 << 27):
        nb = (n + 7) // 8
        full = ((1 << n) - 1).to_bytes(nb, "little")
        one = (1).to_bytes(nb, "little")
        assert _native.hash_host(one, full, one, n, n // 2) == bytes((n // 2 + 7) // 8)


def test_prefix_property_and_offset_linearity():
    # y_r = y_n >> (n - r) for all r; and T(d1) - T(d2) = d1 - d2 mod 2^n
    n = 10_000_000
    x, c, d = workloads.block_inputs(n, 5)
    full = int.from_bytes(_native.hash_host(x, c, d, n, n), "little")
    for r in (1, 7, 31, 32, 33, 1_000_001, n - 1):
        got = int.from_bytes(_native.hash_host(x, c, d, n, r), "little")
        assert got == full >> (n - r), r
    d2 = workloads.block_inputs(n, 6)[2]
    full2 = int.from_bytes(_native.hash_host(x, c, d2, n, n), "little")
    dv, dv2 = int.from_bytes(d, "little"), int.from_bytes(d2, "little")
    assert (full - full2) % (1 << n) == (dv - dv2) % (1 << n)


@pytest.mark.parametrize("batch", [1, 300])
def test_unaligned_shift_across_tiles(batch, coef_words):
    # (n - r) % 32 != 0 with outputs spanning many carry tiles, one block and
    # many blocks in flight (look-back carry)
    n = 300_007 if batch > 1 else 3_000_013
    rng = np.random.default_rng(21 + batch)
    nb = (n + 7) // 8
    arr = rng.integers(0, 256, size=(3, batch, nb), dtype=np.uint8)
    arr[:, :, -1] &= (1 << (n % 8)) - 1
    arr[1, :, 0] |= 1
    dx, dc, dd = (torch.from_numpy(a).cuda() for a in arr)
    for r in (n - 1, n // 2 + 3, 4097 * 32 + 5):
        out = HashEngine(n, r, max_batch=batch).hash_device(dx, dc, dd).cpu().numpy()
        for i in sorted({0, batch // 2, batch - 1}):
            want = oracle.compress(arr[0, i].tobytes(), arr[1, i].tobytes(), arr[2, i].tobytes(),
                                   n, r)
            assert out[i].tobytes() == want, (batch, r, i)


@pytest.mark.parametrize("n", [1 << 27, 32 * ((5 * 2**22 + 1) // 2)])
def test_max_size_and_range_errors(n):
    assert _native.max_bits() >= n
    rng = random.Random(9)
    nb = n // 8
    x = rng.randbytes(nb)
    c = bytearray(rng.randbytes(nb))
    c[0] |= 1
    d = rng.randbytes(nb)
    got = _native.hash_host(x, bytes(c), d, n, 12_345)
    assert got == oracle.compress(x, bytes(c), d, n, 12_345)
    if n == _native.max_bits():
        with pytest.raises(ValueError):
            _native.hash_host(x + b"\0", bytes(c) + b"\0", d + b"\0", n + 1, 5)


def _plan_sweep_sizes(limit=1 << 27):
    """One block size per distinct (radix, lg_rows, lg_cols) plan up to `limit` bits."""
    seen, sizes = set(), []
    n = 2000
    while n < limit:
        key = _native.plan_info(n)
        if key not in seen:
            seen.add(key)
            sizes.append(n)
        n = int(n * 1.09) + 7
    return sizes


def test_every_transform_plan_matches_oracle(coef_words):
    # forced 64-bit coefficients end at the five-prime CRT bound
    sizes = _plan_sweep_sizes(1 << 27 if coef_words == 1 else 121_295_104)
    radices = {_native.plan_info(n)[0] for n in sizes}
    assert radices == {1, 3, 5}, radices
    rng = np.random.default_rng(77)
    for n in sizes:
        r = int(rng.integers(1, n + 1))
        nb = (n + 7) // 8
        nblk = 2 if n < (1 << 24) else 1
        arr = rng.integers(0, 256, size=(3, nblk, nb), dtype=np.uint8)
        if n % 8:
            arr[:, :, -1] &= (1 << (n % 8)) - 1
        arr[1, :, 0] |= 1
        dx, dc, dd = (torch.from_numpy(a).cuda() for a in arr)
        out = HashEngine(n, r, max_batch=2).hash_device(dx, dc, dd).cpu().numpy()
        for i in range(nblk):
            want = oracle.compress(arr[0, i].tobytes(), arr[1, i].tobytes(), arr[2, i].tobytes(),
                                   n, r)
            assert out[i].tobytes() == want, (n, r, _native.plan_info(n))


def test_msf_large_block():
    n, r = 3_000_001, 1_234_567
    rng = random.Random(12)
    nb = (n + 7) // 8
    vals = [rng.getrandbits(n) for _ in range(3)]
    vals[1] |= 1
    x, c, d = (v.to_bytes(nb, "big") for v in vals)
    got = _native.hash_host(x, c, d, n, r, 1, _native.ORDER_MSF)
    assert got == oracle.compress(x, c, d, n, r, msf=True)


def test_ten_million_bit_product():
    # pkg/tests/test_ntt.py:256-262: a 10^7-bit product equals the interpreter's
    rng = random.Random(63)
    a = rng.getrandbits(10**7)
    b = rng.getrandbits(10**7)
    assert pab.mul(a, b).value == oracle.mul(a, b)


def test_unbalanced_and_trivial_products(coef_words):
    rng = random.Random(6)
    for _ in range(30):
        a = rng.getrandbits(rng.randrange(1, 400_000))
        b = rng.getrandbits(rng.randrange(1, 130))
        assert pab.mul(a, b).value == a * b
    assert pab.mul(0, 12345).value == 0
    assert pab.mul(12345, 1).value == 12345
    w = (1 << 64) - 1
    assert pab.mul(w, w).value == (1 << 128) - (1 << 65) + 1


def test_exhaustive_alpha6_on_gpu_batched():
    # pkg/tests/test_pa.py:151-161: every (c, d, x) at alpha=6, beta in {1,3,6}, one launch each
    alpha = 6
    cs_, ds_, xs_ = np.meshgrid(np.arange(1, 64, 2), np.arange(64), np.arange(64), indexing="ij")
    c = torch.from_numpy(cs_.reshape(-1, 1).astype(np.uint8)).cuda()
    d = torch.from_numpy(ds_.reshape(-1, 1).astype(np.uint8)).cuda()
    x = torch.from_numpy(xs_.reshape(-1, 1).astype(np.uint8)).cuda()
    for beta in (1, 3, 6):
        out = HashEngine(alpha, beta, max_batch=4096).hash_device(x, c, d).cpu().numpy()[:, 0]
        want = ((cs_ * xs_ + ds_) % 64) >> (alpha - beta)
        assert np.array_equal(out, want.reshape(-1).astype(np.uint8))


@pytest.mark.parametrize("mode", ["seq", "lb"])
def test_alternate_carry_modes_match_oracle(mode):
    # the warp-striped carries (production only for 32-bit coefficients; with
    # 64-bit coefficients the lane-contiguous k_carry_wide runs): one CTA per
    # block walking its tiles (seq) or the decoupled look-back (lb), forced
    # through their development switch in a fresh process
    import os
    import subprocess
    import sys

    code = """
import numpy as np, torch, oracle
from paper_1910_04429_b200.batch import HashEngine
from paper_1910_04429_b200 import _native
for cw in (2, 1):
    _native.force_coef_words(cw)
    for n, r, B in ((300_007, 123_457, 3), (2_000_000, 999_999, 2)):
        rng = np.random.default_rng(n + cw)
        nb = (n + 7) // 8
        arr = rng.integers(0, 256, size=(3, B, nb), dtype=np.uint8)
        if n % 8:
            arr[:, :, -1] &= (1 << (n % 8)) - 1
        arr[1, :, 0] |= 1
        out = HashEngine(n, r, max_batch=B).hash_device(*(torch.from_numpy(a).cuda() for a in arr))
        out = out.cpu().numpy()
        for i in range(B):
            want = oracle.compress(*(arr[j, i].tobytes() for j in range(3)), n, r)
            assert out[i].tobytes() == want, (cw, n, i)
print("SEQ_OK")
"""
    env = dict(os.environ, PAB_CARRY_MODE=mode)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert res.returncode == 0 and "SEQ_OK" in res.stdout, res.stderr[-2000:]


@pytest.mark.parametrize("n,cw", [(200_000_000, 0), (45_505_408, 1)])
def test_fused_mixed_radix_forward_with_32bit_coefficients(n, cw):
    # the fused radix-3 forward pass at (m=3, lgR=10, lgC=12)
    # must not take its 8-byte-coefficient fast path for 32-bit coefficients with
    # an even word count (n = 2e8 by default plan; 45,505,408 with cw forced to 1)
    assert (n // 32) % 2 == 0
    _native.force_coef_words(cw)
    try:
        rng = random.Random(n)
        nb = n // 8
        x = rng.randbytes(nb)
        c = bytearray(rng.randbytes(nb))
        c[0] |= 1
        d = rng.randbytes(nb)
        for r in (n // 2, 1_000_003):
            got = _native.hash_host(x, bytes(c), d, n, r)
            assert got == oracle.compress(x, bytes(c), d, n, r), (n, cw, r, _native.plan_info(n))
    finally:
        _native.force_coef_words(0)
