"""Edge cases of the C ABI: size-class boundaries, strides, misaligned pointers,
byte order through the batched API, and concurrent callers.  All bit-exact vs the oracle."""
import threading

import numpy as np
import pytest
import torch

import oracle
import paper_1910_04429_b200 as pab
from paper_1910_04429_b200 import _native
from paper_1910_04429_b200.batch import HashEngine

pytestmark = pytest.mark.gpu


def _rand_blocks(rng, n, B, odd=True):
    nb = (n + 7) // 8
    arr = rng.integers(0, 256, size=(3, B, nb), dtype=np.uint8)
    if n % 8:
        arr[:, :, -1] &= (1 << (n % 8)) - 1
    if odd:
        arr[1, :, 0] |= 1
    return arr


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 2047, 2048, 2049, 4096, 65_504, 65_536,
                               65_537, 65_600])
def test_size_class_boundaries(n, coef_words):
    # tiny (<= 2048 bits, host path), single-CTA (L <= 4096), four-step
    rng = np.random.default_rng(n)
    arr = _rand_blocks(rng, n, 3)
    for r in sorted({1, max(1, n // 3), n}):
        for i in range(3):
            x, c, d = (arr[j, i].tobytes() for j in range(3))
            assert _native.hash_host(x, c, d, n, r) == oracle.compress(x, c, d, n, r), (n, r, i)
        dx, dc, dd = (torch.from_numpy(a).cuda() for a in arr)
        out = HashEngine(n, r, max_batch=3).hash_device(dx, dc, dd).cpu().numpy()
        for i in range(3):
            want = oracle.compress(*(arr[j, i].tobytes() for j in range(3)), n, r)
            assert out[i].tobytes() == want, (n, r, i)


def test_strided_and_misaligned_device_buffers():
    # rows padded to odd strides and a 1-byte offset: the pack/unpack path
    n, r, B = 100_007, 40_001, 5
    nb, rb = (n + 7) // 8, (r + 7) // 8
    rng = np.random.default_rng(7)
    arr = _rand_blocks(rng, n, B)
    stride = nb + 13
    big = torch.zeros((3, B * stride + 1), dtype=torch.uint8)
    for j in range(3):
        for i in range(B):
            big[j, 1 + i * stride: 1 + i * stride + nb] = torch.from_numpy(arr[j, i])
    dev = big.cuda()
    views = [dev[j, 1:1 + B * stride].view(B, stride) for j in range(3)]  # misaligned by 1 byte
    out_big = torch.zeros(B * (rb + 5) + 3, dtype=torch.uint8, device="cuda")
    out = out_big[3:].view(B, rb + 5)
    eng = HashEngine(n, r, max_batch=2)
    eng.hash_device(views[0], views[1], views[2], out)
    got = out.cpu().numpy()
    for i in range(B):
        want = oracle.compress(*(arr[j, i].tobytes() for j in range(3)), n, r)
        assert got[i, :rb].tobytes() == want, i
        assert not got[i, rb:].any()  # nothing written past the key


def test_msf_through_batched_api():
    n, r, B = 250_001, 99_999, 4
    rng = np.random.default_rng(8)
    vals = [[int.from_bytes(rng.bytes((n + 7) // 8), "little") & ((1 << n) - 1) for _ in range(B)]
            for _ in range(3)]
    for i in range(B):
        vals[1][i] |= 1
    nb = (n + 7) // 8
    arr = np.array([[np.frombuffer(v.to_bytes(nb, "big"), np.uint8) for v in row] for row in vals])
    dx, dc, dd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arr)
    out = HashEngine(n, r, max_batch=B, order=_native.ORDER_MSF).hash_device(dx, dc, dd).cpu()
    for i in range(B):
        want = ((vals[1][i] * vals[0][i] + vals[2][i]) % (1 << n)) >> (n - r)
        assert int.from_bytes(out[i].numpy().tobytes(), "big") == want


def test_concurrent_compress_threads():
    # the drop-in API is reentrant (per-device host context behind a lock)
    rng = np.random.default_rng(9)
    jobs = []
    for n in (64, 3000, 70_000, 300_000):
        x = pab.BitBlock(int.from_bytes(rng.bytes((n + 7) // 8), "little") & ((1 << n) - 1), n)
        s = pab.gen_seed(n, int(rng.integers(1 << 30)))
        jobs.append((x, s, n // 3 + 1))
    want = [((s.c.value * x.value + s.d.value) % (1 << x.n)) >> (x.n - r) for x, s, r in jobs]
    errors = []

    def worker(k):
        try:
            for _ in range(5):
                for (x, s, r), w in zip(jobs, want):
                    assert pab.compress(x, s, r).value == w
        except BaseException as e:
            errors.append(e)

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[0]


def test_zero_batch_and_errors():
    lib = _native.load()
    assert lib.pab_hash_batch(None, None, None, 16, 100, 50, 0, 0, None, 16, None, 0, None) == 0
    with pytest.raises(ValueError):
        _native.hash_host(b"\x01", b"\x01", b"\x01", 8, 9)
    with pytest.raises(ValueError):
        HashEngine(100, 0)


@pytest.mark.parametrize("n", [500_000, 65_504, 4_000_032])
def test_four_byte_aligned_rows_direct(n, coef_words):
    # n = 32 mod 64: ceil(n/8) % 8 == 4, so rows alternate between 8- and 4-byte
    # alignment and the word count is odd (the last 64-bit coefficient has no
    # high word); read in place, without the pack kernel
    rng = np.random.default_rng(n + 1)
    B = 5
    arr = _rand_blocks(rng, n, B)
    dx, dc, dd = (torch.from_numpy(a).cuda() for a in arr)
    for r in (n // 2, n - 7):
        out = HashEngine(n, r, max_batch=B).hash_device(dx, dc, dd).cpu().numpy()
        for i in range(B):
            want = oracle.compress(*(arr[j, i].tobytes() for j in range(3)), n, r)
            assert out[i].tobytes() == want, (n, r, i)
