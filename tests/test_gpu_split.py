"""NTT primes split over GPUs for one batch (pab_hash_host_split, SURVEY.md §8f
single-block multi-GPU): share s computes the residues of its primes, devices[0]
gathers them and does the CRT + carry.  On a one-GPU box the shares run on the
same device (separate streams, nothing waits on another share's kernels but the
gather), which exercises the partition, the residue gather and the carry-only
pass; with two or more GPUs the shares are real peers.  Bit-exact vs the oracle."""
import numpy as np
import pytest
import torch

import oracle
from paper_1910_04429_b200 import _native

pytestmark = pytest.mark.gpu


def _blocks(n, B, seed):
    rng = np.random.default_rng(seed)
    nb = (n + 7) // 8
    arr = rng.integers(0, 256, size=(3, B, nb), dtype=np.uint8)
    if n % 8:
        arr[:, :, -1] &= (1 << (n % 8)) - 1
    arr[1, :, 0] |= 1
    return arr


@pytest.mark.parametrize("n,r,B", [(1000, 333, 3), (65_537, 20_000, 2), (1_000_000, 500_000, 3),
                                   (10_000_000, 2_000_000, 1)])
@pytest.mark.parametrize("shares", [1, 2, 3, 5, 7])
def test_split_primes_match_oracle(n, r, B, shares, coef_words):
    arr = _blocks(n, B, n + shares)
    got = _native.hash_host_split(arr[0].tobytes(), arr[1].tobytes(), arr[2].tobytes(), n, r, B,
                                  devices=[0] * shares)
    rb = (r + 7) // 8
    for i in range(B):
        want = oracle.compress(arr[0, i].tobytes(), arr[1, i].tobytes(), arr[2, i].tobytes(), n, r)
        assert got[i * rb:(i + 1) * rb] == want, (n, r, shares, i)


def test_split_msf_and_repeat_calls():
    n, r, B = 300_007, 123_457, 2
    arr = _blocks(n, B, 9)
    for shares in (2, 4):
        got = _native.hash_host_split(arr[0].tobytes(), arr[1].tobytes(), arr[2].tobytes(), n, r,
                                      B, order=_native.ORDER_MSF, devices=[0] * shares)
        rb = (r + 7) // 8
        for i in range(B):
            want = oracle.compress(arr[0, i].tobytes(), arr[1, i].tobytes(), arr[2, i].tobytes(),
                                   n, r, msf=True)
            assert got[i * rb:(i + 1) * rb] == want


def test_split_across_gpus_when_present():
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU: the peer path needs two")
    n, r = 10_000_000, 5_000_000
    arr = _blocks(n, 1, 3)
    devs = list(range(torch.cuda.device_count()))
    got = _native.hash_host_split(arr[0].tobytes(), arr[1].tobytes(), arr[2].tobytes(), n, r, 1,
                                  devices=devs)
    assert got == oracle.compress(arr[0, 0].tobytes(), arr[1, 0].tobytes(), arr[2, 0].tobytes(), n, r)


def test_split_errors():
    with pytest.raises(ValueError, match="at least one device"):
        _native.check(_native.load().pab_hash_host_split(b"\x01", b"\x01", b"\x00", 8, 4, 1, 0,
                                                         ctypes_out(1), None, 0))
    with pytest.raises(ValueError):
        _native.hash_host_split(b"\x01", b"\x01", b"\x00", 8, 9, 1, devices=[0])


def ctypes_out(nbytes):
    import ctypes

    return ctypes.create_string_buffer(nbytes)
