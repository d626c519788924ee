"""Memory-safety and race checks of our own (compute-sanitizer is closed on this
GPU pool: profiles/r2/compute_sanitizer_closed.log).

* Guard bands: every buffer pab_hash_batch / pab_mul_add / pab_seed_expand writes
  (workspace, key rows, seed rows) sits inside a larger allocation filled with a
  canary pattern; after the call every byte outside the documented extents must
  still hold the canary (an out-of-bounds store anywhere shows up).
* Look-back races: the decoupled look-back carry (k_carry_wide, and the
  warp-striped k_carry_lb for 32-bit coefficients) is run many times over
  multi-tile batches while other kernels perturb the CTA schedule; every run
  must be identical and equal to the oracle.
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle
from paper_1910_04429_b200 import _native
from paper_1910_04429_b200.batch import HashEngine

pytestmark = pytest.mark.gpu

CANARY = 0xA5
GUARD = 1 << 16


def _guarded(nbytes):
    buf = torch.full((nbytes + 2 * GUARD,), CANARY, dtype=torch.uint8, device="cuda")
    return buf, buf[GUARD:GUARD + nbytes]


def _outside_untouched(buf, lo, hi):
    host = buf.cpu().numpy()
    return bool((host[:GUARD + lo] == CANARY).all() and (host[GUARD + hi:] == CANARY).all())


@pytest.mark.parametrize("n,r,B", [(5_000, 1_777, 3), (300_007, 150_001, 4),
                                   (1_000_000, 500_000, 3), (10_000_000, 2_000_001, 1)])
def test_hash_batch_stays_inside_its_buffers(n, r, B, coef_words):
    lib = _native.load()
    nb, rb = (n + 7) // 8, (r + 7) // 8
    in_stride = nb + 13  # odd stride: 4-byte rows and the pack path
    out_stride = rb + 5
    rng = np.random.default_rng(n + coef_words)
    host = rng.integers(0, 256, size=(3, B, in_stride), dtype=np.uint8)
    host[:, :, nb:] = 0
    if n % 8:
        host[:, :, nb - 1] &= (1 << (n % 8)) - 1
    host[1, :, 0] |= 1
    ins = torch.from_numpy(host).cuda()
    ws_bytes = int(lib.pab_hash_workspace_bytes(n, B))
    wbuf, ws = _guarded(ws_bytes)
    obuf, out = _guarded(B * out_stride)
    _native.check(lib.pab_hash_batch(ins[0].data_ptr(), ins[1].data_ptr(), ins[2].data_ptr(),
                                     in_stride, n, r, B, _native.ORDER_LSF, out.data_ptr(),
                                     out_stride, ws.data_ptr(), ws_bytes,
                                     ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    assert _outside_untouched(wbuf, 0, ws_bytes), "workspace guard band written"
    # key rows: only the first rb bytes of each row may change
    o = obuf.cpu().numpy()
    assert (o[:GUARD] == CANARY).all() and (o[GUARD + B * out_stride:] == CANARY).all()
    rows = o[GUARD:GUARD + B * out_stride].reshape(B, out_stride)
    assert (rows[:, rb:] == CANARY).all(), "key row padding written"
    for i in range(B):
        want = oracle.compress(host[0, i, :nb].tobytes(), host[1, i, :nb].tobytes(),
                               host[2, i, :nb].tobytes(), n, r)
        assert rows[i, :rb].tobytes() == want


def test_mul_add_and_seed_expand_stay_inside_their_buffers():
    lib = _native.load()
    rng = np.random.default_rng(5)
    acc, a, b = (rng.integers(0, 256, size=k, dtype=np.uint8) for k in (70_001, 40_003, 50_007))
    da, db, dacc = (torch.from_numpy(v).cuda() for v in (a, b, acc))
    ob = max(len(a) + len(b), len(acc)) + 1
    ws_bytes = int(lib.pab_mul_add_workspace_bytes(len(acc), len(a), len(b)))
    wbuf, ws = _guarded(ws_bytes)
    obuf, out = _guarded(ob)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _native.check(lib.pab_mul_add(dacc.data_ptr(), len(acc), da.data_ptr(), len(a), db.data_ptr(),
                                  len(b), out.data_ptr(), ob, ws.data_ptr(), ws_bytes, st))
    torch.cuda.synchronize()
    assert _outside_untouched(wbuf, 0, ws_bytes) and _outside_untouched(obuf, 0, ob)
    iv = lambda v: int.from_bytes(v.tobytes(), "little")  # noqa: E731
    assert int.from_bytes(out.cpu().numpy().tobytes(), "little") == iv(acc) + iv(a) * iv(b)
    # seed rows: ceil(n/8) bytes per row at `stride`, nothing else
    n, B, stride = 20_001, 5, 2_600
    nb = (n + 7) // 8
    cbuf, c = _guarded(B * stride)
    dbuf, d = _guarded(B * stride)
    m = _native.seed_material(77)
    _native.check(lib.pab_seed_expand(m, len(m), 3, B, n, _native.ORDER_LSF, c.data_ptr(),
                                      d.data_ptr(), stride, st))
    torch.cuda.synchronize()
    for buf in (cbuf, dbuf):
        h = buf.cpu().numpy()
        assert (h[:GUARD] == CANARY).all() and (h[GUARD + B * stride:] == CANARY).all()
        assert (h[GUARD:GUARD + B * stride].reshape(B, stride)[:, nb:] == CANARY).all()


@pytest.mark.parametrize("n,r,B,cw", [(1_000_000, 500_001, 64, 2), (3_000_013, 1_000_003, 4, 2),
                                      (300_007, 150_001, 48, 1)])
def test_lookback_carry_is_deterministic_under_perturbation(n, r, B, cw):
    _native.force_coef_words(cw)
    try:
        nb = (n + 7) // 8
        rng = np.random.default_rng(B)
        arr = rng.integers(0, 256, size=(3, B, nb), dtype=np.uint8)
        if n % 8:
            arr[:, :, -1] &= (1 << (n % 8)) - 1
        arr[1, :, 0] |= 1
        # block 1: x = 2^n - 1, c = d = 1 -> c*x + d = 2^n, a carry through every word
        # and every tile (all look-back predecessors pass the carry on)
        arr[0, 1] = 0xFF
        if n % 8:
            arr[0, 1, -1] = (1 << (n % 8)) - 1
        arr[1, 1], arr[2, 1] = 0, 0
        arr[1, 1, 0] = arr[2, 1, 0] = 1
        dx, dc, dd = (torch.from_numpy(a).cuda() for a in arr)
        eng = HashEngine(n, r, max_batch=B)
        ref = eng.hash_device(dx, dc, dd).cpu()
        side = torch.cuda.Stream()
        junk = torch.empty(1 << 24, device="cuda")
        for it in range(40):
            with torch.cuda.stream(side):  # perturb which CTAs are resident when
                junk.mul_(1.0001).add_(0.5)
            out = eng.hash_device(dx, dc, dd)
            assert torch.equal(out.cpu(), ref), f"run {it} differs"
        torch.cuda.synchronize()
        for i in (0, 1, B - 1):
            want = oracle.compress(arr[0, i].tobytes(), arr[1, i].tobytes(), arr[2, i].tobytes(), n, r)
            assert ref[i].numpy().tobytes() == want
    finally:
        _native.force_coef_words(0)
