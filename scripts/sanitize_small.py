"""Small end-to-end exercise of every kernel path, for compute-sanitizer runs."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
from paper_1910_04429_b200 import _native
from paper_1910_04429_b200.batch import HashEngine
import paper_1910_04429_b200 as pab

rng = np.random.default_rng(1)
# tiny (host path), single-CTA, four-step m=1, m=5, m=3, and a 300-block batch (seq carry)
# + multi-tile look-back carries (k_carry_wide) over several blocks, the C2 shape
# (cp.async-staged all-primes forward columns) and the radix-3 1e8 plan's kernels at 3e7
for n, r, B in [(100, 33, 1), (30_000, 12_345, 2), (300_007, 150_001, 2), (2_229_060, 1_000_003, 1),
                (2_648_360, 333_333, 1), (65_600, 32_800, 300), (300_000, 150_011, 6),
                (1_000_000, 500_000, 4), (30_000_000, 15_000_007, 1)]:
    nb = (n + 7) // 8
    arr = rng.integers(0, 256, size=(3, B, nb), dtype=np.uint8)
    if n % 8:
        arr[:, :, -1] &= (1 << (n % 8)) - 1
    arr[1, :, 0] |= 1
    if B == 1 and n <= 2048:
        got = _native.hash_host(arr[0, 0].tobytes(), arr[1, 0].tobytes(), arr[2, 0].tobytes(), n, r)
        outs = [got]
    else:
        dx, dc, dd = (torch.from_numpy(a).cuda() for a in arr)
        o = HashEngine(n, r, max_batch=B).hash_device(dx, dc, dd).cpu().numpy()
        outs = [o[i].tobytes() for i in range(B)]
    for i in {0, B - 1}:
        assert outs[i] == oracle.compress(arr[0, i].tobytes(), arr[1, i].tobytes(),
                                          arr[2, i].tobytes(), n, r), (n, r, i)
    print("ok", n, r, B, _native.plan_info(n), flush=True)
x = pab.BitBlock(int(rng.integers(1, 1 << 62)), 70)
s = pab.gen_seed(70, 3)
pab.compress(x, s, 20)
assert pab.mul(3**2000, 7**1500).value == 3**2000 * 7**1500
print("sanitize script done")
# seed expansion (lane-pair Keccak) + the seeded host path, LSF and MSF, ragged n
for n, r, B, order in [(1089, 100, 3, _native.ORDER_LSF), (20_001, 777, 2, _native.ORDER_MSF)]:
    nb = (n + 7) // 8
    eng = HashEngine(n, r, order=order, max_batch=B)
    c = torch.empty((B, nb), dtype=torch.uint8, device="cuda")
    d = torch.empty_like(c)
    eng.seed_device(9, 5, B, c, d)
    torch.cuda.synchronize()
    endian = "big" if order == _native.ORDER_MSF else "little"
    for j in range(B):
        sd = pab.gen_seed(n, pab.derive_block_seed(9, 5 + j))
        assert c[j].cpu().numpy().tobytes() == sd.c.value.to_bytes(nb, endian)
        assert d[j].cpu().numpy().tobytes() == sd.d.value.to_bytes(nb, endian)
xs = rng.integers(0, 256, size=(2, 125_000), dtype=np.uint8)
_native.hash_seeded_host(xs.tobytes(), 1_000_000, 500_000, 2, 0, first_index=3)
print("seed paths done")
# the drop-in's Python-int digit path and the fused multiply-add
import random
rr = random.Random(4)
for n in (5_000, 300_001):
    xv, cv, dv = rr.getrandbits(n), rr.getrandbits(n) | 1, rr.getrandbits(n)
    got = _native.hash_ints(xv, cv, dv, n, n // 3)
    nb = (n + 7) // 8
    want = oracle.compress(xv.to_bytes(nb, "little"), cv.to_bytes(nb, "little"),
                           dv.to_bytes(nb, "little"), n, n // 3)
    assert got == int.from_bytes(want, "little")
acc, a, b = rr.getrandbits(90_000), rr.getrandbits(50_000), rr.getrandbits(40_000)
assert pab.fused_mul_add(acc, a, b).value == acc + a * b
print("digit path and mul_add done")
