"""Where a drop-in compress call at n=1e6 spends its time (development aid)."""
import ctypes, sys, time
sys.path.insert(0, ".")
import torch
import paper_1910_04429_b200 as pab
from paper_1910_04429_b200 import _native, _pyint
from paper_1910_04429_b200.batch import HashEngine

n, r = 1_000_000, 500_000
x = pab.BitBlock(pab.pa._expand(1, b"x", n), n)
s = pab.gen_seed(n, 5)


def best(f, k=300):
    f()
    b = 1e9
    for _ in range(k):
        t0 = time.perf_counter()
        f()
        b = min(b, time.perf_counter() - t0)
    return round(b * 1e6, 1)


lib = _native.load()
xa, xn = _pyint.digits(x.value)
ca, cn = _pyint.digits(s.c.value)
da, dn = _pyint.digits(s.d.value)
ond = (r + 29) // 30
out, oa = _pyint.new_uninit(ond)
print("compress", best(lambda: pab.compress(x, s, r)))
print("hash_ints", best(lambda: _native.hash_ints(x.value, s.c.value, s.d.value, n, r)))
print("C pab_hash_digits", best(lambda: lib.pab_hash_digits(xa, xn, ca, cn, da, dn, n, r, oa, ond, 0)))
print("_device()", best(lambda: _native._device()))
eng = HashEngine(n, r, max_batch=1)
nb = n // 8
dx = torch.zeros((1, nb), dtype=torch.uint8, device="cuda")
dc = dx.clone(); dd = dx.clone()
dc[0, 0] = 1
out_d = eng.hash_device(dx, dc, dd)
def dev():
    eng.hash_device(dx, dc, dd, out_d)
    torch.cuda.synchronize()
print("device hash + sync (1 block)", best(dev))
