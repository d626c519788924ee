"""pab_hash_host (one C call; x, c, d from pinned host buffers) vs HashEngine.hash_host
on steps x blocks (development aid)."""
import ctypes
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1910_04429_b200 import _native  # noqa: E402
from paper_1910_04429_b200.batch import HashEngine  # noqa: E402

n, r, B, K = (int(float(v)) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (1e6, 5e5, 1024, 8)))
nb, rb = (n + 7) // 8, (r + 7) // 8
lib = _native.load()
x, c, d = (torch.randint(0, 256, (K * B, nb), dtype=torch.uint8).pin_memory() for _ in range(3))
c[:, 0] |= 1
out = torch.empty((K * B, rb), dtype=torch.uint8).pin_memory()
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
call = lambda: _native.check(lib.pab_hash_host(P(x), P(c), P(d), n, r, K * B, _native.ORDER_LSF, P(out), 0))  # noqa: E731
call()
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    call()
    ts.append(round((time.perf_counter() - t0) * 1e3 / K, 3))
eng = HashEngine(n, r, max_batch=B)
out2 = torch.empty_like(out).pin_memory()
eng.hash_host(x, c, d, out2)
torch.cuda.synchronize()
tp = []
for _ in range(3):
    t0 = time.perf_counter()
    eng.hash_host(x, c, d, out2)
    torch.cuda.synchronize()
    tp.append(round((time.perf_counter() - t0) * 1e3 / K, 3))
print(json.dumps({"n": n, "r": r, "blocks": K * B, "native_ms_per_step": ts, "engine_ms_per_step": tp,
                  "equal": bool(torch.equal(out, out2)),
                  "native_mbps": round(B * n / min(ts) / 1e3, 1)}), flush=True)
