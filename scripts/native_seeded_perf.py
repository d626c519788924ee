"""pab_hash_seeded_host (one C call, host buffers) on a key file of steps x blocks
(development aid): pinned vs pageable host buffers."""
import ctypes
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1910_04429_b200 import _native  # noqa: E402

n, r, B, K = (int(float(v)) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (1e6, 5e5, 1024, 20)))
nb, rb = (n + 7) // 8, (r + 7) // 8
lib = _native.load()
m = _native.seed_material(0)
res = {}
for name, pin in (("pinned", True), ("pageable", False)):
    x = torch.randint(0, 256, (K * B, nb), dtype=torch.uint8)
    out = torch.empty((K * B, rb), dtype=torch.uint8)
    if pin:
        x, out = x.pin_memory(), out.pin_memory()
    call = lambda: _native.check(lib.pab_hash_seeded_host(  # noqa: E731
        ctypes.c_void_p(x.data_ptr()), n, r, K * B, _native.ORDER_LSF, m, len(m), 0,
        ctypes.c_void_p(out.data_ptr()), 0))
    call()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        call()
        ts.append(round((time.perf_counter() - t0) * 1e3 / K, 3))
    res[name] = {"ms_per_step": ts, "mbps_best": round(B * n / min(ts) / 1e3, 1)}
print(json.dumps({"n": n, "r": r, "blocks": K * B, "steps": K, "wall_clock": res}), flush=True)
