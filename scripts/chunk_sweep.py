"""Blocks per launch vs throughput for one 1024-block C2 batch (development aid):
smaller launches keep each launch's intermediate transforms L2-resident."""
import json, sys
import torch
sys.path.insert(0, ".")
from paper_1910_04429_b200.batch import HashEngine
from paper_1910_04429_b200 import _native

n, r, B = 1_000_000, 500_000, 1024
nb = n // 8
g = torch.Generator(device="cuda").manual_seed(0)
x, c, d = (torch.randint(0, 256, (B, nb), dtype=torch.uint8, device="cuda", generator=g) for _ in range(3))
for chunk in [int(v) for v in (sys.argv[1:] or ["1024", "512", "256", "128", "96", "64", "48", "32"])]:
    eng = HashEngine(n, r, max_batch=chunk)
    assert eng.chunk == chunk
    out = eng.hash_device(x, c, d)
    for _ in range(2):
        eng.hash_device(x, c, d, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        eng.hash_device(x, c, d, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    _native.profile_enable(True)
    eng.hash_device(x, c, d, out)
    torch.cuda.synchronize()
    _native.profile_enable(False)
    prof = _native.profile_collect()
    print(json.dumps({"chunk": chunk, "ms": round(ms, 4), "mbps": round(B * n / ms / 1e3),
                      "kernels_ms": {k: round(v[1], 4) for k, v in prof.items()}}), flush=True)
