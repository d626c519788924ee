"""Seed expansion on the GPU: k_seed_expand time per batch, and the run_pa-style
e2e (x only over PCIe, seeds on the device) vs the (x, c, d) host path (development aid)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_04429_b200 import _native  # noqa: E402
from paper_1910_04429_b200.batch import HashEngine  # noqa: E402

cases = [(10**6, 5 * 10**5, 1024), (10**7, 2 * 10**6, 64), (10**8, 5 * 10**7, 16)]
if len(sys.argv) > 1:
    cases = [tuple(int(float(v)) for v in a.split(",")) for a in sys.argv[1:]]


def timed(fn, k=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


for n, r, B in cases:
    nb = (n + 7) // 8
    eng = HashEngine(n, r, max_batch=min(B, 256 if n <= 10**6 else 16))
    c = torch.empty((B, nb), dtype=torch.uint8, device="cuda")
    d = torch.empty_like(c)
    seed_ms = timed(lambda: eng.seed_device(0, 0, B, c, d), k=2)
    x = torch.randint(0, 256, (B, nb), dtype=torch.uint8).pin_memory()
    hc = torch.randint(0, 256, (B, nb), dtype=torch.uint8).pin_memory()
    hd = torch.randint(0, 256, (B, nb), dtype=torch.uint8).pin_memory()
    out = torch.empty((B, (r + 7) // 8), dtype=torch.uint8).pin_memory()
    host_ms = timed(lambda: eng.hash_host(x, hc, hd, out))
    seeded_ms = timed(lambda: eng.hash_seeded_host(x, 0, 0, out))
    print(json.dumps({"n": n, "r": r, "batch": B, "chunk": eng.chunk,
                      "seed_expand_ms": round(seed_ms, 3),
                      "e2e_xcd_ms": round(host_ms, 3), "e2e_xcd_mbps": round(B * n / host_ms / 1e3),
                      "e2e_seeded_ms": round(seeded_ms, 3),
                      "e2e_seeded_mbps": round(B * n / seeded_ms / 1e3)}), flush=True)
