"""Stream priorities of the seeded e2e pipeline (development aid)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_04429_b200 import batch  # noqa: E402
from paper_1910_04429_b200.batch import HashEngine  # noqa: E402

n, r, B, K = (int(float(v)) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (1e6, 5e5, 1024, 20)))
nb = (n + 7) // 8
px = torch.randint(0, 256, (B, nb), dtype=torch.uint8).pin_memory()
res = {}
for name, seed_prio, comp_prio in (("default", 0, 0), ("seeds_high", -1, 0), ("hash_high", 0, -1)):
    eng = HashEngine(n, r, max_batch=B)
    hout = torch.empty((B, eng.rbytes), dtype=torch.uint8).pin_memory()
    eng._pipe = (torch.cuda.Stream(eng.device), torch.cuda.Stream(eng.device, priority=comp_prio),
                 torch.cuda.Stream(eng.device))
    orig = torch.cuda.Stream

    def mk(*a, **k):
        return orig(*a, priority=seed_prio, **k)

    def streamed():
        for i in range(K):
            eng.hash_seeded_host(px, None, 0, hout, join_in=i == 0, join_out=False, protocol="bench")
        eng.join()

    torch.cuda.Stream = mk  # the seed window streams are created on first use
    try:
        streamed()
    finally:
        torch.cuda.Stream = orig
    ts = []
    for rep in range(3):
        streamed()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        streamed()
        e1.record()
        torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1) / K, 3))
    res[name] = ts
    del eng
    torch.cuda.empty_cache()
print(json.dumps({"n": n, "r": r, "blocks": B, "steps": K, "ms_per_step": res}), flush=True)
