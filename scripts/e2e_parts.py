"""Where the streamed seeded e2e step goes (development aid): the same pipeline with
the seed expansion and / or the hashing switched off."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_04429_b200.batch import HashEngine  # noqa: E402

n, r, B, K = (int(float(v)) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (1e6, 5e5, 1024, 20)))
nb = (n + 7) // 8
px = torch.randint(0, 256, (B, nb), dtype=torch.uint8).pin_memory()
res = {}
for name, seeds, hashing in (("full", True, True), ("no_seeds", False, True),
                             ("copies_only", False, False), ("seeds_and_copies", True, False)):
    eng = HashEngine(n, r, max_batch=B)
    hout = torch.empty((B, eng.rbytes), dtype=torch.uint8).pin_memory()
    if not seeds:
        eng.seed_device = lambda *a, **k: None
    if not hashing:
        eng.hash_device = lambda *a, **k: None

    def streamed():
        for i in range(K):
            eng.hash_seeded_host(px, None, 0, hout, join_in=i == 0, join_out=False, protocol="bench")
        eng.join()

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
