"""Seed windows in flight vs the streamed seeded e2e step (development aid):
python scripts/seed_window_sweep.py n r blocks steps -- one line per seed budget."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_04429_b200.batch import HashEngine  # noqa: E402

n, r, B, K = (int(float(v)) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (1e6, 5e5, 1024, 20)))
nb = (n + 7) // 8
px = torch.randint(0, 256, (B, nb), dtype=torch.uint8).pin_memory()
for budget_mb in [int(v) for v in (sys.argv[5].split(",") if len(sys.argv) > 5 else
                                   "512,768,1024,1536,2048,4096".split(","))]:
    eng = HashEngine(n, r, max_batch=B)
    hout = torch.empty((B, eng.rbytes), dtype=torch.uint8).pin_memory()

    def streamed():
        for i in range(K):
            eng.hash_seeded_host(px, None, 0, hout, join_in=i == 0, join_out=False,
                                 seed_budget=budget_mb << 20, protocol="bench")
        eng.join()

    ts = []
    for rep in range(4):
        streamed()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        streamed()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / K)
    print(json.dumps({"n": n, "r": r, "blocks": B, "steps": K, "seed_budget_mb": budget_mb,
                      "windows": eng._sw_key[0], "window_blocks": eng._sw_key[1],
                      "ms_per_step": [round(t, 3) for t in ts],
                      "mbps_best": round(B * n / min(ts) / 1e3, 1)}), flush=True)
    del eng
    torch.cuda.empty_cache()
