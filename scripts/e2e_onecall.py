"""One hash_seeded_host call over steps x blocks (a key file): the exclusive seed
schedule vs the concurrent windows, by seed budget (development aid)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_04429_b200.batch import HashEngine  # noqa: E402

n, r, B, K = (int(float(v)) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (1e6, 5e5, 1024, 20)))
nb = (n + 7) // 8
px = torch.randint(0, 256, (B, nb), dtype=torch.uint8).repeat(K, 1).pin_memory()
ref = None
SL = [int(v) for v in (sys.argv[5].split(",") if len(sys.argv) > 5 else ["3"])]
for excl, budget_mb, slots in [(False, 4096, 3)] + [(True, mb, sl) for mb in (512, 1024, 2048, 4096) for sl in SL]:
    eng = HashEngine(n, r, max_batch=B)
    hout = torch.empty((K * B, eng.rbytes), dtype=torch.uint8).pin_memory()

    def call():
        eng.hash_seeded_host(px, None, 0, hout, seed_budget=budget_mb << 20, protocol="bench",
                             exclusive=excl, streams=slots)

    ts = []
    call()
    torch.cuda.synchronize()
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1) / K, 3))
    if ref is None:
        ref = hout.clone()
    print(json.dumps({"n": n, "r": r, "blocks": K * B, "exclusive": excl, "seed_budget_mb": budget_mb, "slots": slots,
                      "window_blocks": getattr(eng, "_xw_win", None), "ms_per_1024_blocks": ts,
                      "mbps_best": round(B * n / min(ts) / 1e3, 1),
                      "keys_equal_first_variant": bool(torch.equal(hout, ref))}), flush=True)
    del eng
    torch.cuda.empty_cache()
