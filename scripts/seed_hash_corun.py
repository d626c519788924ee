"""Seed expansion and hashing sharing the GPU, no copies (development aid)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_04429_b200.batch import HashEngine  # noqa: E402

n, r, B, K = (int(float(v)) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (1e6, 5e5, 1024, 32)))
NW = int(sys.argv[5]) if len(sys.argv) > 5 else 8
nb = (n + 7) // 8
eng = HashEngine(n, r, max_batch=B)
dx = torch.randint(0, 256, (B, nb), dtype=torch.uint8, device="cuda")
bufs = [(torch.empty((B, nb), dtype=torch.uint8, device="cuda"), torch.empty((B, nb), dtype=torch.uint8, device="cuda"),
         torch.cuda.Stream(), torch.cuda.Event(), torch.cuda.Event()) for _ in range(NW)]
dout = torch.empty((B, eng.rbytes), dtype=torch.uint8, device="cuda")
s_comp = torch.cuda.Stream()


def run(seeds, hashing):
    for i in range(K):
        c, d, st, ready, free = bufs[i % NW]
        if seeds:
            st.wait_event(free)
            eng.seed_device(None, 0, B, c, d, stream=st, protocol="bench")
            ready.record(st)
        if hashing:
            if seeds:
                s_comp.wait_event(ready)
            eng.hash_device(dx, c, d, dout, stream=s_comp)
            free.record(s_comp)
    for b in bufs:
        torch.cuda.current_stream().wait_stream(b[2])
    torch.cuda.current_stream().wait_stream(s_comp)


res = {}
for name, a, b in (("seeds_only", True, False), ("hash_only", False, True), ("both", True, True)):
    ts = []
    for rep in range(3):
        run(a, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(a, b)
        e1.record()
        torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1) / K, 3))
    res[name] = ts
print(json.dumps({"n": n, "r": r, "blocks": B, "steps": K, "windows": NW, "ms_per_step": res}), flush=True)
