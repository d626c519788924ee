"""H2D bandwidth from pinned memory with k concurrent streams (development aid)."""
import json
import torch

nbytes = 384_000_000
h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
for k in (1, 2, 3, 4, 8):
    ss = [torch.cuda.Stream() for _ in range(k)]
    part = nbytes // k
    def go():
        cur = torch.cuda.current_stream()
        for i, s in enumerate(ss):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        for s in ss:
            cur.wait_stream(s)
    go(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        go()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(json.dumps({"streams": k, "ms": round(ms, 3), "GBps": round(nbytes / ms / 1e6, 1)}))
