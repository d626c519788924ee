"""Does splitting a batch over S streams (overlapping kernels of different chunks) help?"""
import sys, json
import torch
sys.path.insert(0, ".")
from paper_1910_04429_b200.batch import HashEngine

for n, r, B in [(10**6, 5 * 10**5, 1024), (10**8, 5 * 10**7, 8)]:
    nb = (n + 7) // 8
    g = torch.Generator(device="cuda").manual_seed(0)
    x, c, d = (torch.randint(0, 256, (B, nb), dtype=torch.uint8, device="cuda", generator=g) for _ in range(3))
    for S in (1, 2, 4):
        if B % S:
            continue
        eng = HashEngine(n, r, max_batch=B // S)
        sts = [torch.cuda.Stream() for _ in range(S)]
        outs = [torch.empty((B // S, (r + 7) // 8), dtype=torch.uint8, device="cuda") for _ in range(S)]
        def step():
            cur = torch.cuda.current_stream()
            for i, st in enumerate(sts):
                st.wait_stream(cur)
                sl = slice(i * B // S, (i + 1) * B // S)
                eng.hash_device(x[sl], c[sl], d[sl], outs[i], stream=st)
            for st in sts:
                cur.wait_stream(st)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(json.dumps({"n": n, "B": B, "streams": S, "ms": round(ms, 4),
                          "mbps": round(B * n / ms / 1e3, 1)}), flush=True)
