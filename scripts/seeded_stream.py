"""run_pa-scope streaming on the GPU (development aid): K streamed hash_seeded_host
calls vs one call over K x B blocks vs the pieces alone (seed expansion, hashing)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_04429_b200.batch import HashEngine  # noqa: E402

n, r, B, K = (int(float(v)) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (1e6, 5e5, 1024, 10)))
CH = int(sys.argv[5]) if len(sys.argv) > 5 else None  # hashing chunk (blocks per launch)
nb = (n + 7) // 8
eng = HashEngine(n, r, max_batch=B)
px = torch.randint(0, 256, (B, nb), dtype=torch.uint8).pin_memory()
hout = torch.empty((B, eng.rbytes), dtype=torch.uint8).pin_memory()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def streamed():
    for i in range(K):
        eng.hash_seeded_host(px, 0, 0, hout, join_in=i == 0, join_out=False, chunk=CH)
    eng.join()


big = px.repeat(K, 1).pin_memory()
bout = torch.empty((K * B, eng.rbytes), dtype=torch.uint8).pin_memory()
c = torch.empty((B, nb), dtype=torch.uint8, device="cuda")
d = torch.empty_like(c)
dx = px.cuda()
dout = torch.empty((B, eng.rbytes), dtype=torch.uint8, device="cuda")
res = {
    "streamed_ms_per_step": timed(streamed) / K,
    "one_call_ms_per_step": timed(lambda: eng.hash_seeded_host(big, 0, 0, bout)) / K,
    "seed_only_ms_per_step": timed(lambda: [eng.seed_device(0, i * B, B, c, d) for i in range(K)]) / K,
    "hash_only_ms_per_step": timed(lambda: [eng.hash_device(dx, c, d, dout) for _ in range(K)]) / K,
}
res = {k: round(v, 3) for k, v in res.items()}
res.update(n=n, r=r, B=B, K=K, chunk=CH, mbps_streamed=round(B * n / res["streamed_ms_per_step"] / 1e3, 1),
           mbps_one_call=round(B * n / res["one_call_ms_per_step"] / 1e3, 1))
print(json.dumps(res), flush=True)
