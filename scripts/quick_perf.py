"""Quick device-resident throughput + per-kernel breakdown (development aid)."""
import os, sys, time, json
import torch
sys.path.insert(0, ".")
from paper_1910_04429_b200.batch import HashEngine
from paper_1910_04429_b200 import _native

cases = [(10**6, 5 * 10**5, 1024), (10**7, 2 * 10**6, 64), (10**8, 5 * 10**7, 8)]
if len(sys.argv) > 1:
    cases = [tuple(int(float(v)) for v in a.split(",")) for a in sys.argv[1:]]
modes = [int(v) for v in os.environ.get("QP_CW", "0").split(",")]
for n, r, B, cw in [(n, r, B, cw) for (n, r, B) in cases for cw in modes]:
    _native.force_coef_words(cw)
    try:
        _native.plan_info(n)
    except ValueError:
        continue
    nb = (n + 7) // 8
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randint(0, 256, (B, nb), dtype=torch.uint8, device="cuda", generator=g)
    c = torch.randint(0, 256, (B, nb), dtype=torch.uint8, device="cuda", generator=g)
    d = torch.randint(0, 256, (B, nb), dtype=torch.uint8, device="cuda", generator=g)
    eng = HashEngine(n, r, max_batch=B)
    out = eng.hash_device(x, c, d)
    torch.cuda.synchronize()
    for _ in range(2):
        eng.hash_device(x, c, d, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 5
    e0.record()
    for _ in range(K):
        eng.hash_device(x, c, d, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    _native.profile_enable(True)
    eng.hash_device(x, c, d, out)
    torch.cuda.synchronize()
    _native.profile_enable(False)
    prof = _native.profile_collect()
    print(json.dumps({"n": n, "r": r, "batch": B, "ms_per_batch": round(ms, 4),
                      "mbps": round(B * n / (ms * 1e-3) / 1e6, 1), "chunk": eng.chunk,
                      "plan": _native.plan_info(n), "width": _native.plan_width(n),
                      "kernels_ms": {k: round(v[1], 4) for k, v in prof.items()}}), flush=True)
