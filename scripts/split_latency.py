"""Single-block latency: pab_hash_host vs pab_hash_host_split over k shares (development aid).
On one GPU the shares share the device, so this measures the split's overhead (gather +
carry-only pass); the latency gain needs the shares on different GPUs."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1910_04429_b200 import _native  # noqa: E402

n, r = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000, None
r = n // 2
nb = (n + 7) // 8
rng = np.random.default_rng(0)
x, c, d = (rng.integers(0, 256, nb, dtype=np.uint8).tobytes() for _ in range(3))
ndev = torch.cuda.device_count()


def t(fn, k=5):
    fn()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return round(1e3 * sorted(ts)[len(ts) // 2], 3)


res = {"n": n, "gpus": ndev, "host_ms": t(lambda: _native.hash_host(x, c, d, n, r))}
for k in (1, 2, 5):
    res[f"split{k}_same_gpu_ms"] = t(lambda: _native.hash_host_split(x, c, d, n, r, devices=[0] * k))
if ndev > 1:
    res["split_all_gpus_ms"] = t(lambda: _native.hash_host_split(x, c, d, n, r,
                                                                 devices=list(range(ndev))))
print(json.dumps(res))
