"""Randomised parity soak on the GPU (development aid): batched hashes of random ragged
sizes, ratios and structured operands against the direct formula with Python ints.
python scripts/soak.py [seconds] [seed]"""
import random
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1910_04429_b200.batch import HashEngine  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
t0 = time.time()
cases = blocks = 0


def operand(n, kind):
    if kind == 0:
        return rng.getrandbits(n)
    if kind == 1:
        return (1 << n) - 1
    if kind == 2:
        return rng.getrandbits(max(1, n // 64))  # small
    if kind == 3:
        return ((1 << n) - 1) ^ rng.getrandbits(max(1, n // 97))  # ones with low noise
    return (rng.getrandbits(n) >> (n // 2)) << (n // 2)  # low half zero


while time.time() - t0 < budget:
    # sizes around word, coefficient, tile and plan boundaries, and a few big ones
    base = rng.choice([64, 2048, 4096, 65536, 65600, 131072, 10**6, 3 * 10**6, 2**22, 10**7])
    n = max(1, base + rng.randint(-130, 130)) if rng.random() < 0.8 else rng.randint(1, 3 * 10**6)
    r = rng.choice([1, n, max(1, n // 2), rng.randint(1, n), max(1, n - rng.randint(0, 70))])
    B = rng.choice([1, 2, 3, 7]) if n > 10**6 else rng.choice([1, 2, 5, 33])
    nb, rb = (n + 7) // 8, (r + 7) // 8
    xs = [operand(n, rng.randrange(5)) for _ in range(B)]
    cs = [operand(n, rng.randrange(5)) | 1 for _ in range(B)]
    ds = [operand(n, rng.randrange(5)) for _ in range(B)]
    t = lambda vs: torch.from_numpy(np.frombuffer(b"".join(v.to_bytes(nb, "little") for v in vs),  # noqa: E731
                                                  np.uint8).reshape(B, nb).copy()).cuda()
    eng = HashEngine(n, r, max_batch=rng.choice([1, 2, B]))
    out = eng.hash_host(t(xs).cpu().pin_memory(), t(cs).cpu().pin_memory(), t(ds).cpu().pin_memory()) \
        if rng.random() < 0.3 else eng.hash_device(t(xs), t(cs), t(ds)).cpu()
    torch.cuda.synchronize()
    for j in range(B):
        want = (((cs[j] * xs[j] + ds[j]) & ((1 << n) - 1)) >> (n - r)).to_bytes(rb, "little")
        got = out[j].numpy().tobytes()
        if got != want:
            print("MISMATCH", {"n": n, "r": r, "B": B, "j": j}, flush=True)
            sys.exit(1)
    cases += 1
    blocks += B
print(f"soak ok: {cases} cases, {blocks} blocks in {time.time() - t0:.0f} s", flush=True)
