"""Per-call latency of the drop-in compress() at small sizes (development aid)."""
import sys, time, random
sys.path.insert(0, ".")
import paper_1910_04429_b200 as pab
rng = random.Random(1)
for n, calls in ((4, 2000), (64, 2000), (1024, 2000), (4096, 1000), (100_000, 300), (1_000_000, 100)):
    x = pab.BitBlock(rng.getrandbits(n), n)
    s = pab.gen_seed(n, 5)
    r = max(1, n // 2)
    pab.compress(x, s, r)
    t0 = time.perf_counter()
    for _ in range(calls):
        pab.compress(x, s, r)
    dt = (time.perf_counter() - t0) / calls
    print(f"compress n={n:>8}: {dt * 1e6:8.1f} us/call")
