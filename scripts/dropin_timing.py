"""Per-call timing of the drop-in compress at tiny and 1e6 sizes (development aid)."""
import sys, time
sys.path.insert(0, ".")
import paper_1910_04429_b200 as pab

for alpha in (7, 64, 2048, 100_000, 1_000_000):
    x = pab.BitBlock(pab.pa._expand(1, b"x", alpha), alpha)
    s = pab.gen_seed(alpha, 5)
    r = max(1, alpha // 2)
    pab.compress(x, s, r)
    k = 20000 if alpha <= 2048 else 200
    t0 = time.perf_counter()
    for _ in range(k):
        pab.compress(x, s, r)
    dt = (time.perf_counter() - t0) / k
    for ratio in (0.125, 0.9):
        rr = max(1, int(alpha * ratio))
        t1 = time.perf_counter()
        for _ in range(min(k, 200)):
            pab.compress(x, s, rr)
        print(f"alpha={alpha} r/n={ratio}: {(time.perf_counter() - t1) / min(k, 200) * 1e6:.1f} us")
    print(f"alpha={alpha}: {dt * 1e6:.1f} us per compress", flush=True)
