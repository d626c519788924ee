"""Per-call timing of the drop-in pieces at 1e6 bits by compression ratio (development aid)."""
import sys, time
sys.path.insert(0, ".")
import paper_1910_04429_b200 as pab

n = 1_000_000
x = pab.BitBlock(pab.pa._expand(1, b"x", n), n)
raw = pab.export_block(x)
s = pab.gen_seed(n, 5)


def best(f, k=200):
    f()
    b = 1e9
    for _ in range(k):
        t0 = time.perf_counter()
        f()
        b = min(b, time.perf_counter() - t0)
    return b * 1e6


print("import_block", round(best(lambda: pab.import_block(raw, n)), 1), "us")
for ratio in (0.125, 0.5, 0.9):
    r = int(n * ratio)
    out = pab.compress(x, s, r)
    print(ratio, "compress", round(best(lambda: pab.compress(x, s, r)), 1),
          "export", round(best(lambda: pab.export_block(out)), 1),
          "round", round(best(lambda: pab.export_block(pab.pa_round(pab.import_block(raw, n), pab.PAParams(n=n, r=r), s, enforce=False))), 1))
