"""Generate the golden fixtures for the PA hash path FROM THE REFERENCE ITSELF.

Run once in the build container (the reference is importable there, not on
the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed):
  tests/golden/configs.json  -- per block of configs C1..C5: SHA-256 of the
      derived inputs (x, c, d as ceil(n/8) LSF bytes) and of the output key
      (export_block LSF of compress), computed by `modpa`.
  tests/golden/small.json    -- raw hex vectors at small sizes (KATs, ragged
      n/r, MSF order, edge operands) plus full products for `mul`.

Input derivation is the reference's bench protocol:
  x      = pa._expand(s, b"bench-input-%d" % n, n)          pkg/src/modpa/bench.py:108-111
  (c, d) = pa.gen_seed(n, pa.derive_block_seed(s, n))        pkg/src/modpa/bench.py:156
For C5 the product is formed once per block with the reference primitives
fused_mul_add -> mod_pow2 and shift_right is applied per ratio; that this
equals compress is the reference's own test pkg/tests/test_pa.py:163-173.
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import time
from multiprocessing import Pool

from modpa import pa, bignum  # the reference (PYTHONPATH=/root/reference/pkg/src)
from modpa.bignum import BigNat, WordOrder

HERE = os.path.dirname(os.path.abspath(__file__))
LSF = WordOrder.LEAST_SIGNIFICANT_FIRST
MSF = WordOrder.MOST_SIGNIFICANT_FIRST

CONFIGS = {
    "C1": dict(n=1_000_000, ms=[500_000], seeds=[0]),
    "C2": dict(n=1_000_000, ms=[500_000], seeds=list(range(1024))),
    "C3": dict(n=10_000_000, ms=[2_000_000], seeds=list(range(64))),
    "C4": dict(n=100_000_000, ms=[50_000_000], seeds=[7]),
    "C5": dict(n=100_000_000, ms=[10_000_000, 50_000_000, 90_000_000], seeds=list(range(64))),
}


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def block_job(args):
    n, ms, s = args
    x = pa.BitBlock(pa._expand(s, b"bench-input-%d" % n, n), n)
    seed = pa.gen_seed(n, pa.derive_block_seed(s, n))
    nb = (n + 7) // 8
    rec = {
        "seed": s,
        "x": sha(x.value.to_bytes(nb, "little")),
        "c": sha(seed.c.value.to_bytes(nb, "little")),
        "d": sha(seed.d.value.to_bytes(nb, "little")),
        "out": {},
    }
    if len(ms) == 1:
        y = pa.compress(x, seed, ms[0])
        rec["out"][str(ms[0])] = sha(pa.export_block(y))
    else:
        t = bignum.mod_pow2(bignum.fused_mul_add(seed.d, seed.c, BigNat(x.value)), n)
        for m in ms:
            y = pa.BitBlock(bignum.shift_right(t, n - m).value, m)
            rec["out"][str(m)] = sha(pa.export_block(y))
    return rec


def gen_configs(procs: int) -> dict:
    out = {}
    for name, cfg in CONFIGS.items():
        t0 = time.time()
        jobs = [(cfg["n"], cfg["ms"], s) for s in cfg["seeds"]]
        with Pool(procs) as pool:
            recs = pool.map(block_job, jobs, chunksize=1)
        out[name] = {"n": cfg["n"], "ms": cfg["ms"], "blocks": recs}
        print(f"{name}: {len(recs)} blocks in {time.time() - t0:.1f}s", flush=True)
    return out


def hexb(v: int, nbytes: int, order=LSF) -> str:
    return v.to_bytes(nbytes, "little" if order is LSF else "big").hex()


def gen_small() -> dict:
    rng = random.Random(0x50A1)
    cases = []

    def add(n, r, c, d, x, order=LSF, tag=""):
        nb = (n + 7) // 8
        seed = pa.HashSeed(c=BigNat(c), d=BigNat(d), alpha=n)
        y = pa.compress(pa.BitBlock(x, n), seed, r)
        cases.append({
            "tag": tag, "n": n, "r": r, "order": order.value,
            "x": hexb(x, nb, order), "c": hexb(c, nb, order), "d": hexb(d, nb, order),
            "y": pa.export_block(y, order).hex(),
        })

    # the reference's worked examples, pkg/tests/test_pa.py:125-133
    add(4, 2, 3, 1, 5, tag="kat1")
    add(4, 2, 5, 2, 7, tag="kat2")
    # ragged n, r (including non-multiples of 8/32/64), random members
    for n in [1, 2, 3, 5, 7, 8, 9, 31, 32, 33, 63, 64, 65, 100, 127, 128, 129, 255,
              256, 257, 400, 511, 1000, 1023, 1024, 1025, 2047, 4095, 4096, 4097,
              10_000, 65_535, 65_536, 65_537, 100_000, 131_073]:
        for _ in range(2 if n < 65_536 else 1):
            r = rng.randrange(1, n + 1)
            s = pa.gen_seed(n, rng.randrange(1 << 30))
            x = rng.getrandbits(n)
            add(n, r, s.c.value, s.d.value, x, tag="ragged")
    # MSF byte order
    for n in [8, 12, 64, 100, 4096, 70_000]:
        r = max(1, n // 3)
        s = pa.gen_seed(n, rng.randrange(1 << 30))
        add(n, r, s.c.value, s.d.value, rng.getrandbits(n), order=MSF, tag="msf")
    # edge operands
    for n in [64, 1000, 65_536]:
        full = (1 << n) - 1
        add(n, n // 2, full, 1, 1, tag="fullcarry")          # c=2^n-1, x=1, d=1 -> 0
        add(n, n, 1, 0, rng.getrandbits(n), tag="identity")  # c=1, d=0 -> x
        add(n, n // 2, full, full, full, tag="allones")
        add(n, n // 2, full | 1, 0, 0, tag="zero")
        add(n, 1, full, full, full, tag="r1")
    # full products (bignum.mul), pkg/tests/test_bignum.py style
    prods = []
    w = (1 << 64) - 1
    pairs = [(w, w), (0, 5), (1, 98765), (3, 5)]
    for _ in range(40):
        a_bits = rng.choice([1, 17, 64, 100, 1000, 4096, 40_000, 100_003])
        b_bits = rng.choice([1, 17, 64, 130, 1000, 4096, 40_000])
        pairs.append((rng.getrandbits(a_bits), rng.getrandbits(b_bits)))
    for a, b in pairs:
        p = bignum.mul(a, b).value
        prods.append({"a": format(a, "x"), "b": format(b, "x"), "p": format(p, "x")})
    return {"hash": cases, "mul": prods}


def gen_runpa() -> dict:
    """Key files hashed by the reference's own batch driver (bench.run_pa, bench.py:223-265)."""
    import tempfile

    from modpa import bench

    rng = random.Random(0x9A)
    cases = []
    for n, nblocks, extra, kw, order in [
        (4096, 3, 0, dict(ratio=0.5), LSF),
        (64, 5, 3, dict(out_bits=32), LSF),
        (1024, 4, 0, dict(ratio=0.3), MSF),
        (100_000, 3, 7, dict(out_bits=33_333), LSF),
    ]:
        data = rng.randbytes(nblocks * n // 8 + extra)
        with tempfile.TemporaryDirectory() as td:
            inp, out = os.path.join(td, "key.bin"), os.path.join(td, "out.bin")
            open(inp, "wb").write(data)
            cfg = bench.RunConfig(sizes=(n,), rng_seed=rng.randrange(1000), in_path=inp,
                                  out_path=out, order=order, **kw)
            bench.run_pa(cfg)
            cases.append({"n": n, "rng_seed": cfg.rng_seed, "order": order.value,
                          "kw": kw, "data": data.hex(), "out": open(out, "rb").read().hex()})
    return {"cases": cases}


if __name__ == "__main__":
    if "--runpa-only" in sys.argv:
        with open(os.path.join(HERE, "runpa.json"), "w") as f:
            json.dump(gen_runpa(), f, indent=0)
        print("runpa done")
        sys.exit(0)
    procs = int(os.environ.get("GOLDEN_PROCS", os.cpu_count() or 1))
    small = gen_small()
    with open(os.path.join(HERE, "small.json"), "w") as f:
        json.dump(small, f, indent=0)
    print(f"small: {len(small['hash'])} hash cases, {len(small['mul'])} products", flush=True)
    if "--small-only" in sys.argv:
        sys.exit(0)
    cfgs = gen_configs(procs)
    with open(os.path.join(HERE, "configs.json"), "w") as f:
        json.dump(cfgs, f, indent=0)
    print("done", flush=True)
