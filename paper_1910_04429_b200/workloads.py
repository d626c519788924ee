"""Seeded synthetic PA workloads (the reference's bench protocol).

Block with seed s at size n (pkg/src/modpa/bench.py:108-111, 156):
    x      = _expand(s, b"bench-input-%d" % n, n)
    (c, d) = gen_seed(n, derive_block_seed(s, n))
All serialized LSF, ceil(n/8) bytes.  The configs are BASELINE.json's C1..C5.
No dataset is involved: the reference benchmarks SHAKE-derived pseudorandom
blocks, and these are exactly those blocks.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import pa

CONFIGS = {
    "C1": dict(n=1_000_000, ms=(500_000,), seeds=(0,)),
    "C2": dict(n=1_000_000, ms=(500_000,), seeds=tuple(range(1024))),
    "C3": dict(n=10_000_000, ms=(2_000_000,), seeds=tuple(range(64))),
    "C4": dict(n=100_000_000, ms=(50_000_000,), seeds=(7,)),
    "C5": dict(n=100_000_000, ms=(10_000_000, 50_000_000, 90_000_000), seeds=tuple(range(64))),
}


def block_inputs(n: int, s: int) -> tuple[bytes, bytes, bytes]:
    """(x, c, d) of block seed s at size n as ceil(n/8) LSF bytes each."""
    nb = (n + 7) // 8
    x = pa._expand(s, b"bench-input-%d" % n, n)
    seed = pa.gen_seed(n, pa.derive_block_seed(s, n))
    return (x.to_bytes(nb, "little"), seed.c.value.to_bytes(nb, "little"),
            seed.d.value.to_bytes(nb, "little"))


def batch_inputs(n: int, seeds, threads: int | None = None) -> tuple[np.ndarray, np.ndarray,
                                                                     np.ndarray]:
    """Three uint8 arrays [len(seeds), ceil(n/8)] (x, c, d), derived in parallel."""
    nb = (n + 7) // 8
    seeds = list(seeds)
    xs = np.empty((len(seeds), nb), np.uint8)
    cs = np.empty_like(xs)
    ds = np.empty_like(xs)

    def one(i):
        x, c, d = block_inputs(n, seeds[i])
        xs[i] = np.frombuffer(x, np.uint8)
        cs[i] = np.frombuffer(c, np.uint8)
        ds[i] = np.frombuffer(d, np.uint8)

    with ThreadPoolExecutor(threads or min(16, os.cpu_count() or 1)) as ex:
        list(ex.map(one, range(len(seeds))))
    return xs, cs, ds
