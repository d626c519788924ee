"""The reference's benchmark protocol on the GPU, in its report schema.

Mirrors pkg/src/modpa/bench.py:138-183 (run_bench): deterministic inputs per
size (bench_input / gen_seed(n, derive_block_seed(rng_seed, n)),
bench.py:108-111, 156), `trials` rounds visited round-robin over the sizes,
median per size, throughput = n / median / 1e6 Mbps, sizes whose working set
does not fit skipped on MemoryError with a diagnostic.  Records serialize
with the reference's CSV/JSON schema (report.py:19-47).

Scopes:
  "pipeline"  import_block -> pa_round(enforce per cfg) -> export_block through
              the drop-in API (host ints, like the reference's timed round,
              bench.py:127-135);
  "multiply"  the product c*x only (bignum.mul on the GPU, bench.py:122-126);
  "device"    one block already resident in HBM through HashEngine (CUDA-event
              timed) -- the GPU's own cost without the Python int boundary.
"""
from __future__ import annotations

import json
import statistics
import sys
import time
from dataclasses import dataclass
from typing import Sequence

from . import pa
from .bignum import BigNat, mul
from .runpa import RunConfig, resolve_out_bits

BENCH_CSV_COLUMNS = ("block_size", "algorithm", "trials", "elapsed_ms", "throughput_mbps")
ALGORITHM = "b200-ntt"  # multi-prime NTT convolution on the GPU


@dataclass(frozen=True)
class BenchRecord:
    """One timing measurement at a single block size (bench.py:39-47)."""

    block_size: int
    algorithm: str
    trials: int
    elapsed_median: float  # seconds
    throughput_mbps: float


def bench_input(cfg: RunConfig, n: int) -> pa.BitBlock:
    """Deterministic pseudorandom n-bit benchmark block (bench.py:108-111)."""
    return pa.BitBlock(value=pa._expand(cfg.rng_seed, b"bench-input-%d" % n, n), n=n)


def _device_timer(state):
    import torch

    from .batch import HashEngine

    n, r = state["n"], state["params"].r
    nb = (n + 7) // 8
    if "eng" not in state:
        t = lambda v: torch.frombuffer(bytearray(v.to_bytes(nb, "little")),  # noqa: E731
                                       dtype=torch.uint8).view(1, -1).cuda()
        state["eng"] = HashEngine(n, r, max_batch=1)
        state["dev"] = (t(state["block"].value), t(state["seed"].c.value), t(state["seed"].d.value))
    eng, (dx, dc, dd) = state["eng"], state["dev"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.hash_device(dx, dc, dd)
    e0.record()
    eng.hash_device(dx, dc, dd)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e-3


def _timed_round(cfg: RunConfig, state: dict, scope: str) -> float:
    if scope == "device":
        return _device_timer(state)
    if scope == "multiply":
        x = BigNat(state["block"].value)
        t0 = time.perf_counter()
        mul(state["seed"].c, x)
        return time.perf_counter() - t0
    n = state["params"].n
    t0 = time.perf_counter()
    block = pa.import_block(state["raw"], n, cfg.order)
    out = pa.pa_round(block, state["params"], state["seed"], enforce=state["enforce"])
    pa.export_block(out, cfg.order)
    return time.perf_counter() - t0


def run_bench(cfg: RunConfig, *, quiet: bool = False, scope: str | None = None) -> list[BenchRecord]:
    """Median of `trials` rounds per size, sizes visited round-robin (bench.py:138-183)."""
    scope = scope or cfg.timing
    if scope not in ("pipeline", "multiply", "device"):
        raise ValueError(f"unknown timing scope {scope!r}")
    enforce = cfg.epsilon is not None and cfg.h_min is not None
    states: list[dict] = []
    for n in cfg.sizes:
        try:
            block = bench_input(cfg, n)
            states.append({
                "n": n, "block": block, "raw": pa.export_block(block, cfg.order),
                "seed": pa.gen_seed(n, pa.derive_block_seed(cfg.rng_seed, n)),
                "params": pa.PAParams(n=n, r=resolve_out_bits(cfg, n), epsilon=cfg.epsilon,
                                      h_min=cfg.h_min),
                "enforce": enforce, "elapsed": [],
            })
        except MemoryError:
            if not quiet:
                print(f"skipping block size {n}: not enough memory", file=sys.stderr)
    for _ in range(cfg.trials):
        for state in list(states):
            try:
                state["elapsed"].append(_timed_round(cfg, state, scope))
            except MemoryError:
                if not quiet:
                    print(f"skipping block size {state['n']}: not enough memory",
                          file=sys.stderr)
                states.remove(state)
    return [
        BenchRecord(block_size=s["n"], algorithm=ALGORITHM, trials=cfg.trials,
                    elapsed_median=statistics.median(s["elapsed"]),
                    throughput_mbps=s["n"] / statistics.median(s["elapsed"]) / 1e6)
        for s in states
    ]


def measure_ratio_spread(n: int, ratios: tuple[float, ...] = (0.125, 0.5, 0.9),
                         trials: int = 11, rng_seed: int = 0) -> dict[float, float]:
    """Best drop-in round time per compression ratio at one block size (bench.py:185-208).

    Trials interleave over the ratios; the first interleaved pass is warm-up
    and the minimum per ratio is reported (scheduling noise only adds).
    """
    cfg = RunConfig(sizes=(n,), rng_seed=rng_seed)
    raw = pa.export_block(bench_input(cfg, n), cfg.order)
    seed = pa.gen_seed(n, pa.derive_block_seed(rng_seed, n))
    best: dict[float, float] = {}
    for trial in range(trials + 1):
        for ratio in ratios:
            params = pa.PAParams(n=n, r=max(1, int(ratio * n)))
            t0 = time.perf_counter()
            out = pa.pa_round(pa.import_block(raw, n, cfg.order), params, seed, enforce=False)
            pa.export_block(out, cfg.order)
            dt = time.perf_counter() - t0
            if trial:
                best[ratio] = min(best.get(ratio, dt), dt)
    return best


def _bench_row(rec: BenchRecord) -> dict:
    return {"block_size": rec.block_size, "algorithm": rec.algorithm, "trials": rec.trials,
            "elapsed_ms": round(rec.elapsed_median * 1e3, 6),
            "throughput_mbps": round(rec.throughput_mbps, 6)}


def bench_csv(records: Sequence[BenchRecord]) -> str:
    """CSV in the reference's schema (report.py:19-43)."""
    lines = [",".join(BENCH_CSV_COLUMNS)]
    for rec in records:
        row = _bench_row(rec)
        lines.append(",".join(str(row[c]) for c in BENCH_CSV_COLUMNS))
    return "\n".join(lines) + "\n"


def bench_json(records: Sequence[BenchRecord]) -> str:
    """JSON mirroring the CSV fields (report.py:46-47)."""
    return json.dumps([_bench_row(r) for r in records], indent=2) + "\n"


if __name__ == "__main__":  # python -m paper_1910_04429_b200.benchrun [scope] [sizes...]
    args = sys.argv[1:]
    sc = args.pop(0) if args and args[0] in ("pipeline", "multiply", "device") else "pipeline"
    sizes = tuple(int(float(a)) for a in args) or (1_000_000, 10_000_000, 100_000_000)
    print(bench_csv(run_bench(RunConfig(sizes=sizes, trials=5), scope=sc)), end="")
