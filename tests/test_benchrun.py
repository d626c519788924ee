"""run_bench protocol + report schema (pkg/src/modpa/bench.py:138-183, report.py:19-47)."""
import json

import pytest

from paper_1910_04429_b200 import benchrun
from paper_1910_04429_b200.benchrun import BenchRecord, bench_csv, bench_json, run_bench
from paper_1910_04429_b200.runpa import RunConfig

RECORDS = [
    BenchRecord(block_size=1_000_000, algorithm="ssa", trials=5, elapsed_median=0.2,
                throughput_mbps=5.0),
    BenchRecord(block_size=2_000_000, algorithm="ssa", trials=5, elapsed_median=0.5,
                throughput_mbps=4.0),
]


def test_csv_schema_matches_reference():
    # the reference's own expectations, pkg/tests/test_cli.py:166-176
    lines = bench_csv(RECORDS).strip().split("\n")
    assert lines[0] == "block_size,algorithm,trials,elapsed_ms,throughput_mbps"
    assert lines[1] == "1000000,ssa,5,200.0,5.0"
    doc = json.loads(bench_json(RECORDS))
    assert doc[0] == {"block_size": 1_000_000, "algorithm": "ssa", "trials": 5,
                      "elapsed_ms": 200.0, "throughput_mbps": 5.0}


def test_bench_inputs_are_the_reference_protocol(config_golden):
    import hashlib

    # bench_input(RunConfig(rng_seed=s), n) is the C-config x of seed s
    rec = config_golden["C1"]["blocks"][0]
    x = benchrun.bench_input(RunConfig(rng_seed=0), 1_000_000)
    assert hashlib.sha256(x.value.to_bytes(125_000, "little")).hexdigest() == rec["x"]


def test_unknown_scope_rejected():
    with pytest.raises(ValueError):
        run_bench(RunConfig(sizes=(64,), trials=1), scope="bogus")


@pytest.mark.gpu
@pytest.mark.parametrize("scope", ["pipeline", "multiply", "device"])
def test_run_bench_on_gpu(scope):
    recs = run_bench(RunConfig(sizes=(50_000, 100_000), trials=2), scope=scope)
    assert [r.block_size for r in recs] == [50_000, 100_000]
    assert all(r.algorithm == benchrun.ALGORITHM and r.throughput_mbps > 0 for r in recs)
    assert bench_csv(recs).startswith("block_size,algorithm,trials,elapsed_ms,throughput_mbps")


@pytest.mark.gpu
def test_run_bench_rounds_compute_the_reference_keys(monkeypatch):
    # run_bench only returns timings; spy on what each scope's timed call computed and
    # check it against the oracle (pipeline, device) or Python's own product (multiply)
    import oracle
    from paper_1910_04429_b200 import batch

    sizes = (50_000, 1_000_000)
    rounds, products, device = [], [], []
    real_round, real_mul, real_hash = benchrun.pa.pa_round, benchrun.mul, batch.HashEngine.hash_device

    def spy_round(block, params, seed, enforce=True):
        out = real_round(block, params, seed, enforce=enforce)
        rounds.append((block, params, seed, out))
        return out

    def spy_mul(a, b, *args, **kw):
        out = real_mul(a, b, *args, **kw)
        products.append((a, b, out))
        return out

    def spy_hash(self, x, c, d, *args, **kw):
        out = real_hash(self, x, c, d, *args, **kw)
        device.append((self.n, self.r, x, c, d, out))
        return out

    monkeypatch.setattr(benchrun.pa, "pa_round", spy_round)
    monkeypatch.setattr(benchrun, "mul", spy_mul)
    monkeypatch.setattr(batch.HashEngine, "hash_device", spy_hash)
    for scope in ("pipeline", "multiply", "device"):
        run_bench(RunConfig(sizes=sizes, trials=2), scope=scope)
    assert len(rounds) == 4 and len(products) == 4 and len(device) == 8
    for block, params, seed, out in rounds:
        nb = (params.n + 7) // 8
        want = oracle.compress(block.value.to_bytes(nb, "little"), seed.c.value.to_bytes(nb, "little"),
                               seed.d.value.to_bytes(nb, "little"), params.n, params.r)
        assert out.n == params.r and out.value == int.from_bytes(want, "little")
    for a, b, out in products:
        assert out.value == a.value * b.value
    import torch
    torch.cuda.synchronize()
    for n, r, x, c, d, out in device:
        want = oracle.compress(bytes(x[0].cpu().numpy()), bytes(c[0].cpu().numpy()),
                               bytes(d[0].cpu().numpy()), n, r)
        assert bytes(out[0].cpu().numpy()) == want
