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
