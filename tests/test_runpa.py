"""Batched key-file hashing (runpa.run_pa) vs the reference's own run_pa output.

tests/golden/runpa.json holds key files hashed by modpa's bench.run_pa
(pkg/src/modpa/bench.py:223-265).  CPU tests drive run_pa's host logic
(validation, seed derivation, sharding, ordering, atomic write) with the
oracle as the per-batch hasher -- including a world_size-2 gloo run; the GPU
test uses the default CUDA hasher.
"""
import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_1910_04429_b200 import pa
from paper_1910_04429_b200.bignum import WordOrder
from paper_1910_04429_b200.runpa import RunConfig, run_pa, shard_range

HERE = os.path.dirname(os.path.abspath(__file__))


def load_cases():
    with open(os.path.join(HERE, "golden", "runpa.json")) as f:
        return json.load(f)["cases"]


def oracle_hasher(x, c, d, n, r, order):
    msf = order is WordOrder.MOST_SIGNIFICANT_FIRST
    out = oracle.compress_batch(np.ascontiguousarray(x).tobytes(), c.tobytes(), d.tobytes(),
                                n, r, x.shape[0], threads=4, msf=msf)
    return np.frombuffer(out, np.uint8).reshape(x.shape[0], -1)


def _cfg(case, tmp_path, tag=""):
    inp = tmp_path / f"key{tag}.bin"
    out = tmp_path / f"out{tag}.bin"
    inp.write_bytes(bytes.fromhex(case["data"]))
    return RunConfig(sizes=(case["n"],), rng_seed=case["rng_seed"], in_path=str(inp),
                     out_path=str(out), order=WordOrder(case["order"]), **case["kw"]), out


def test_run_pa_matches_reference_files(tmp_path):
    for i, case in enumerate(load_cases()):
        cfg, out = _cfg(case, tmp_path, str(i))
        res = run_pa(cfg, hasher=oracle_hasher, chunk_blocks=2)
        assert out.read_bytes().hex() == case["out"], case["n"]
        assert res.blocks == len(bytes.fromhex(case["data"])) // (case["n"] // 8)


def test_run_pa_validation(tmp_path):
    key = tmp_path / "k.bin"
    key.write_bytes(bytes(100))
    with pytest.raises(ValueError, match="exactly one"):
        run_pa(RunConfig(sizes=(64, 128), in_path=str(key), out_path=str(tmp_path / "o")),
               hasher=oracle_hasher)
    with pytest.raises(ValueError, match="whole number of bytes"):
        run_pa(RunConfig(sizes=(12,), in_path=str(key), out_path=str(tmp_path / "o")),
               hasher=oracle_hasher)
    with pytest.raises(ValueError, match="both an input and an output"):
        run_pa(RunConfig(sizes=(64,), in_path=str(key)), hasher=oracle_hasher)
    with pytest.raises(ValueError, match="shorter"):
        run_pa(RunConfig(sizes=(4096,), in_path=str(key), out_path=str(tmp_path / "o")),
               hasher=oracle_hasher)


def test_budget_violation_leaves_no_output(tmp_path):
    # pkg/tests/test_cli.py:128-135
    key = tmp_path / "k.bin"
    key.write_bytes(bytes(512))
    out = tmp_path / "out.bin"
    cfg = RunConfig(sizes=(4096,), out_bits=2000, epsilon=2**-40, h_min=1000.0,
                    in_path=str(key), out_path=str(out))
    with pytest.raises(pa.SecurityBoundError):
        run_pa(cfg, hasher=oracle_hasher)
    assert not out.exists()


def test_shard_ranges_cover_in_order():
    for nb in (1, 2, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            spans = [shard_range(nb, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nb
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, inp, outp, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = RunConfig(sizes=(case["n"],), rng_seed=case["rng_seed"], in_path=inp,
                        out_path=outp, order=WordOrder(case["order"]), **case["kw"])
        run_pa(cfg, hasher=oracle_hasher, dist=dist, chunk_blocks=1)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("which", [0, 3])
def test_run_pa_gloo_world2_matches_reference(tmp_path, which):
    case = load_cases()[which]
    inp = tmp_path / "key.bin"
    inp.write_bytes(bytes.fromhex(case["data"]))
    outp = tmp_path / "out.bin"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, str(inp), str(outp), q))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    results = dict(q.get(timeout=5) for _ in procs)
    assert results == {0: "ok", 1: "ok"}, results
    assert outp.read_bytes().hex() == case["out"]


@pytest.mark.gpu
def test_run_pa_gpu_matches_reference_files(tmp_path):
    # default path: key blocks to the GPU, seeds expanded there (pab_seed_expand)
    for i, case in enumerate(load_cases()):
        cfg, out = _cfg(case, tmp_path, str(i))
        run_pa(cfg)
        assert out.read_bytes().hex() == case["out"], case["n"]


@pytest.mark.gpu
def test_run_pa_gpu_host_seeds_matches_reference_files(tmp_path):
    from paper_1910_04429_b200.runpa import gpu_hasher

    for i, case in enumerate(load_cases()):
        cfg, out = _cfg(case, tmp_path, "h" + str(i))
        run_pa(cfg, hasher=gpu_hasher(), chunk_blocks=3)
        assert out.read_bytes().hex() == case["out"], case["n"]


@pytest.mark.gpu
def test_run_pa_gpu_long_seed_material(tmp_path):
    # seed material beyond the device expander's 1 KiB (an rng_seed >= 2^8192):
    # run_pa derives the seeds on the host instead and still hashes on the GPU
    big = (1 << 9000) + 12345
    rng = np.random.default_rng(9)
    key = tmp_path / "k.bin"
    key.write_bytes(rng.integers(0, 256, size=3 * 512, dtype=np.uint8).tobytes())
    outs = []
    for tag, kw in (("gpu", {}), ("oracle", {"hasher": oracle_hasher})):
        out = tmp_path / f"{tag}.bin"
        run_pa(RunConfig(sizes=(4096,), ratio=0.5, rng_seed=big, in_path=str(key),
                         out_path=str(out)), **kw)
        outs.append(out.read_bytes())
    assert outs[0] == outs[1] and len(outs[0]) == 3 * 256


@pytest.mark.gpu
@pytest.mark.parametrize("n,blocks,ratio", [(1_000_000, 40, 0.5), (4_160, 4_200, 0.25)])
def test_run_pa_gpu_at_config_size(tmp_path, n, blocks, ratio):
    # a key file of C2-size blocks (and one big enough for the seed windows to run on
    # the hashing stream: >= 4096 blocks), every key against the oracle on host-derived
    # seeds -- what the reference's run_pa computes block by block (bench.py:256-262)
    rng = np.random.default_rng(blocks)
    nb = n // 8
    data = rng.integers(0, 256, size=blocks * nb, dtype=np.uint8)
    key, out = tmp_path / "key.bin", tmp_path / "out.bin"
    key.write_bytes(data.tobytes())
    res = run_pa(RunConfig(sizes=(n,), ratio=ratio, rng_seed=77, in_path=str(key),
                           out_path=str(out)))
    r = max(1, int(ratio * n))
    rb = (r + 7) // 8
    got = out.read_bytes()
    assert res.blocks == blocks and len(got) == blocks * rb
    x = data.reshape(blocks, nb)
    step = 1 if n >= 1_000_000 else 97
    for i in list(range(0, blocks, step)) + [blocks - 1]:
        s = pa.gen_seed(n, pa.derive_block_seed(77, i))
        want = oracle.compress(x[i].tobytes(), s.c.value.to_bytes(nb, "little"),
                               s.d.value.to_bytes(nb, "little"), n, r)
        assert got[i * rb:(i + 1) * rb] == want, i
