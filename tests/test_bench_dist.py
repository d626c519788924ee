"""Multi-rank host logic of bench.py on CPU (gloo, world_size 2): max-over-ranks
timing and the weak-scaling block-seed assignment (no GPU needed)."""
import os
import socket

import torch.multiprocessing as mp

import bench


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = bench.max_over_ranks(1.5 + rank, dist)
        seeds = bench.rank_seeds(tuple(range(4)), rank)
        q.put((rank, m, seeds))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_and_seed_shards_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(60)
    res = {r: (m, s) for r, m, s in (q.get(timeout=5) for _ in ps)}
    assert res[0][0] == res[1][0] == 2.5
    assert res[0][1] == [0, 1, 2, 3] and res[1][1] == [4, 5, 6, 7]


def test_kernel_model_positive():
    m = bench.kernel_model(10**6, 5 * 10**5, 1024) if os.path.exists(
        os.path.join(bench.ROOT, "paper_1910_04429_b200", "_lib", "libpa_b200.so")) else None
    if m:
        assert set(m) >= {"k_col_fwd", "k_row", "k_col_inv", "k_carry"}
        assert all(v["bytes"] > 0 for k, v in m.items() if k.startswith("k_"))


def test_gpus_flag_self_launches_ranks():
    # `python bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks
    # (torch.distributed.run on 127.0.0.1); --dry-run keeps it on CPU/gloo
    import json
    import subprocess
    import sys

    res = subprocess.run([sys.executable, os.path.join(bench.ROOT, "bench.py"), "--gpus", "2",
                          "--dry-run", "--steps", "3"], capture_output=True, text=True,
                         timeout=240, cwd=bench.ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"] is True
    assert d["max_over_ranks_check"] == 2.0  # rank 1 reported 2.0, rank 0 1.0
    assert d["rank0_seeds"] == [0, 1023]


def test_world_size_must_match_gpus():
    import subprocess
    import sys

    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, os.path.join(bench.ROOT, "bench.py"), "--gpus", "1",
                          "--dry-run"], capture_output=True, text=True, timeout=120, env=env,
                         cwd=bench.ROOT)
    assert res.returncode != 0 and "WORLD_SIZE=2" in res.stderr
