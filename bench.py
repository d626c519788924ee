#!/usr/bin/env python
"""PA hash throughput on B200 (BASELINE.json metric: input Mbps, % of roofline, bit-exact).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2|C3|C4|C5] [--no-extra] [--no-cpu] [--dry-run]

A step hashes one batch of synthetic blocks (the reference's bench protocol,
SURVEY.md §8d).  Default workload C2: 1024 blocks/rank at n=1e6, r=5e5, block
seeds rank*1024 .. rank*1024+1023 (rank 0 = BASELINE's seeds 0..1023); weak
scaling (blocks shard by index, no collective on the data path).

`--gpus N` without torchrun re-launches itself as N ranks (torch.distributed.run,
127.0.0.1); under torchrun WORLD_SIZE must equal N.

`value`  : device-resident Mbps (inputs already in HBM), max-over-ranks time.
`e2e`    : same metric and the same blocks through the public batched API from
           pinned host memory, every copy inside the timed region: the key blocks x
           go H2D, each block's (c, d) -- BASELINE's per-block seeds, derived as the
           reference bench protocol does (gen_seed(n, derive_block_seed(s, n))) -- is
           expanded on the GPU, the keys come back D2H; bit-identical to `value`'s
           keys.  `e2e.xcd` ships x, c and d instead (the only e2e at n=1e8, where one
           seed stream is a ~0.3 s Keccak chain).
`e2e_run_pa`: run_pa's scope (n <= 1e7): only the key blocks x cross PCIe; each
           block's (c, d) is expanded on the GPU (SHAKE-256) beside the hashing.
`roofline`: the dominant kernel against the integer-issue roofline (148 SMs x
           128 int32 lanes/clk x the SM clock sampled under load), its executed
           instructions from the committed ncu counts of the same batch; HBM beside.
`n1e8`   : BASELINE configs[4] (C5): 64 blocks/rank at n=1e8, m/n 0.5 timed with its
           own e2e, cpu_baseline and roofline; m/n 0.1 and 0.9 as `ratio_sweep`.
`c1`, `c4`: BASELINE configs[0] / [3]: one n=1e6 / n=1e8 block, device latency.
`--impl reference`: the reference's CPU algorithm (the C port under oracle/,
           all host threads, rank 0 only) on the same 1024 C2 blocks per step.
`--dry-run`: CPU only (gloo): the launcher, rank plumbing and JSON line, no kernels.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PA input throughput (Mbps) at n=1e6 and n=1e8; % of NTT roofline; bit-exact"


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], None, set()
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names[1:], parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ model
def plan_geometry(n: int) -> dict:
    from paper_1910_04429_b200 import _native

    m, lg, lr, lc = _native.plan_info(n)
    cbits, primes = _native.plan_width(n)
    return {"m": m, "lg": lg, "lgR": lr, "lgC": lc, "L": m << lg, "K": (n + 31) // 32,
            "Kc": (n + cbits - 1) // cbits, "cw": cbits // 32, "P": primes}


def kernel_model(n: int, r: int, blocks: int) -> dict:
    """Algorithmic HBM bytes and integer ops per launch of each kernel.

    Bytes count what the kernel must move at least once; int ops count the
    canonical 7 ops per radix-2 butterfly (Harvey/Shoup lazy butterfly, 3 on
    the FMA pipe + 4 on the ALU pipe), 6 per Montgomery product, 8 per
    four-step twiddle application, 3 (9 for a 64-bit coefficient) per input
    reduction and a Garner CRT of 35 (3 primes) / 85 (5 primes) ops per
    coefficient plus 25 per output word for the carry.  K = words, Kc =
    coefficients (K / cw), P = NTT primes of the plan's mode.
    """
    g = plan_geometry(n)
    L, K, Kc, lgR, lgC, mr = g["L"], g["K"], g["Kc"], g["lgR"], g["lgC"], g["m"]
    nb, rb, mw = (n + 7) // 8, (r + 7) // 8, (r + 31) // 32
    P = g["P"]
    red_in = L * 3 + (Kc * 6 if g["cw"] == 2 else 0)
    crt = {3: 35, 5: 85}[P]
    rad = {1: 0, 3: 25, 5: 56}[mr]  # ops per radix-m group (incl. its twiddles)
    bf = lambda lg: (L // 2) * lg  # butterflies of one length-L transform restricted to lg stages
    m = {}
    m["k_pack"] = dict(bytes=blocks * 3 * (nb + 4 * K), ops=0)
    m["k_unpack"] = dict(bytes=blocks * (4 * mw + rb), ops=0)
    m["k_carry"] = dict(bytes=blocks * (P * 4 * Kc + 4 * K + 4 * mw),
                        ops=blocks * (Kc * crt + K * 25))
    if lgR == 0:
        m["k_row_single"] = dict(bytes=blocks * (2 * 4 * K + P * 4 * Kc),
                                 ops=blocks * P * (3 * bf(lgC) * 7 + L * 6 + 2 * red_in))
    else:
        m["k_col_fwd"] = dict(bytes=blocks * 2 * (4 * K + P * 4 * L),
                              ops=blocks * 2 * P * (bf(lgR) * 7 + red_in + (L // mr) * rad))
        m["k_row"] = dict(bytes=blocks * P * 3 * 4 * L,
                          ops=blocks * P * (3 * bf(lgC) * 7 + L * 6 + 3 * L * 8))
        m["k_col_inv"] = dict(bytes=blocks * P * (4 * L + 4 * Kc),
                              ops=blocks * P * (bf(lgR) * 7 + L * 4 + (L // mr) * rad))
    return m


SMS = 148            # B200 (2 dies x 74)
INT_LANES_PER_CLK = 128  # per SM: 4 SMSPs x (16-lane ALU pipe + 16-lane FMA pipe), 1 warp-instr/clk/SMSP


def peaks(sm_mhz: float | None = None) -> dict:
    """Roofline denominators: HBM from MEASURED_PEAKS.json (driver-measured copy
    bandwidth); the integer-issue peak is the hardware dispatch limit, 148 SMs x
    128 int32 lanes/clk at the SM clock sampled under load (else the measured max)."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    mp = {}
    if os.path.exists(path):
        with open(path) as f:
            mp = json.load(f)
    hbm = mp.get("hbm_gbs")
    src = "MEASURED_PEAKS.json" if hbm else "fallback B200_PROFILING.md"
    clk = sm_mhz or mp.get("sm_max_mhz") or 1965.0
    int_peak = SMS * INT_LANES_PER_CLK * clk * 1e6 / 1e12
    return {"hbm_gbs": hbm or 6650.0, "hbm_src": src, "int_tops": round(int_peak, 3),
            "sm_mhz": clk,
            "int_src": "%d SMs x %d int32 lanes/clk x %.0f MHz (hardware issue limit; the ALU "
                       "and FMA pipes are 64 lanes/clk/SM each)" % (SMS, INT_LANES_PER_CLK, clk)}


def ncu_counts(workload: str | None, batch: int | None) -> dict:
    """Per-launch ncu counters of each kernel, committed from a capture of the same
    workload at the same blocks per launch (profiles/ncu_counts.json, written by
    scripts/ncu_counts.py): executed warp instructions, issue-active, ALU / FMA pipe
    utilisation and DRAM bytes."""
    path = os.path.join(ROOT, "profiles", "ncu_counts.json")
    if not workload or not os.path.exists(path):
        return {}
    with open(path) as f:
        rec = json.load(f).get("workloads", {}).get(workload)
    if not rec or (batch is not None and rec.get("batch") != batch):
        return {}
    return rec


# ------------------------------------------------------------------ CPU arm
def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


PORT_NOTE = ("oracle/modpa_ssa.c: C restatement of the reference's SSA route "
             "(pkg/src/modpa/ntt.py); its Toom-3 band (bignum.py:275-323) is served by "
             "Karatsuba -- the same exact products, slightly different CPU cost")


def run_reference(args, cfg) -> dict:
    """The reference's algorithm on the host (oracle/ C port), all host threads, on
    the same blocks as the GPU arm's step (all 1024 C2 blocks: ~0.8 s per step on 16
    threads) unless that would not finish --steps K within ~3 minutes."""
    import oracle
    from paper_1910_04429_b200 import workloads

    n, r = cfg["n"], cfg["ms"][0]
    threads = cpu_threads()
    blocks = len(cfg["seeds"])
    xs, cs, ds = workloads.batch_inputs(n, cfg["seeds"])
    probe = min(blocks, 2 * threads)
    t0 = time.perf_counter()
    oracle.compress_batch(xs[:probe].tobytes(), cs[:probe].tobytes(), ds[:probe].tobytes(), n, r,
                          probe, threads)
    per_block = (time.perf_counter() - t0) / probe
    budget = 180.0 / max(1, args.steps + args.warmup)  # seconds per step
    per_step = max(1, min(blocks, int(budget / max(per_block, 1e-9))))
    xb, cb, db = (a[:per_step].tobytes() for a in (xs, cs, ds))
    for _ in range(args.warmup):
        oracle.compress_batch(xb, cb, db, n, r, per_step, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.compress_batch(xb, cb, db, n, r, per_step, threads)
    dt = time.perf_counter() - t0
    mbps = args.steps * per_step * n / dt / 1e6
    sample = f"{per_step} of the {blocks} {cfg['name']} blocks (n={n}, r={r}) per step"
    return {"value": mbps, "ms_per_step": dt / args.steps * 1e3, "threads": threads,
            "sample": sample, "same_config": per_step == blocks}


def cpu_gmp_sample(cfg, xs, cs, ds, blocks: int) -> dict | None:
    """Context row: the paper's own CPU method (GMP mpz sequence, oracle/gmp_ref.py)."""
    try:
        from oracle import gmp_ref
    except Exception:  # pragma: no cover
        return None
    if not gmp_ref.available():
        return None
    n, r = cfg["n"], cfg["ms"][0]
    threads = cpu_threads()
    rows = [(xs[i].tobytes(), cs[i].tobytes(), ds[i].tobytes()) for i in range(blocks)]
    t0 = time.perf_counter()
    gmp_ref.compress_batch([a for a, _, _ in rows], [b for _, b, _ in rows],
                           [c for _, _, c in rows], n, r, threads)
    dt = time.perf_counter() - t0
    return {"value": round(blocks * n / dt / 1e6, 2), "unit": "Mbps",
            "cores": min(threads, blocks), "kind": "gmp (paper's method, PAPER.md:205-267)",
            "sample": f"{blocks} blocks of {cfg['name']}, {dt:.2f}s wall"}


def cpu_baseline_sample(cfg, xs=None, cs=None, ds=None) -> dict:
    """Bounded sample of the workload on the oracle port (rank 0, N=1 only), all
    host threads (one block per thread at a time), plus the GMP context row."""
    import oracle
    from paper_1910_04429_b200 import workloads

    n, r = cfg["n"], cfg["ms"][0]
    threads = cpu_threads()
    blocks = min(len(cfg["seeds"]), cfg.get("cpu_blocks", 4 * threads))
    if xs is None:
        xs, cs, ds = workloads.batch_inputs(n, cfg["seeds"][:blocks])
    xs, cs, ds = xs[:blocks], cs[:blocks], ds[:blocks]
    t0 = time.perf_counter()
    out = oracle.compress_batch(xs.tobytes(), cs.tobytes(), ds.tobytes(), n, r, blocks, threads)
    dt = time.perf_counter() - t0
    gmp = cpu_gmp_sample(cfg, xs, cs, ds, blocks)
    return {"value": round(blocks * n / dt / 1e6, 2), "unit": "Mbps",
            "cores": min(threads, blocks), "kind": "port",
            "sample": f"{blocks} blocks of {cfg['name']} (n={n}, r={r}), {dt:.2f}s wall",
            "note": PORT_NOTE, "context_gmp": gmp, "_out": out, "_blocks": blocks}


# ------------------------------------------------------------------ GPU arm
def time_device(eng, dx, dc, dd, dout, steps, warmup, dist, profile=True):
    import torch
    from paper_1910_04429_b200 import _native

    for _ in range(warmup):
        eng.hash_device(dx, dc, dd, dout)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _native.profile_collect()
    _native.profile_enable(profile)
    e0.record(st)
    for _ in range(steps):
        eng.hash_device(dx, dc, dd, dout)
    e1.record(st)
    torch.cuda.synchronize()
    _native.profile_enable(False)
    prof = _native.profile_collect()
    if dist:
        dist.barrier()
    return e0.elapsed_time(e1), prof


def max_over_ranks(v: float, dist) -> float:
    """Max of a per-rank timing over all ranks (NCCL on GPUs, gloo on CPU)."""
    if not dist:
        return v
    import torch

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def rank_seeds(cfg_seeds, rank: int) -> list[int]:
    """Weak scaling: rank k hashes seeds k*B .. k*B+B-1 (rank 0 = BASELINE's seeds)."""
    per_rank = len(cfg_seeds)
    return [rank * per_rank + s for s in cfg_seeds]


def run_leg(args, cfg, rank, world, dist, steps) -> dict:
    """One workload on this rank's GPU: device-resident timing (the contract's
    `value`), determinism across steps, the streamed e2e leg from pinned host
    memory, run_pa's seeded e2e (n <= 1e7) and the m/n sweep (C5)."""
    import torch
    from paper_1910_04429_b200 import workloads
    from paper_1910_04429_b200.batch import HashEngine

    n, r = cfg["n"], cfg["ms"][0]
    per_rank = len(cfg["seeds"])
    seeds = rank_seeds(cfg["seeds"], rank)
    xs, cs, ds = workloads.batch_inputs(n, seeds)
    px, pc, pd = (torch.from_numpy(a).pin_memory() for a in (xs, cs, ds))
    dx, dc, dd = (t.cuda() for t in (px, pc, pd))
    chunk = cfg.get("chunk", per_rank)
    eng = HashEngine(n, r, max_batch=chunk, max_workspace=cfg.get("max_workspace", 4 << 30))
    dout = eng.hash_device(dx, dc, dd)
    torch.cuda.synchronize()
    first_out = dout.cpu()

    clk = ClockSampler(torch.cuda.current_device())
    clk.start()
    # K steps with a CUDA event pair around every kernel (the per-kernel durations of the
    # roofline), then the timed region proper: the same K steps without those events (8
    # event records per step stand between the launches and cost ~1% at C2, ~40% at C1)
    ms_ev, prof = time_device(eng, dx, dc, dd, dout, steps, args.warmup, dist)
    ms_ev = max_over_ranks(ms_ev / steps, dist)
    ms, _ = time_device(eng, dx, dc, dd, dout, steps, 1, dist, profile=False)
    ms_step = max_over_ranks(ms / steps, dist)
    bits_step = world * per_rank * n
    value = bits_step / (ms_step * 1e-3) / 1e6
    assert torch.equal(dout.cpu(), first_out), "keys changed across steps"

    # end to end through the public batched API from pinned host memory
    hout = torch.empty((per_rank, eng.rbytes), dtype=torch.uint8, pin_memory=True)
    for _ in range(max(1, args.warmup)):
        eng.hash_host(px, pc, pd, hout, streams=3, chunk=cfg.get("e2e_chunk"))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(steps):  # streamed: each step's head overlaps the previous tail
        eng.hash_host(px, pc, pd, hout, streams=3, chunk=cfg.get("e2e_chunk"),
                      join_in=i == 0, join_out=False)
    eng.join(st)
    e1.record(st)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / steps, dist)
    assert torch.equal(hout, first_out), "e2e keys differ from device-resident keys"
    # the PCIe bound of that leg: the same pinned H2D + D2H bytes, copies only
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(2, min(steps, 10))
    torch.cuda.synchronize()
    c0.record(st)
    s_in.wait_stream(st)
    s_out.wait_stream(st)
    for _ in range(reps):
        with torch.cuda.stream(s_in):
            dx.copy_(px, non_blocking=True)
            dc.copy_(pc, non_blocking=True)
            dd.copy_(pd, non_blocking=True)
        with torch.cuda.stream(s_out):
            hout.copy_(dout, non_blocking=True)
    st.wait_stream(s_in)
    st.wait_stream(s_out)
    c1.record(st)
    torch.cuda.synchronize()
    copy_ms = max_over_ranks(c0.elapsed_time(c1) / reps, dist)
    e2e_xcd = {"value": round(bits_step / (e2e_ms * 1e-3) / 1e6, 1), "unit": "Mbps",
               "h2d_bytes_per_step": 3 * per_rank * eng.nbytes,
               "d2h_bytes_per_step": per_rank * eng.rbytes, "ms_per_step": round(e2e_ms, 4),
               "copy_only_ms_per_step": round(copy_ms, 4),
               "h2d_gbps": round(3 * per_rank * eng.nbytes / (e2e_ms * 1e-3) / 1e9, 1),
               "frac_of_copy_bound": round(copy_ms / e2e_ms, 4),
               "scope": "HashEngine.hash_host: pinned x, c, d -> GPU, keys -> pinned host, "
                        "consecutive steps streamed"}
    # headline e2e (n <= 1e7): the same blocks, only the key blocks x cross PCIe; each
    # block's (c, d) = gen_seed(n, derive_block_seed(s, n)) -- BASELINE's per-block
    # seeds, the reference bench protocol -- is expanded on the GPU in the timed region.
    # At 1e8 one seed stream is a 92K-permutation chain (~0.3 s), so there the e2e is
    # the (x, c, d) copy path.
    e2e = e2e_xcd
    if n <= 10_000_000 and seeds == list(range(seeds[0], seeds[0] + per_rank)):
        sout = torch.empty(hout.shape, dtype=torch.uint8, pin_memory=True)
        for _ in range(max(1, args.warmup)):
            eng.hash_seeded_host(px, None, seeds[0], sout, protocol="bench")
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for i in range(steps):
            eng.hash_seeded_host(px, None, seeds[0], sout, join_in=i == 0, join_out=False,
                                 protocol="bench")
        eng.join(st)
        e1.record(st)
        torch.cuda.synchronize()
        c_ms = max_over_ranks(e0.elapsed_time(e1) / steps, dist)
        assert torch.equal(sout, first_out), "seeded e2e keys differ from device-resident keys"
        per_call = {"value": round(bits_step / (c_ms * 1e-3) / 1e6, 1), "unit": "Mbps",
                    "ms_per_step": round(c_ms, 4),
                    "scope": "one hash_seeded_host call per step (the step's seeds repeated), "
                             "calls streamed; expansion and hashing share the GPU"}
        # the e2e: the K steps as ONE call over K x per_rank blocks (a key file handed to
        # the engine, as run_pa does): block j's seed is seeds[0] + j, x repeats the step's
        # key blocks.  Calls this size expand each seed window on the hashing stream right
        # before its chunks (the two do not share the SMs); H2D and D2H overlap both.
        from paper_1910_04429_b200 import batch as _batch
        one_call = (steps * per_rank >= _batch.kExclusiveMin and
                    (4 << 30) // (2 * eng.nbytes) >= _batch.kExclusiveMin)
    if n <= 10_000_000 and seeds == list(range(seeds[0], seeds[0] + per_rank)) and not one_call:
        # calls too small (or blocks too long) for the exclusive seed schedule: the
        # streamed per-step calls are the e2e
        e2e = dict(per_call, h2d_bytes_per_step=per_rank * eng.nbytes,
                   d2h_bytes_per_step=per_rank * eng.rbytes, xcd=e2e_xcd)
        e2e["scope"] = ("HashEngine.hash_seeded_host(protocol='bench'): pinned x -> GPU, each "
                        "block's (c, d) = gen_seed(n, derive_block_seed(s, n)) expanded on the "
                        "GPU (SHAKE-256), keys -> pinned host, consecutive steps streamed; keys "
                        "bit-identical to the device-resident leg")
    elif n <= 10_000_000 and seeds == list(range(seeds[0], seeds[0] + per_rank)):
        # (at most kCallSteps steps per call, so the pinned key file stays a few GB
        # whatever --steps is: K steps = ceil(K / kCallSteps) calls back to back)
        groups = call_groups(steps)
        pbig = px.repeat(max(groups), 1).pin_memory()
        sbig = torch.empty((max(groups) * per_rank, eng.rbytes), dtype=torch.uint8,
                           pin_memory=True)

        def calls(grp=groups):  # each a synchronous call: the engine hands it to the C-ABI
            t = 0               # pipeline, pab_hash_seeded_host_bench (host buffers in, keys out)
            for g in grp:       # (every call's keys land in the same host buffer)
                eng.hash_seeded_host(pbig[:g * per_rank], None, seeds[0] + t * per_rank,
                                     sbig[:g * per_rank], protocol="bench")
                t += g

        calls()  # warm-up (buffers)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0.record(st)
        calls()
        e1.record(st)
        torch.cuda.synchronize()
        s_ms = max_over_ranks(e0.elapsed_time(e1) / steps, dist)
        calls(groups[:1])  # the first call once more, its keys checked step by step
        torch.cuda.synchronize()
        assert torch.equal(sbig[:per_rank], first_out), \
            "seeded e2e keys differ from device-resident keys"
        vc, vd = torch.empty_like(dx), torch.empty_like(dx)
        for t in range(1, groups[0]):  # later steps: seeds expanded and hashed device-resident
            eng.seed_device(None, seeds[0] + t * per_rank, per_rank, vc, vd, protocol="bench")
            want = eng.hash_device(dx, vc, vd).cpu()
            assert torch.equal(sbig[t * per_rank:(t + 1) * per_rank], want), \
                "seeded e2e keys of step %d differ from the device-resident path" % t
        del pbig, vc, vd
        e2e = {"value": round(bits_step / (s_ms * 1e-3) / 1e6, 1), "unit": "Mbps",
               "h2d_bytes_per_step": per_rank * eng.nbytes,
               "d2h_bytes_per_step": per_rank * eng.rbytes, "ms_per_step": round(s_ms, 4),
               "calls": len(groups),
               "scope": "HashEngine.hash_seeded_host(protocol='bench') -> one C-ABI call "
                        "(pab_hash_seeded_host_bench: host buffers in, keys out) over the "
                        "%d steps' %d blocks (at most 32 steps per call): pinned x -> GPU, "
                        "block j's (c, d) = gen_seed(n, "
                        "derive_block_seed(s0 + j, n)) expanded on the GPU (SHAKE-256), keys -> "
                        "pinned host; checked on the first call: its first step's keys "
                        "bit-identical to the device-resident leg, its other steps' to the "
                        "device-resident path on the same seeds"
                        % (steps, steps * per_rank),
               "per_step_calls": per_call, "xcd": e2e_xcd}
    clocks = clk.stop()  # sampled across the device-resident and the e2e timed regions

    e2e_seeded = run_pa_e2e(args, eng, px, per_rank, rank, n, bits_step, dist, steps) \
        if n <= 10_000_000 else None

    sweep = None
    if len(cfg["ms"]) > 1:  # C5 (BASELINE configs[4]): m/n in {0.1, 0.5, 0.9}, same blocks
        sweep = []
        for rr in cfg["ms"][1:]:
            e_r = HashEngine(n, rr, max_batch=chunk, max_workspace=cfg.get("max_workspace", 4 << 30))
            o_r = e_r.hash_device(dx, dc, dd)
            k = max(3, min(steps, 10))
            ms_r, _ = time_device(e_r, dx, dc, dd, o_r, k, 3, dist, profile=False)
            ms_r = max_over_ranks(ms_r / k, dist)
            sr = step_roofline(n, rr, per_rank, ms_r, clocks.get("sm_mhz"))
            sweep.append({"r": rr, "ratio": round(rr / n, 3),
                          "value": round(bits_step / (ms_r * 1e-3) / 1e6, 1),
                          "ms_per_step": round(ms_r, 4), "steps": k,
                          "step_roofline_frac": sr["frac"]})
            del e_r, o_r
    return {"ms_step": ms_step, "ms_step_events": ms_ev, "value": value, "prof": prof,
            "clocks": clocks, "e2e": e2e,
            "e2e_seeded": e2e_seeded, "ratio_sweep": sweep, "out": first_out,
            "per_rank": per_rank, "n": n, "r": r, "eng": eng, "seeds": seeds, "steps": steps,
            "inputs": (xs, cs, ds), "chunk": eng.chunk}


kCallSteps = 32  # steps handed to one hash_seeded_host call in the e2e legs


def call_groups(steps: int) -> list[int]:
    """K steps as ceil(K / kCallSteps) calls of nearly equal size."""
    k = -(-steps // kCallSteps)
    return [steps // k + (1 if i < steps % k else 0) for i in range(k)]


def run_pa_e2e(args, eng, px, per_rank, rank, n, bits_step, dist, steps) -> dict:
    """run_pa's scope end to end (pkg/src/modpa/bench.py:256-262): the key blocks
    from pinned host memory, block i hashed with gen_seed(n, derive_block_seed(0, i))
    expanded on the GPU (HashEngine.hash_seeded_host), keys back to the host.  Only
    x crosses PCIe.  Rank k hashes run_pa blocks k*B .. k*B+B-1."""
    import torch
    from paper_1910_04429_b200 import pa

    from paper_1910_04429_b200 import batch as _batch

    # calls big enough for the exclusive seed schedule: one call over the K steps' blocks,
    # as run_pa hands a rank its whole shard (rank k hashes run_pa blocks k*K*B ..
    # (k+1)*K*B - 1, x repeats the step's key blocks); else one streamed call per step
    one_call = (steps * per_rank >= _batch.kExclusiveMin and
                (4 << 30) // (2 * eng.nbytes) >= _batch.kExclusiveMin)
    groups = call_groups(steps) if one_call else [1]
    reps = max(groups)
    first = rank * per_rank * reps
    total = per_rank * reps
    pbig = px.repeat(reps, 1).pin_memory() if one_call else px
    hout = torch.empty((total, eng.rbytes), dtype=torch.uint8, pin_memory=True)
    for _ in range(1 if one_call else max(1, args.warmup)):
        eng.hash_seeded_host(pbig, 0, first, hout, streams=3)  # warm-up (buffers)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    if one_call:
        for g in groups:  # (each call re-hashes the file's first g steps; synchronous calls:
            # the engine hands each to the C-ABI pipeline, pab_hash_seeded_host)
            eng.hash_seeded_host(pbig[:g * per_rank], 0, first, hout[:g * per_rank])
    else:
        for i in range(steps):
            eng.hash_seeded_host(pbig, 0, first, hout, streams=3, join_in=i == 0, join_out=False)
        eng.join(st)
    e1.record(st)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, dist)
    # spot check: blocks against host-derived seeds through the device path
    nb = eng.nbytes
    idx = [0, per_rank - 1, total - 1]
    dx = pbig[idx].cuda()
    del pbig
    dc = torch.empty((len(idx), nb), dtype=torch.uint8)
    dd = torch.empty_like(dc)
    for j, i in enumerate(idx):
        sd = pa.gen_seed(n, pa.derive_block_seed(0, first + i))
        dc[j] = torch.frombuffer(bytearray(sd.c.value.to_bytes(nb, "little")), dtype=torch.uint8)
        dd[j] = torch.frombuffer(bytearray(sd.d.value.to_bytes(nb, "little")), dtype=torch.uint8)
    want = eng.hash_device(dx, dc.cuda(), dd.cuda()).cpu()
    assert torch.equal(hout[idx], want), "run_pa e2e keys differ from host-derived seeds"
    return {"value": round(bits_step / (ms * 1e-3) / 1e6, 1), "unit": "Mbps",
            "scope": "run_pa: %s; x pinned host -> GPU, (c, d) = "
                     "gen_seed(n, derive_block_seed(0, i)) expanded on the GPU (SHAKE-256), "
                     "keys -> host" % ("one call over the %d steps' blocks" % steps if one_call
                                       else "one streamed call per step"),
            "h2d_bytes_per_step": per_rank * nb, "d2h_bytes_per_step": per_rank * eng.rbytes,
            "ms_per_step": round(ms, 4)}


def roofline_obj(prof: dict, n: int, r: int, blocks: int, workload: str | None,
                 sm_mhz: float | None) -> tuple[dict, dict]:
    """The contract's `roofline` for the dominant kernel plus a per-kernel table.

    The NTT kernels are integer-pipe bound (HBM < 0.5), so `bound` is "int":
    achieved = executed thread-instructions per launch (ncu smsp__inst_executed x 32,
    same workload and batch) / the live CUDA-event launch time, peak = the hardware
    issue limit at the sampled clock.  frac is therefore the kernel's issue-slot
    occupancy and should agree with ncu's issue-active.  The algorithmic-op rate
    (DESIGN.md §4 cost model) and the HBM fraction of the algorithmic bytes sit beside.
    """
    model = kernel_model(n, r, blocks)
    pk = peaks(sm_mhz)
    cnt = ncu_counts(workload, blocks)
    kcnt = cnt.get("kernels", {})
    total = sum(v[1] for v in prof.values()) or 1.0
    kernels = {}
    for name, (c, ms) in prof.items():
        avg_s = ms / max(c, 1) * 1e-3
        mdl = model.get(name, {"bytes": 0, "ops": 0})
        k = {"launches": c, "avg_ms": round(avg_s * 1e3, 4), "share": round(ms / total, 4),
             "GBps": round(mdl["bytes"] / avg_s / 1e9, 1),
             "alg_Tops": round(mdl["ops"] / avg_s / 1e12, 2)}
        if name in kcnt:
            k["issue_frac"] = round(kcnt[name]["inst"] * 32 / avg_s / 1e12 / pk["int_tops"], 4)
            k["fmaheavy_frac_ncu"] = kcnt[name].get("pipe_fmaheavy")
        kernels[name] = k
    if not prof:
        return None, kernels
    dom = max(prof.items(), key=lambda kv: kv[1][1])[0]
    c, ms = prof[dom]
    avg_s = ms / max(c, 1) * 1e-3
    mdl = model.get(dom, {"bytes": 0, "ops": 0})
    gbps = mdl["bytes"] / avg_s / 1e9
    hbm = {"achieved": round(gbps, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
           "frac": round(gbps / pk["hbm_gbs"], 4), "peak_src": pk["hbm_src"],
           "algorithmic_bytes_per_launch": mdl["bytes"]}
    alg = {"ops_per_launch": mdl["ops"], "achieved": round(mdl["ops"] / avg_s / 1e12, 3),
           "unit": "Tops/s", "frac_of_issue_peak": round(mdl["ops"] / avg_s / 1e12 / pk["int_tops"], 4),
           "model": "DESIGN.md §4: 7 ops per radix-2 butterfly, 6 per Montgomery product, "
                    "8 per four-step twiddle, CRT 85 (5 primes) / 35 (3) per coefficient"}
    kc = kcnt.get(dom)
    if kc:
        ops = kc["inst"] * 32
        ach = ops / avg_s / 1e12
        roof = {"bound": "int", "kernel": dom, "achieved": round(ach, 3), "peak": pk["int_tops"],
                "unit": "Tops/s", "frac": round(ach / pk["int_tops"], 4),
                "traffic": kc.get("dram_bytes"), "peak_src": pk["int_src"],
                "ops_per_launch": ops,
                "ops_src": "smsp__inst_executed.sum x 32 of %s (profiles/ncu_counts.json: %s, "
                           "%d blocks/launch)" % (dom, workload, blocks),
                "ncu": {x: kc.get(x) for x in ("issue_active", "pipe_alu", "pipe_fma",
                                                "pipe_fmaheavy", "duration_ms", "sm_mhz")},
                "hbm": hbm, "algorithmic": alg,
                "binding": dict({"resource": "fma-heavy pipe (IMAD, IMAD.HI, IMAD.WIDE: every "
                                             "integer multiply; 64 lanes/clk/SM)",
                                 "frac_ncu": kc.get("pipe_fmaheavy")},
                                **mix_ceiling(ach / pk["int_tops"]))}
    else:  # no matching capture committed: report the algorithmic HBM fraction only
        roof = dict(hbm, bound="hbm", kernel=dom, traffic=None, algorithmic=alg,
                    note="no ncu counts for this workload/batch: int fraction unavailable")
    return roof, kernels


def mix_ceiling(issue_frac: float) -> dict:
    """The issue fraction a stream of Shoup butterflies can reach at all: measured
    per-instruction pipe costs (scripts/pipe_rates.cu -> profiles/r2/pipe_rates.json):
    IMAD 2 clk per warp per SMSP, IMAD.HI and IMAD.WIDE 4, so a Shoup product holds the
    FMA pipe 8 clk and a 6-instruction butterfly cannot issue above 6/8 of the slots."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2", "pipe_rates.json")) as f:
            pr = json.load(f)
        ceil_frac = 6.0 * pr["shoup_products"]
    except (OSError, ValueError, KeyError):
        return {}
    return {"pipe_clk_per_warp_instr": {k: round(1.0 / pr[k], 2) for k in
                                        ("imad", "imad_hi", "imad_wide", "iadd3", "viaddmnmx", "lop3")},
            "shoup_product_clk": round(1.0 / pr["shoup_products"], 2),
            "butterfly_clk_ideal_stream": round(1.0 / pr["butterflies"], 2),
            "issue_ceiling_butterfly_mix": round(ceil_frac, 4),
            "issue_frac_of_ceiling": round(issue_frac / ceil_frac, 4),
            "src": "profiles/r2/pipe_rates.json (scripts/pipe_rates.cu on this B200 pool)"}


def step_roofline(n: int, r: int, blocks: int, ms_step: float, sm_mhz: float | None,
                  workload: str | None = None, chunk: int | None = None) -> dict:
    """North-star roofline of a whole step: the slower of (the step's algorithmic int
    ops at the hardware issue peak) and (its algorithmic HBM bytes at the measured
    copy bandwidth), vs the measured step time; plus, where the ncu counts of this
    batch are committed, the executed instructions at the same peak (issue_frac)."""
    pk = peaks(sm_mhz)
    model = kernel_model(n, r, blocks)
    ops = sum(v["ops"] for v in model.values())
    byts = sum(v["bytes"] for v in model.values())
    t_int = ops / (pk["int_tops"] * 1e12) * 1e3
    t_hbm = byts / (pk["hbm_gbs"] * 1e9) * 1e3
    t_roof = max(t_int, t_hbm)
    out = {"t_int_ms": round(t_int, 4), "t_hbm_ms": round(t_hbm, 4), "t_roof_ms": round(t_roof, 4),
           "measured_ms": round(ms_step, 4), "frac": round(t_roof / ms_step, 4),
           "bound": "int" if t_int >= t_hbm else "hbm",
           "roofline_mbps": round(blocks * n / t_roof / 1e3, 1),
           "peak": {"int_tops": pk["int_tops"], "hbm_gbs": pk["hbm_gbs"]}}
    cnt = ncu_counts(workload, chunk or blocks).get("kernels", {})
    if cnt:
        launches = max(1, blocks // (chunk or blocks))
        inst = sum(v["inst"] for v in cnt.values()) * 32 * launches
        out["issue_frac"] = round(inst / (pk["int_tops"] * 1e12) * 1e3 / ms_step, 4)
    return out


def baseline_roofline(n: int, r: int, blocks: int, ms_step: float, sm_mhz: float | None) -> dict:
    """BASELINE.md §4's frozen yardstick: the canonical G16 design (Goldilocks prime,
    16-bit coefficients, 26 ops per radix-2 butterfly, 2 HBM passes per NTT) at the
    hardware int issue peak and the measured HBM bandwidth.  This design does far
    fewer ops per bit (5 primes x 64-bit coefficients, 7-op Shoup butterflies), so
    its frac exceeds 1 without any skipped work."""
    pk = peaks(sm_mhz)
    K = -(-n // 16)
    L = 1 << (2 * K - 2).bit_length()
    lg = L.bit_length() - 1
    ops = 3 * (L // 2) * lg * 26 + 16 * L + 12 * K
    byts = 80 * L + 3 * n // 8 + r // 8
    t_int = blocks * ops / (pk["int_tops"] * 1e12) * 1e3
    t_hbm = blocks * byts / (pk["hbm_gbs"] * 1e9) * 1e3
    t_roof = max(t_int, t_hbm)
    return {"design": "G16 (BASELINE.md §4)", "L": L, "int_ops_per_block": ops,
            "hbm_bytes_per_block": byts, "t_roof_ms": round(t_roof, 4),
            "measured_ms": round(ms_step, 4), "frac": round(t_roof / ms_step, 4),
            "bound": "int" if t_int >= t_hbm else "hbm",
            "roofline_mbps": round(blocks * n / t_roof / 1e3, 1)}


def dropin_timing(n: int, r: int, calls: int = 10) -> dict:
    """Timing scope (iii) of SURVEY §8d: the drop-in Python call the reference's
    users make, pa.compress(BitBlock, HashSeed, r), including int <-> bytes and
    the host <-> device copies, one block per call (median of `calls`)."""
    import paper_1910_04429_b200 as pab
    from paper_1910_04429_b200 import workloads

    x = workloads.block_inputs(n, 0)[0]
    xb = pab.import_block(x, n)
    seed = pab.gen_seed(n, pab.derive_block_seed(0, n))  # the reference's derivation (untimed)
    pab.compress(xb, seed, r)
    ts = []
    for _ in range(calls):
        t0 = time.perf_counter()
        pab.compress(xb, seed, r)
        ts.append(time.perf_counter() - t0)
    ms = sorted(ts)[len(ts) // 2] * 1e3
    return {"value": round(n / (ms * 1e-3) / 1e6, 1), "unit": "Mbps", "ms_per_call": round(ms, 3),
            "scope": "pa.compress(BitBlock, HashSeed, r): one n=%d block per call, incl. "
                     "int<->bytes and host<->device copies (median of %d)" % (n, calls)}


def leg_line(args, cfg, res, world, cpu=None) -> dict:
    """The JSON fields of one measured workload."""
    n, r, per_rank = res["n"], res["r"], res["per_rank"]
    sm = res["clocks"].get("sm_mhz")
    roof, kernels = roofline_obj(res["prof"], n, r, res["chunk"], cfg["name"], sm)
    return {
        "value": round(res["value"], 1), "unit": "Mbps", "ms_per_step": round(res["ms_step"], 4),
        "steps": res["steps"],
        "with_kernel_events": {
            "ms_per_step": round(res["ms_step_events"], 4),
            "value": round(res["value"] * res["ms_step"] / res["ms_step_events"], 1),
            "note": "the same K steps, run right before the timed region, with a CUDA event "
                    "pair around every kernel launch: the source of `kernels` and of the "
                    "roofline's launch durations"},
        "config": {"workload": cfg["name"], "n": n, "r": r, "blocks_per_rank": per_rank,
                   "blocks_per_launch": res["chunk"],
                   "block_seeds": "rank*%d + 0..%d" % (per_rank, per_rank - 1),
                   "parallelism": f"blocks sharded by index over {world} GPU(s), no collective",
                   "l2": "inputs %.0f MB/rank > 126 MB L2 (no flush needed)"
                         % (3 * per_rank * ((n + 7) // 8) / 1e6),
                   "timing": "K steps between CUDA events on the launching stream, barrier + "
                             "synchronize on both sides, max over ranks; the per-kernel event "
                             "pairs run over the K steps before (with_kernel_events)"},
        "e2e": res["e2e"], "e2e_run_pa": res["e2e_seeded"],
        "gpu_launches": sum(v[0] for v in res["prof"].values()),
        "roofline": roof,
        "step_roofline": step_roofline(n, r, per_rank, res["ms_step"], sm, cfg["name"],
                                       res["chunk"]),
        "baseline_roofline": baseline_roofline(n, r, per_rank, res["ms_step"], sm),
        "kernels": kernels, "clocks": res["clocks"], "cpu_baseline": cpu,
        "ratio_sweep": res["ratio_sweep"],
    }


def cpu_leg(cfg, res) -> dict:
    """cpu_baseline of a leg on its own blocks, with the bit-exactness check."""
    xs, cs, ds = res["inputs"]
    cpu = cpu_baseline_sample(cfg, xs, cs, ds)
    k = cpu.pop("_blocks")
    cpu_out = cpu.pop("_out")
    cpu["bit_exact_vs_gpu"] = cpu_out == res["out"][:k].numpy().tobytes()
    return cpu


def single_leg(args, dist, name: str = "C4") -> dict:
    """A single-block config: BASELINE configs[0] (C1: n=1e6, seed 0) or configs[3]
    (C4: n=1e8, seed 7) -- device latency of one block's hash, per-kernel times and
    the drop-in compress call on the same block."""
    import torch
    from paper_1910_04429_b200 import workloads
    from paper_1910_04429_b200.batch import HashEngine

    cfg = workloads.CONFIGS[name]
    n, r = cfg["n"], cfg["ms"][0]
    xs, cs, ds = workloads.batch_inputs(n, cfg["seeds"])
    dx, dc, dd = (torch.from_numpy(a).cuda() for a in (xs, cs, ds))
    eng = HashEngine(n, r, max_batch=1)
    dout = eng.hash_device(dx, dc, dd)
    steps = max(3, min(args.steps, 20))
    # the latency without the per-kernel events (at one 1e6-bit block they cost ~40% and
    # stand between the programmatic dependent launches), then the same steps with them
    ms, _ = time_device(eng, dx, dc, dd, dout, steps, 3, dist, profile=False)
    ms = max_over_ranks(ms / steps, dist)
    ms_prof, prof = time_device(eng, dx, dc, dd, dout, steps, 1, dist)
    roof, kernels = roofline_obj(prof, n, r, 1, name, None)
    out = {"workload": f"{name}: 1 block, n={n}, r={r}, seed {cfg['seeds'][0]}",
           "ms_per_block": round(ms, 4),
           "ms_per_block_with_kernel_events": round(ms_prof / steps, 4),
           "value": round(n / (ms * 1e-3) / 1e6, 1), "unit": "Mbps", "steps": steps,
           "kernels": kernels, "roofline": roof}
    if not args.no_extra and (not dist or dist.get_rank() == 0):
        out["dropin"] = dropin_timing(n, r, calls=3 if n > 10_000_000 else 10)
    return out


def relaunch(args) -> int:
    """--gpus N outside torchrun: run this script as N ranks (one per GPU)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def dry_run(args, rank, world) -> None:
    """CPU-only check of the multi-rank plumbing (gloo): barrier, max-over-ranks,
    block shards, one JSON line from rank 0.  Measures nothing."""
    import torch.distributed as tdist

    dist = None
    if world > 1:
        tdist.init_process_group("gloo")
        dist = tdist
        dist.barrier()
    from paper_1910_04429_b200.workloads import CONFIGS

    seeds = rank_seeds(CONFIGS[args.config]["seeds"], rank)
    t = max_over_ranks(float(rank + 1), dist)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "value": None, "unit": "Mbps",
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "max_over_ranks_check": t, "rank0_seeds": [seeds[0], seeds[-1]],
                          "config": {"workload": args.config}}), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=["C2", "C3", "C4", "C5"])
    ap.add_argument("--no-extra", action="store_true", help="skip the n=1e8 legs and drop-in timing")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline legs")
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo plumbing check, no kernels")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, local_rank, world = dist_env()
    under_launcher = "WORLD_SIZE" in os.environ
    if args.gpus > 1 and not under_launcher and args.impl == "ours":
        sys.exit(relaunch(args))
    if under_launcher and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        return dry_run(args, rank, world)

    from paper_1910_04429_b200.workloads import CONFIGS

    cfg = dict(CONFIGS[args.config])
    cfg["name"] = args.config
    if args.config in ("C4", "C5"):
        cfg["cpu_blocks"] = cpu_threads()
        cfg["chunk"] = 64            # one launch per 64-block step (10.5 GiB workspace)
        cfg["max_workspace"] = 12 << 30
        cfg["e2e_chunk"] = 2
        if args.config == "C5":
            cfg["ms"] = (50_000_000, 10_000_000, 90_000_000)  # main line m/n = 0.5, then the sweep
    elif args.config == "C3":
        cfg["cpu_blocks"] = 16
        cfg["e2e_chunk"] = 8
    else:
        cfg["e2e_chunk"] = 128
        cfg["cpu_blocks"] = 1024

    if args.impl == "reference":
        if rank != 0:
            return
        ref = run_reference(args, cfg)
        line = {"metric": METRIC, "impl": "reference", "value": round(ref["value"], 2),
                "unit": "Mbps", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ref["ms_per_step"], 3),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "u32", "data": "synthetic (SHAKE-256 seeded blocks, reference bench protocol)",
                "config": {"workload": cfg["name"], "n": cfg["n"], "r": cfg["ms"][0],
                           "blocks_per_step": ref["sample"], "same_config": ref["same_config"]},
                "cpu_baseline": {"value": round(ref["value"], 2), "unit": "Mbps",
                                 "cores": ref["threads"], "kind": "port",
                                 "sample": ref["sample"], "note": PORT_NOTE},
                "e2e": {"value": round(ref["value"], 2), "unit": "Mbps",
                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    # development switches for exercising the N-rank path on a one-GPU box: every rank
    # on cuda:0 (PAB_BENCH_SAME_DEVICE=1) with host-side collectives (PAB_BENCH_BACKEND=gloo)
    dev = 0 if os.environ.get("PAB_BENCH_SAME_DEVICE") == "1" else local_rank
    backend = os.environ.get("PAB_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as tdist

        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            tdist.init_process_group(backend)
        dist = tdist
    solo = rank == 0 and world == 1

    res = run_leg(args, cfg, rank, world, dist, args.steps)
    cpu = cpu_leg(cfg, res) if solo and not args.no_cpu else None
    line = leg_line(args, cfg, res, world, cpu)
    line["dropin"] = dropin_timing(res["n"], res["r"]) if solo and not args.no_extra else None
    eng = res.pop("eng")
    del res, eng
    torch.cuda.empty_cache()

    side = {}
    if not args.no_extra and args.config == "C2":
        c5 = dict(CONFIGS["C5"], name="C5", ms=(50_000_000, 10_000_000, 90_000_000),
                  chunk=64, max_workspace=12 << 30, e2e_chunk=2, cpu_blocks=cpu_threads())
        r5 = run_leg(args, c5, rank, world, dist, max(3, min(args.steps, 10)))
        cpu5 = cpu_leg(c5, r5) if solo and not args.no_cpu else None
        side["n1e8"] = leg_line(args, c5, r5, world, cpu5)
        del r5
        torch.cuda.empty_cache()
        side["c4"] = single_leg(args, dist, "C4")
        side["c1"] = single_leg(args, dist, "C1")

    if rank == 0:
        out = {"metric": METRIC, "value": line.pop("value"), "unit": "Mbps", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": line.pop("ms_per_step"), "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "u32",
               "data": "synthetic (SHAKE-256 seeded blocks, reference bench protocol)"}
        line.pop("steps")
        out.update(line)
        out.update(side)
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
