"""Batched key-file hashing: the reference's `run_pa` on B200.

Mirrors pkg/src/modpa/bench.py:50-105 (RunConfig, resolve_out_bits) and
pkg/src/modpa/bench.py:223-265 (run_pa): same validation and messages, same
per-block seeds gen_seed(n, derive_block_seed(rng_seed, i)), same output
layout (ceil(r/8) bytes per block, concatenated in block order, byte order
cfg.order), and the output file is written only after every block succeeded.

What changes is the execution: blocks are hashed in batches on the GPU
(HashEngine: many blocks per launch, copies overlapped on streams), seeds are
derived on host threads, and under torch.distributed the blocks are sharded
by contiguous index ranges over the ranks (one GPU each); rank 0 gathers the
keys in block order and writes the file.  The gather is the only exchange and
it happens once, after hashing (there is none on the data path).
"""
from __future__ import annotations

import os
import sys
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from pathlib import Path
from typing import Callable

import numpy as np

from . import _native, pa, security
from .bignum import DEFAULT_THRESHOLDS, MulAlgorithm, ThresholdTable, WordOrder

DEFAULT_SIZE_LADDER = (
    1_000_000, 2_000_000, 4_000_000, 8_000_000, 10_000_000,
    16_000_000, 32_000_000, 64_000_000, 100_000_000,
)


@dataclass(frozen=True)
class RunConfig:
    """Subcommand configuration (pkg/src/modpa/bench.py:50-95)."""

    sizes: tuple[int, ...] = DEFAULT_SIZE_LADDER
    out_bits: int | None = None
    ratio: float | None = None
    epsilon: float | None = None
    h_min: float | None = None
    rng_seed: int = 0
    in_path: str | None = None
    out_path: str | None = None
    report_format: str = "csv"
    alg: MulAlgorithm = MulAlgorithm.AUTO
    thresholds: ThresholdTable = DEFAULT_THRESHOLDS
    order: WordOrder = WordOrder.LEAST_SIGNIFICANT_FIRST
    trials: int = 5
    timing: str = "pipeline"
    # accepted for drop-in compatibility (bench.py:72-76); plots and the
    # universality audit are outside the hash path and ignore-only here
    plot: bool = True
    alpha: int = 6
    beta: int = 3
    seed_sample: int | None = None

    def __post_init__(self) -> None:
        if self.out_bits is not None and self.ratio is not None:
            raise ValueError("give either an output bit count or a ratio, not both")
        if self.ratio is not None and not 0 < self.ratio <= 1:
            raise ValueError(f"ratio must lie in (0, 1], got {self.ratio}")
        if self.out_bits is not None and self.out_bits < 1:
            raise ValueError(f"output bit count must be >= 1, got {self.out_bits}")
        if self.trials < 1:
            raise ValueError(f"trials must be >= 1, got {self.trials}")
        if self.timing not in ("pipeline", "multiply"):
            raise ValueError(f"unknown timing scope {self.timing!r}")
        if self.report_format not in ("csv", "json"):
            raise ValueError(f"unknown report format {self.report_format!r}")
        if not self.sizes:
            raise ValueError("at least one block size is required")
        for n in self.sizes:
            if n < 1:
                raise ValueError(f"block sizes must be >= 1, got {n}")


def resolve_out_bits(cfg: RunConfig, n: int) -> int:
    """Output length for an n-bit block (ratio default 0.5), bench.py:98-105."""
    if cfg.out_bits is not None:
        if cfg.out_bits > n:
            raise ValueError(f"out_bits={cfg.out_bits} exceeds block size {n}")
        return cfg.out_bits
    ratio = 0.5 if cfg.ratio is None else cfg.ratio
    return max(1, int(ratio * n))


@dataclass(frozen=True)
class PaRunResult:
    blocks: int
    n: int
    r: int
    budget: security.SecurityBudget | None
    out_path: str


# hasher(x, c, d, n, r, order) -> [B, ceil(r/8)] uint8; x, c, d are [B, ceil(n/8)] uint8
Hasher = Callable[[np.ndarray, np.ndarray, np.ndarray, int, int, WordOrder], np.ndarray]


def _default_devices() -> list[int]:
    """Every visible GPU; under torch.distributed a rank owns only its current one."""
    import torch
    import torch.distributed as tdist

    if tdist.is_available() and tdist.is_initialized():
        return [torch.cuda.current_device()]
    n = torch.cuda.device_count()
    if n == 0:
        raise _native.NativeUnavailable("no CUDA device visible (there is no CPU fallback)")
    return list(range(n))


def gpu_hasher(batch: int = 256, devices: list[int] | None = None) -> Hasher:
    """Default hasher: the CUDA path over pinned staging.  `devices` = GPUs of this
    process to shard each batch over (default: every visible GPU, block-sharded
    with no inter-GPU traffic; under torch.distributed every rank owns one GPU)."""

    def run(x, c, d, n, r, order):
        import torch

        from .batch import hash_host_multi

        devs = devices if devices is not None else _default_devices()
        px, pc, pd = (torch.from_numpy(np.array(a, copy=True)).pin_memory() for a in (x, c, d))
        out = hash_host_multi(px, pc, pd, n, r, devices=devs, max_batch=batch,
                              order=_native.ORDER_MSF if order is WordOrder.MOST_SIGNIFICANT_FIRST
                              else _native.ORDER_LSF)
        return out.numpy()

    return run


# seeded(x, n, r, order, rng_seed, first_index) -> [B, ceil(r/8)] uint8: block j of x is
# run_pa block first_index + j; its seed is derived by the implementation itself
SeededHasher = Callable[[np.ndarray, int, int, WordOrder, int, int], np.ndarray]


def gpu_seeded_hasher(batch: int = 256, devices: list[int] | None = None) -> SeededHasher:
    """Default run_pa path: only the key blocks go to the GPU; each block's
    gen_seed(n, derive_block_seed(rng_seed, i)) is expanded there (SHAKE-256,
    pab_seed_expand), beside the hashing of the previous chunk."""

    def run(x, n, r, order, rng_seed, first_index):
        import torch

        from .batch import hash_host_multi

        devs = devices if devices is not None else _default_devices()
        px = torch.from_numpy(np.array(x, copy=True)).pin_memory()
        out = hash_host_multi(px, None, None, n, r, devices=devs, max_batch=batch,
                              rng_seed=rng_seed, first_index=first_index,
                              order=_native.ORDER_MSF if order is WordOrder.MOST_SIGNIFICANT_FIRST
                              else _native.ORDER_LSF)
        return out.numpy()

    return run


def derive_seeds(n: int, rng_seed: int, indices, order: WordOrder,
                 threads: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """(c, d) of the given block indices, serialized in `order` (pa.py:156-172)."""
    nb = (n + 7) // 8
    idx = list(indices)
    cs = np.empty((len(idx), nb), np.uint8)
    ds = np.empty_like(cs)
    endian = "little" if order is WordOrder.LEAST_SIGNIFICANT_FIRST else "big"

    def one(j):
        s = pa.gen_seed(n, pa.derive_block_seed(rng_seed, idx[j]))
        cs[j] = np.frombuffer(s.c.value.to_bytes(nb, endian), np.uint8)
        ds[j] = np.frombuffer(s.d.value.to_bytes(nb, endian), np.uint8)

    with ThreadPoolExecutor(threads or min(16, os.cpu_count() or 1)) as ex:
        list(ex.map(one, range(len(idx))))
    return cs, ds


def shard_range(nblocks: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block range [lo, hi) of `rank` (balanced to within one block)."""
    base, extra = divmod(nblocks, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def run_pa(cfg: RunConfig, *, hasher: Hasher | None = None, dist=None,
           chunk_blocks: int | None = None, seeded: SeededHasher | None = None) -> PaRunResult:
    """Hash every complete n-bit block of cfg.in_path into r bits (bench.py:223-265).

    `dist` is torch.distributed (initialised) for multi-GPU runs; each rank
    hashes its contiguous share and rank 0 writes the file.  By default the
    GPU derives the seeds and hashes (`gpu_seeded_hasher`); an injected
    `hasher` gets host-derived (c, d) instead (tests use the oracle), an
    injected `seeded` replaces the default seeded path.
    """
    if len(cfg.sizes) != 1:
        raise ValueError("batch hashing needs exactly one block size")
    n = cfg.sizes[0]
    if n % 8 != 0:
        raise ValueError(f"block size must be a whole number of bytes, got {n} bits")
    if cfg.in_path is None or cfg.out_path is None:
        raise ValueError("batch hashing needs both an input and an output path")
    data = Path(cfg.in_path).read_bytes()
    block_bytes = n // 8
    nblocks = len(data) // block_bytes
    if nblocks == 0:
        raise ValueError(
            f"input holds {len(data) * 8} bits, shorter than one {n}-bit block")
    rank = dist.get_rank() if dist else 0
    world = dist.get_world_size() if dist else 1
    if len(data) % block_bytes and rank == 0:
        print(f"ignoring {len(data) % block_bytes} trailing bytes "
              f"(not a whole block)", file=sys.stderr)

    r = resolve_out_bits(cfg, n)
    enforce = cfg.epsilon is not None and cfg.h_min is not None
    params = pa.PAParams(n=n, r=r, epsilon=cfg.epsilon, h_min=cfg.h_min)
    budget = None
    if enforce:  # pa_round's check, once for the whole file (same r for every block)
        check = security.validate(params)
        if not check.ok:
            raise pa.SecurityBoundError(params.r, check.r_max)
        budget = security.SecurityBudget.evaluate(cfg.h_min, cfg.epsilon, r)

    if hasher is None and seeded is None:
        if len(_native.seed_material(cfg.rng_seed)) <= _native.MAX_SEED_MATERIAL:
            seeded = gpu_seeded_hasher()
        else:  # the device expander absorbs <= 1 KiB of master material: expand on the host
            hasher = gpu_hasher()
    lo, hi = shard_range(nblocks, rank, world)
    arr = np.frombuffer(data, np.uint8, count=nblocks * block_bytes).reshape(nblocks, block_bytes)
    rb = (r + 7) // 8
    parts = []
    # one call per shard by default: the GPU seed path keeps many blocks' XOF
    # chains in flight at once and overlaps them with the hashing
    step = chunk_blocks or max(1, hi - lo)
    for b0 in range(lo, hi, step):
        b1 = min(hi, b0 + step)
        x = arr[b0:b1]
        # import_block's check: no bits beyond n (n % 8 == 0 here, so none exist)
        if seeded is not None:
            y = seeded(x, n, r, cfg.order, cfg.rng_seed, b0)
        else:
            c, d = derive_seeds(n, cfg.rng_seed, range(b0, b1), cfg.order)
            y = hasher(x, c, d, n, r, cfg.order)
        parts.append(np.asarray(y, np.uint8).reshape(b1 - b0, rb))
    mine = np.concatenate(parts) if parts else np.empty((0, rb), np.uint8)

    if dist and world > 1:
        gathered = [None] * world if rank == 0 else None
        dist.gather_object(mine.tobytes(), gathered, dst=0)
        if rank == 0:
            out = b"".join(gathered)
        dist.barrier()
    else:
        out = mine.tobytes()
    if rank == 0:
        Path(cfg.out_path).write_bytes(out)
    return PaRunResult(blocks=nblocks, n=n, r=r, budget=budget, out_path=cfg.out_path)
