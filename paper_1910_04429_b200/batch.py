"""Batched PA hashing on one GPU: device-resident and host-streamed paths.

This is the "batched scheduler" of the north star (host
scheduler row): many independent blocks per launch (grid dimension = block),
per-stream workspaces, pinned host staging, and H2D / compute / D2H of
successive chunks overlapped on separate CUDA streams.  It generalises the
reference's sequential batch loop (pkg/src/modpa/bench.py:256-262).

PyTorch is used only as plumbing (device memory, pinned host memory, streams
and events); every byte of hashing runs in the C-ABI library.
"""
from __future__ import annotations

import ctypes

import torch

from . import _native


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


# hash_seeded_host: smallest seed window (blocks) expanded on the hashing stream
# (2 XOF streams per block: >= 8192 lane pairs per launch, throughput-bound)
kExclusiveMin = 4096
kTaperMin = 32  # the last chunk of an exclusive call is hashed in quarters of >= this many blocks


def exclusive_windows(nchunks: int, target: int, cap: int) -> list[int]:
    """Seed windows (in hashing chunks) of a call of `nchunks` chunks on the exclusive
    schedule: as even as possible, none above `target` chunks (a longer expansion
    starves the copies) -- except a call of up to 1.5 targets, which is one window
    (two short windows would each be one chain long) -- and none above `cap`."""
    if nchunks <= min(cap, target + target // 2):
        return [nchunks]
    k = -(-nchunks // min(target, cap))
    return [nchunks // k + (1 if i < nchunks % k else 0) for i in range(k)]


class HashEngine:
    """Hash batches of n-bit blocks down to r bits on one CUDA device.

    Inputs are uint8 tensors of shape [batch, ceil(n/8)] (x, c, d) in the
    reference's serialized layout; outputs [batch, ceil(r/8)].
    """

    def __init__(self, n: int, r: int, *, device: int | torch.device | None = None,
                 order: int = _native.ORDER_LSF, max_batch: int = 64,
                 max_workspace: int = 4 << 30):
        if not 1 <= r <= n:
            raise ValueError(f"output length r={r} must satisfy 1 <= r <= n={n}")
        self.lib = _native.load()
        if not torch.cuda.is_available():
            raise _native.NativeUnavailable("no CUDA device (there is no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self.n, self.r, self.order = n, r, order
        self.nbytes, self.rbytes = (n + 7) // 8, (r + 7) // 8
        chunk = max(1, max_batch)
        while chunk > 1 and self.lib.pab_hash_workspace_bytes(n, chunk) > max_workspace:
            chunk //= 2
        self.chunk = chunk
        self.ws_bytes = int(self.lib.pab_hash_workspace_bytes(n, chunk))
        if self.ws_bytes == 0:
            _native.check(_native.PAB_EINVAL)
        self._ws = {}

    def _workspace(self, stream: torch.cuda.Stream) -> torch.Tensor:
        key = stream.cuda_stream
        ws = self._ws.get(key)
        if ws is None:
            ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
            self._ws[key] = ws
        return ws

    def hash_device(self, x: torch.Tensor, c: torch.Tensor, d: torch.Tensor,
                    out: torch.Tensor | None = None,
                    stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """Hash device-resident blocks (enqueued on `stream`, asynchronous)."""
        b = x.shape[0]
        for t in (x, c, d):
            if t.device != self.device or t.dtype != torch.uint8 or t.dim() != 2:
                raise ValueError("x, c, d must be 2-D uint8 tensors on the engine's device")
            if t.shape[0] != b or t.shape[1] < self.nbytes or t.stride(1) != 1:
                raise ValueError("x, c, d must be [batch, >= ceil(n/8)] with unit byte stride")
        if not (x.stride(0) == c.stride(0) == d.stride(0)):
            raise ValueError("x, c, d must share one row stride")
        st = stream or torch.cuda.current_stream(self.device)
        if out is None:
            out = torch.empty((b, self.rbytes), dtype=torch.uint8, device=self.device)
        ws = self._workspace(st)
        with torch.cuda.device(self.device):  # the C ABI works on the current device
            _native.check(self.lib.pab_hash_batch(
                _ptr(x), _ptr(c), _ptr(d), x.stride(0), self.n, self.r, b, self.order,
                _ptr(out), out.stride(0), _ptr(ws), self.ws_bytes, ctypes.c_void_p(st.cuda_stream)))
        return out

    def hash_host(self, x: torch.Tensor, c: torch.Tensor, d: torch.Tensor,
                  out: torch.Tensor | None = None, streams: int = 3,
                  chunk: int | None = None, join_in: bool = True,
                  join_out: bool = True) -> torch.Tensor:
        """End-to-end from (pinned) host tensors: H2D, hash, D2H, overlapped.

        A triple-buffered pipeline: one stream each for H2D, hashing and D2H,
        `streams` device buffer slots, and per-slot events so the copy engines
        only wait for a slot to be free (the H2D of chunk i+slots waits for the
        hashing of chunk i to have read its inputs).  The slot events persist
        across calls.  Returns host [batch, ceil(r/8)] (complete once the
        caller's current stream is synced).

        Streaming use: join_in=False skips ordering the copies after the
        caller's stream (the inputs are ready host memory), join_out=False skips
        making the caller's stream wait for the keys; consecutive calls then
        overlap (one call's head with the previous call's tail) and the caller
        calls join() once before reading the keys.
        """
        b = x.shape[0]
        if out is None:
            out = torch.empty((b, self.rbytes), dtype=torch.uint8, pin_memory=True)
        chunk = chunk or self.chunk
        nslots = max(1, streams)
        s_in, s_comp, s_out = self._pipe_streams()
        bufs = self._io_buffers(nslots, chunk)
        ev = self._slot_events(nslots)
        cur = torch.cuda.current_stream(self.device)
        if join_in:
            for s in (s_in, s_comp, s_out):
                s.wait_stream(cur)
        for i, b0 in enumerate(range(0, b, chunk)):
            k = (self._slot_next + i) % nslots  # slots rotate across calls too
            dx, dc, dd, dout = bufs[k]
            nb = min(chunk, b - b0)
            s_in.wait_event(ev["comp"][k])       # slot k's inputs consumed
            with torch.cuda.stream(s_in):
                dx[:nb].copy_(x[b0:b0 + nb], non_blocking=True)
                dc[:nb].copy_(c[b0:b0 + nb], non_blocking=True)
                dd[:nb].copy_(d[b0:b0 + nb], non_blocking=True)
                ev["in"][k].record(s_in)
            s_comp.wait_event(ev["in"][k])
            s_comp.wait_event(ev["out"][k])      # slot k's output drained
            self.hash_device(dx[:nb], dc[:nb], dd[:nb], dout[:nb], stream=s_comp)
            ev["comp"][k].record(s_comp)
            s_out.wait_event(ev["comp"][k])
            with torch.cuda.stream(s_out):
                out[b0:b0 + nb].copy_(dout[:nb], non_blocking=True)
                ev["out"][k].record(s_out)
        self._slot_next = (self._slot_next + -(-b // chunk)) % nslots
        if join_out:
            self.join(cur)
        return out

    def join(self, stream: torch.cuda.Stream | None = None) -> None:
        """Make `stream` (default: the current one) wait for every pipelined call."""
        cur = stream or torch.cuda.current_stream(self.device)
        for s in self._pipe_streams():
            cur.wait_stream(s)

    def seed_device(self, rng_seed, first_index: int, batch: int, c: torch.Tensor,
                    d: torch.Tensor, stream: torch.cuda.Stream | None = None,
                    protocol: str = "run_pa") -> None:
        """(c, d) of blocks first_index .. first_index+batch-1, SHAKE-256 on the device
        into rows of c and d (asynchronous on `stream`), derived as
          protocol "run_pa": gen_seed(n, derive_block_seed(rng_seed, i))
                             (pkg/src/modpa/bench.py:258, pa.py:138-172);
          protocol "bench":  gen_seed(n, derive_block_seed(i, n)) -- the reference's
                             benchmark inputs (bench.py:156), i = the block seed,
                             rng_seed unused (BASELINE configs' per-block seeds)."""
        if protocol not in ("run_pa", "bench"):
            raise ValueError(f"unknown seed protocol {protocol!r}")
        for t in (c, d):
            if t.device != self.device or t.dtype != torch.uint8 or t.dim() != 2:
                raise ValueError("c, d must be 2-D uint8 tensors on the engine's device")
            if t.shape[0] < batch or t.shape[1] < self.nbytes or t.stride(1) != 1:
                raise ValueError("c, d must be [>= batch, >= ceil(n/8)] with unit byte stride")
        if c.stride(0) != d.stride(0):
            raise ValueError("c and d must share one row stride")
        st = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            if protocol == "bench":
                _native.check(self.lib.pab_seed_expand_bench(
                    first_index, batch, self.n, self.n, self.order, _ptr(c), _ptr(d), c.stride(0),
                    ctypes.c_void_p(st.cuda_stream)))
                return
            m = _native.seed_material(rng_seed)
            _native.check(self.lib.pab_seed_expand(
                m, len(m), first_index, batch, self.n, self.order, _ptr(c), _ptr(d), c.stride(0),
                ctypes.c_void_p(st.cuda_stream)))

    def hash_seeded_host(self, x: torch.Tensor, rng_seed, first_index: int = 0,
                         out: torch.Tensor | None = None, streams: int = 3,
                         chunk: int | None = None, join_in: bool = True,
                         join_out: bool = True, seed_budget: int = 4 << 30,
                         protocol: str = "run_pa", exclusive: bool | None = None,
                         native: bool | None = None) -> torch.Tensor:
        """run_pa's step end to end: key blocks x from (pinned) host memory, block
        first_index + j hashed with gen_seed(n, derive_block_seed(rng_seed, first_index + j))
        derived on the GPU (only x crosses PCIe); protocol "bench" derives the
        reference benchmark's seeds instead (see seed_device).

        The seed expansion is latency-bound per XOF stream: a stream's squeeze is
        a chain of ceil(n/8)/136 dependent Keccak-f calls, whatever the number of
        streams.  So seeds are expanded in windows of blocks, each window by one
        launch on its own stream into its own buffer, and several windows are in
        flight at once (up to `seed_budget` bytes of (c, d) rows): the chains of
        all of them run concurrently, and hashing window w (chunk by chunk,
        H2D / hash / D2H pipelined over `streams` slots as in hash_host) overlaps
        the expansion of the windows after it.  Hand a whole key file (shard) to
        one call: the expansion latency is then paid once per `seed_budget` of
        blocks, not once per chunk.  join_in / join_out as in hash_host.

        Big calls at small n take another schedule (`exclusive`, default: chosen by
        size).  Expansion and hashing share an SM badly: the Keccak warps keep the
        ALU pipe the butterflies also need busy, and a 1024-block step of both at
        n = 1e6 measures 2.6-2.8 ms against 0.57 + 1.66 ms one after the other
        (scripts/seed_hash_corun.py).  When `seed_budget` holds one window of at
        least kExclusiveMin blocks (enough XOF streams for the expansion to be
        throughput-bound instead of one chain long), the windows are expanded on
        the hashing stream itself, each right before its chunks are hashed, so the
        two never run together; the copies still overlap both.

        A call on that schedule that is synchronous anyway (join_in and join_out, default
        chunking, packed host rows) is one C call, `pab_hash_seeded_host` /
        `pab_hash_seeded_host_bench` (`native`, default: when eligible): the same pipeline
        driven from C (n = 1e6: 2.58 ms per 1024 blocks against 2.63 from here); it
        returns with the keys complete.
        """
        b = x.shape[0]
        if out is None:
            out = torch.empty((b, self.rbytes), dtype=torch.uint8, pin_memory=True)
        per_block = 2 * self.nbytes
        if protocol not in ("run_pa", "bench"):
            raise ValueError(f"unknown seed protocol {protocol!r}")
        if native is None or native:
            packed = (x.device.type == "cpu" and out.device.type == "cpu" and x.dtype == torch.uint8
                      and out.dtype == torch.uint8 and x.dim() == 2 and out.dim() == 2
                      and x.shape[1] == self.nbytes and out.shape == (b, self.rbytes)
                      and x.is_contiguous() and out.is_contiguous())
            sized = b >= kExclusiveMin and seed_budget // per_block >= kExclusiveMin
            eligible = (packed and join_in and join_out and chunk is None and exclusive is not False
                        and (sized or exclusive)
                        and (protocol == "bench" or _native.seed_material_fits(rng_seed)))
            if native and not eligible:
                raise ValueError("native=True needs a synchronous call (join_in, join_out), default "
                                 "chunking, packed uint8 host tensors and the exclusive schedule")
            if eligible:
                return self._hash_seeded_native(x, rng_seed, first_index, out, protocol)
        chunk = chunk or self.chunk
        nslots = max(1, streams)
        s_in, s_comp, s_out = self._pipe_streams()
        bufs = self._io_buffers(nslots, chunk)
        ev = self._slot_events(nslots)
        # exclusive windows: long enough to be throughput-bound, short enough for the
        # (nslots - 1) prefetched chunks to keep PCIe busy while one expands (measured at
        # n = 1e6: 4096-block windows with 3 slots, 2.62 ms per 1024 blocks; 8192: 2.76)
        xmax = seed_budget // per_block // chunk * chunk
        xwin = min(xmax, max(kExclusiveMin, 2 * (nslots - 1) * chunk))
        if exclusive is None:
            exclusive = xwin >= kExclusiveMin and b >= kExclusiveMin
        if exclusive and xwin >= chunk:
            wins = exclusive_windows(-(-b // chunk), xwin // chunk, xmax // chunk)
            return self._hash_seeded_exclusive(x, rng_seed, first_index, out, nslots, chunk,
                                               [w * chunk for w in wins], join_in, join_out,
                                               protocol)
        # windows of `win` blocks (whole hashing chunks) over `nbuf` rotating buffers:
        # up to nbuf windows -- of this call and of the calls queued after it --
        # expand concurrently
        win = max(chunk, min(-(-b // chunk) * chunk,
                             (max(chunk, seed_budget // per_block // 4) // chunk) * chunk))
        nbuf = max(2, min(32, seed_budget // (per_block * win)))
        wins = self._seed_windows(nbuf, win)
        cur = torch.cuda.current_stream(self.device)
        if join_in:
            for s in (s_in, s_comp, s_out):
                s.wait_stream(cur)
        starts = list(range(0, b, win))
        base = self._sw_next

        def expand(w):  # window w into its rotating buffer, on that buffer's stream
            sc, sd, ev_free, ev_ready, st = wins[(base + w) % nbuf]
            st.wait_event(ev_free)  # the buffer's previous window is hashed
            self.seed_device(rng_seed, first_index + starts[w], min(win, b - starts[w]), sc, sd,
                             stream=st, protocol=protocol)
            ev_ready.record(st)

        for w in range(min(nbuf, len(starts))):
            expand(w)
        i = self._slot_next  # slots rotate across calls too
        for w, w0 in enumerate(starts):
            sc, sd, ev_free, ev_ready, _ = wins[(base + w) % nbuf]
            s_comp.wait_event(ev_ready)
            for b0 in range(w0, min(b, w0 + win), chunk):
                k = i % nslots
                i += 1
                dx, _, _, dout = bufs[k]
                nb = min(chunk, b - b0)
                s_in.wait_event(ev["comp"][k])       # slot k's inputs consumed
                with torch.cuda.stream(s_in):
                    dx[:nb].copy_(x[b0:b0 + nb], non_blocking=True)
                    ev["in"][k].record(s_in)
                s_comp.wait_event(ev["in"][k])
                s_comp.wait_event(ev["out"][k])      # slot k's output drained
                self.hash_device(dx[:nb], sc[b0 - w0:b0 - w0 + nb], sd[b0 - w0:b0 - w0 + nb],
                                 dout[:nb], stream=s_comp)
                ev["comp"][k].record(s_comp)
                s_out.wait_event(ev["comp"][k])
                with torch.cuda.stream(s_out):
                    out[b0:b0 + nb].copy_(dout[:nb], non_blocking=True)
                    ev["out"][k].record(s_out)
            ev_free.record(s_comp)
            if w + nbuf < len(starts):
                expand(w + nbuf)
        self._sw_next = (base + len(starts)) % nbuf
        self._slot_next = i % nslots
        if join_out:  # s_comp has waited for every seed window it used
            self.join(cur)
        return out

    def _hash_seeded_native(self, x, rng_seed, first_index, out, protocol):
        """One synchronous C call for the whole key file (pab_hash_seeded_host[_bench])."""
        torch.cuda.current_stream(self.device).synchronize()  # join_in: inputs are ready
        b = x.shape[0]
        px, po = ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr())
        if protocol == "bench":
            _native.check(self.lib.pab_hash_seeded_host_bench(
                px, self.n, self.r, b, self.order, first_index, self.n, po, self.device.index))
        else:
            m = _native.seed_material(rng_seed)
            _native.check(self.lib.pab_hash_seeded_host(
                px, self.n, self.r, b, self.order, m, len(m), first_index, po, self.device.index))
        return out

    def _hash_seeded_exclusive(self, x, rng_seed, first_index, out, nslots, chunk, wins,
                               join_in, join_out, protocol):
        """hash_seeded_host with each window (`wins`: blocks per window) expanded on the
        hashing stream right before its chunks (one (c, d) buffer, reused in stream order)."""
        b = x.shape[0]
        win = max(wins)
        s_in, s_comp, s_out = self._pipe_streams()
        bufs = self._io_buffers(nslots, chunk)
        ev = self._slot_events(nslots)
        if getattr(self, "_xw_win", 0) < win:
            if getattr(self, "_xw_win", 0):
                torch.cuda.synchronize(self.device)  # the old buffer may still be read
            self._xw = tuple(torch.empty((win, self.nbytes), dtype=torch.uint8, device=self.device)
                             for _ in range(2))
            self._xw_win = win
        sc, sd = self._xw
        cur = torch.cuda.current_stream(self.device)
        if join_in:
            for s in (s_in, s_comp, s_out):
                s.wait_stream(cur)
        i = self._slot_next
        w0 = 0
        for wlen in wins:
            w1 = min(b, w0 + wlen)
            self.seed_device(rng_seed, first_index + w0, w1 - w0, sc, sd, stream=s_comp,
                             protocol=protocol)
            pieces = [(b0, min(chunk, w1 - b0)) for b0 in range(w0, w1, chunk)]
            if join_out and w1 >= b and pieces[-1][1] >= 4 * kTaperMin:
                # the call's last chunk in quarters: after the last H2D only a quarter's
                # hashing and D2H remain (measured at C2: 2.85 -> 0.8 ms of drain per call)
                b0, nb = pieces.pop()
                q = -(-nb // 4)
                pieces += [(b0 + j, min(q, nb - j)) for j in range(0, nb, q)]
            for b0, nb in pieces:
                k = i % nslots
                i += 1
                dx, _, _, dout = bufs[k]
                s_in.wait_event(ev["comp"][k])       # slot k's inputs consumed
                with torch.cuda.stream(s_in):
                    dx[:nb].copy_(x[b0:b0 + nb], non_blocking=True)
                    ev["in"][k].record(s_in)
                s_comp.wait_event(ev["in"][k])
                s_comp.wait_event(ev["out"][k])      # slot k's output drained
                self.hash_device(dx[:nb], sc[b0 - w0:b0 - w0 + nb], sd[b0 - w0:b0 - w0 + nb],
                                 dout[:nb], stream=s_comp)
                ev["comp"][k].record(s_comp)
                s_out.wait_event(ev["comp"][k])
                with torch.cuda.stream(s_out):
                    out[b0:b0 + nb].copy_(dout[:nb], non_blocking=True)
                    ev["out"][k].record(s_out)
            w0 = w1
        self._slot_next = i % nslots
        if join_out:
            self.join(cur)
        return out

    def _seed_windows(self, nbuf: int, win: int):
        """nbuf rotating (c, d) window buffers [win, ceil(n/8)], each with its stream
        and free / ready events (kept across calls, so queued calls overlap)."""
        key = (nbuf, win)
        if getattr(self, "_sw_key", None) != key:
            if getattr(self, "_sw_key", None) is not None:
                torch.cuda.synchronize(self.device)  # old windows may still be in use
            mk = lambda: torch.empty((win, self.nbytes), dtype=torch.uint8, device=self.device)  # noqa: E731
            self._sw = [(mk(), mk(), torch.cuda.Event(), torch.cuda.Event(),
                         torch.cuda.Stream(self.device)) for _ in range(nbuf)]
            self._sw_key = key
            self._sw_next = 0
        return self._sw

    def _pipe_streams(self):
        if not hasattr(self, "_pipe"):
            self._pipe = tuple(torch.cuda.Stream(self.device) for _ in range(3))
        return self._pipe

    def _slot_events(self, k: int):
        if getattr(self, "_ev_k", None) != k:
            self._slot_next = 0
            if getattr(self, "_ev_k", None) is not None:
                self.join()  # earlier calls' copies / hashing may still wait on the old events
            mk = lambda: [torch.cuda.Event() for _ in range(k)]  # noqa: E731
            self._ev = {"in": mk(), "comp": mk(), "out": mk(), "seed": mk()}
            self._ev_k = k
        return self._ev

    def _io_buffers(self, k: int, chunk: int):
        key = (k, chunk)
        if getattr(self, "_io_key", None) != key:
            if getattr(self, "_io_key", None) is not None:
                # a join_out=False call may still be copying into / hashing from the
                # old slots: the allocator must not hand their memory out before that
                torch.cuda.synchronize(self.device)
            mk = lambda w: torch.empty((chunk, w), dtype=torch.uint8, device=self.device)  # noqa: E731
            self._io = [(mk(self.nbytes), mk(self.nbytes), mk(self.nbytes), mk(self.rbytes))
                        for _ in range(k)]
            self._io_key = key
        return self._io


def hash_host_multi(x: torch.Tensor, c: torch.Tensor | None, d: torch.Tensor | None, n: int,
                    r: int, *, devices: list[int] | None = None, order: int = _native.ORDER_LSF,
                    max_batch: int = 256, rng_seed=None, first_index: int = 0) -> torch.Tensor:
    """Hash a pinned host batch on several GPUs of this process: one worker thread per
    device, contiguous block shards, keys returned in block order.

    Blocks are independent, so there is no inter-GPU traffic;
    each worker runs HashEngine.hash_host on its shard (copies overlapped with
    compute on that device's streams).  The C ABI releases the GIL, so the
    workers run concurrently.  With c = d = None the seeds are derived on the
    GPUs from `rng_seed` (block i of x is run_pa block first_index + i).
    """
    if (c is None) != (d is None) or (c is None and rng_seed is None):
        raise ValueError("give both c and d, or neither and an rng_seed")
    import threading

    devs = list(range(torch.cuda.device_count())) if devices is None else list(devices)
    if not devs:
        raise _native.NativeUnavailable("no CUDA device (there is no CPU fallback)")
    b = x.shape[0]
    out = torch.empty((b, (r + 7) // 8), dtype=torch.uint8, pin_memory=True)
    spans = []
    base, extra = divmod(b, len(devs))
    lo = 0
    for i, dev in enumerate(devs):
        hi = lo + base + (1 if i < extra else 0)
        spans.append((dev, lo, hi))
        lo = hi
    errors = []

    def work(dev, lo, hi):
        try:
            if hi <= lo:
                return
            torch.cuda.set_device(dev)
            eng = HashEngine(n, r, device=dev, order=order, max_batch=min(max_batch, hi - lo))
            if c is None:
                eng.hash_seeded_host(x[lo:hi], rng_seed, first_index + lo, out[lo:hi], streams=3)
            else:
                eng.hash_host(x[lo:hi], c[lo:hi], d[lo:hi], out[lo:hi], streams=3)
            torch.cuda.synchronize(dev)
        except BaseException as e:  # surfaced in the caller
            errors.append(e)

    threads = [threading.Thread(target=work, args=s) for s in spans]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return out
