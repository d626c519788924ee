"""On-GPU seed expansion (pab_seed_expand) vs the reference's own derivation.

The reference derives block i's hash-family member as
gen_seed(n, derive_block_seed(master, i)) with SHAKE-256 from hashlib
(pkg/src/modpa/pa.py:138-172, called by run_pa at pkg/src/modpa/bench.py:258).
paper_1910_04429_b200.pa restates those functions on the host with hashlib
(the reference's own dependency), which is the checker here.  Cases cover
the sponge's edges: output lengths around the 136-byte rate, n not a multiple
of 8, one- and multi-block absorbs (seed material around the rate), decimal
label widths, MSF layout and unaligned rows.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_1910_04429_b200 import _native, pa
from paper_1910_04429_b200.batch import HashEngine

pytestmark = pytest.mark.gpu


def host_seeds(n, master, first, batch, msf=False):
    nb = (n + 7) // 8
    endian = "big" if msf else "little"
    cs, ds = [], []
    for i in range(first, first + batch):
        s = pa.gen_seed(n, pa.derive_block_seed(master, i))
        cs.append(s.c.value.to_bytes(nb, endian))
        ds.append(s.d.value.to_bytes(nb, endian))
    return cs, ds


def device_seeds(n, master, first, batch, msf=False, stride=None, offset=0):
    nb = (n + 7) // 8
    stride = stride or nb
    eng = HashEngine(n, 1, order=_native.ORDER_MSF if msf else _native.ORDER_LSF,
                     max_batch=max(1, batch))
    raw_c = torch.full((batch * stride + offset + 8,), 0xA5, dtype=torch.uint8, device="cuda")
    raw_d = torch.full_like(raw_c, 0x5A)
    c = raw_c[offset:offset + batch * stride].view(batch, stride)
    d = raw_d[offset:offset + batch * stride].view(batch, stride)
    eng.seed_device(master, first, batch, c, d)
    torch.cuda.synchronize()
    c, d = c.cpu().numpy(), d.cpu().numpy()
    # bytes beyond each row's ceil(n/8) stay untouched
    if stride > nb:
        assert (c[:, nb:] == 0xA5).all() and (d[:, nb:] == 0x5A).all()
    return [c[j, :nb].tobytes() for j in range(batch)], [d[j, :nb].tobytes() for j in range(batch)]


@pytest.mark.parametrize("n", [1, 7, 8, 9, 63, 64, 65, 1080, 1088, 1089, 1096, 2176, 2177,
                               100_001, 1_000_000])
def test_seed_sizes_match_hashlib(n):
    want = host_seeds(n, 5, 0, 3)
    assert device_seeds(n, 5, 0, 3) == want


@pytest.mark.parametrize("master", [0, 1, 255, 256, 2**64 + 3, 2**1000 - 1, b"", b"\x00" * 31,
                                    bytes(range(122)), bytes(range(123)), bytes(range(124)),
                                    bytes(range(200)), bytes(255 - i for i in range(256)),
                                    b"k" * 1024])
def test_seed_material_forms(master):
    # int and bytes material; total message lengths across the 136-byte rate
    n = 4097
    assert device_seeds(n, master, 7, 4) == host_seeds(n, master, 7, 4)


@pytest.mark.parametrize("first", [0, 8, 9, 10, 99, 100, 99_998, 10**12, 2**63 - 3])
def test_seed_block_index_labels(first):
    n = 3000
    assert device_seeds(n, 3, first, 3) == host_seeds(n, 3, first, 3)


def test_seed_msf_and_unaligned_rows():
    for n in (1089, 10_000, 65_537):
        assert device_seeds(n, 11, 2, 3, msf=True) == host_seeds(n, 11, 2, 3, msf=True)
        nb = (n + 7) // 8
        assert device_seeds(n, 11, 2, 3, stride=nb + 5, offset=3) == host_seeds(n, 11, 2, 3)
        assert device_seeds(n, 11, 2, 3, stride=nb + 16) == host_seeds(n, 11, 2, 3)


def test_seed_c_odd_and_masked():
    n = 1_000_003
    cs, ds = device_seeds(n, 42, 0, 8)
    for c, d in zip(cs, ds):
        assert c[0] & 1
        assert c[-1] >> (n % 8) == 0 and d[-1] >> (n % 8) == 0


def test_seed_errors():
    eng = HashEngine(1000, 10, max_batch=1)
    c = torch.empty((1, 125), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError, match="longer than 1024"):
        eng.seed_device(b"x" * 1025, 0, 1, c, c.clone())
    with pytest.raises(ValueError, match="nonnegative"):
        eng.seed_device(-1, 0, 1, c, c.clone())


@pytest.mark.parametrize("n,r", [(64, 31), (4096, 2048), (100_000, 50_000), (1_000_000, 500_000)])
def test_hash_seeded_host_matches_oracle(n, r):
    B = 5
    rng = np.random.default_rng(n)
    nb = (n + 7) // 8
    x = rng.integers(0, 256, size=(B, nb), dtype=np.uint8)
    if n % 8:
        x[:, -1] &= (1 << (n % 8)) - 1
    cs, ds = host_seeds(n, 9, 40, B)
    want = [oracle.compress(x[j].tobytes(), cs[j], ds[j], n, r) for j in range(B)]
    got = _native.hash_seeded_host(x.tobytes(), n, r, B, 9, first_index=40)
    rb = (r + 7) // 8
    assert [got[j * rb:(j + 1) * rb] for j in range(B)] == want
    # the overlapped engine pipeline, several chunks and slots
    eng = HashEngine(n, r, max_batch=2)
    out = eng.hash_seeded_host(torch.from_numpy(x).pin_memory(), 9, first_index=40)
    torch.cuda.synchronize()
    assert [out[j].numpy().tobytes() for j in range(B)] == want


@pytest.mark.parametrize("n,r,B,msf", [(4_160, 2_001, 7_173, False), (4_099, 4_099, 2_500, True),
                                        (200_000, 64_000, 37, False)])
def test_native_seeded_host_pipeline(n, r, B, msf):
    # pab_hash_seeded_host: one C call = H2D / seed windows on the hashing stream / hash /
    # D2H over three streams and three slots (several chunks, two seed windows, padded rows
    # for byte-unaligned and MSF blocks); keys equal the engine's and the oracle's
    order = _native.ORDER_MSF if msf else _native.ORDER_LSF
    rng = np.random.default_rng(B)
    nb, rb = (n + 7) // 8, (r + 7) // 8
    x = rng.integers(0, 256, size=(B, nb), dtype=np.uint8)
    if n % 8:
        x[:, 0 if msf else -1] &= (1 << (n % 8)) - 1
    got = _native.hash_seeded_host(x.tobytes(), n, r, B, 21, first_index=5, order=order)
    assert len(got) == B * rb
    eng = HashEngine(n, r, order=order, max_batch=512)
    want = eng.hash_seeded_host(torch.from_numpy(x).pin_memory(), 21, first_index=5, exclusive=False)
    torch.cuda.synchronize()
    assert got == want.numpy().tobytes()
    cs, ds = host_seeds(n, 21, 5, B, msf=msf)
    for j in (0, 1023, 1024, B - 1):
        if j < B:
            assert got[j * rb:(j + 1) * rb] == oracle.compress(x[j].tobytes(), cs[j], ds[j], n, r,
                                                               msf=msf), j
    # a second call reuses the pipeline's slots and events
    assert _native.hash_seeded_host(x[:3].tobytes(), n, r, 3, 21, first_index=5, order=order) == got[:3 * rb]


@pytest.mark.parametrize("n,r,B,msf", [(4_160, 2_001, 2_500, False), (4_099, 17, 1_100, True)])
def test_native_host_pipeline_with_host_members(n, r, B, msf):
    # pab_hash_host: the same three-stream pipeline with c and d from the host, several
    # chunks of 1024 blocks, packed and padded rows
    order = _native.ORDER_MSF if msf else _native.ORDER_LSF
    rng = np.random.default_rng(n + B)
    nb, rb = (n + 7) // 8, (r + 7) // 8
    x, c, d = (rng.integers(0, 256, size=(B, nb), dtype=np.uint8) for _ in range(3))
    if n % 8:
        for a in (x, c, d):
            a[:, 0 if msf else -1] &= (1 << (n % 8)) - 1
    c[:, -1 if msf else 0] |= 1
    got = _native.hash_host(x.tobytes(), c.tobytes(), d.tobytes(), n, r, B, order=order)
    want = oracle.compress_batch(x.tobytes(), c.tobytes(), d.tobytes(), n, r, B, threads=4, msf=msf)
    assert got == want
    assert _native.hash_host(x[:2].tobytes(), c[:2].tobytes(), d[:2].tobytes(), n, r, 2,
                             order=order) == got[:2 * rb]


@pytest.mark.parametrize("protocol", ["run_pa", "bench"])
def test_engine_hands_synchronous_big_calls_to_the_native_pipeline(protocol):
    # hash_seeded_host: a synchronous call of >= kExclusiveMin packed host blocks is one C call
    # (native=None picks it); native=False keeps the Python-driven schedule; same keys
    from paper_1910_04429_b200 import batch

    n, r = 4_160, 1_999
    B = batch.kExclusiveMin + 11
    nb = n // 8
    x = torch.from_numpy(np.random.default_rng(5).integers(0, 256, size=(B, nb), dtype=np.uint8))
    eng = HashEngine(n, r, max_batch=256)
    seed = None if protocol == "bench" else 12
    calls = []
    real = eng._hash_seeded_native
    eng._hash_seeded_native = lambda *a: calls.append(1) or real(*a)
    a = eng.hash_seeded_host(x.pin_memory(), seed, 7, protocol=protocol)
    assert calls == [1]
    b = eng.hash_seeded_host(x, seed, 7, protocol=protocol, native=False)  # pageable, Python path
    c = eng.hash_seeded_host(x.pin_memory(), seed, 7, protocol=protocol, exclusive=False)
    torch.cuda.synchronize()
    assert calls == [1] and torch.equal(a, b) and torch.equal(a, c)
    with pytest.raises(ValueError, match="native=True"):
        eng.hash_seeded_host(x, seed, 7, protocol=protocol, native=True, join_out=False)
    if protocol == "run_pa":
        cs, ds = host_seeds(n, 12, 7, B)
        for j in (0, B - 1):
            assert a[j].numpy().tobytes() == oracle.compress(x[j].numpy().tobytes(), cs[j], ds[j], n, r)


def test_streamed_calls_without_joins():
    # hash_host / hash_seeded_host chained with join_in / join_out off, one join() at the end
    n, r, B = 100_000, 30_001, 6
    rng = np.random.default_rng(3)
    nb = (n + 7) // 8
    xs = [rng.integers(0, 256, size=(B, nb), dtype=np.uint8) for _ in range(3)]
    cs, ds = host_seeds(n, 4, 0, B)
    c = np.frombuffer(b"".join(cs), np.uint8).reshape(B, nb)
    d = np.frombuffer(b"".join(ds), np.uint8).reshape(B, nb)
    eng = HashEngine(n, r, max_batch=2)
    pc, pd = torch.from_numpy(c.copy()).pin_memory(), torch.from_numpy(d.copy()).pin_memory()
    outs, souts = [], []
    for i, x in enumerate(xs):
        px = torch.from_numpy(x).pin_memory()
        outs.append(eng.hash_host(px, pc, pd, join_in=i == 0, join_out=False))
        souts.append(eng.hash_seeded_host(px, 4, 0, join_in=False, join_out=False))
    eng.join()
    torch.cuda.synchronize()
    for x, o, so in zip(xs, outs, souts):
        want = [oracle.compress(x[j].tobytes(), cs[j], ds[j], n, r) for j in range(B)]
        assert [o[j].numpy().tobytes() for j in range(B)] == want
        assert [so[j].numpy().tobytes() for j in range(B)] == want


@pytest.mark.parametrize("budget_blocks", [1, 4, 1000])
def test_seed_windows_rotate_across_and_within_calls(budget_blocks):
    # windows of seeds over rotating buffers: a budget of 1 block gives one-chunk
    # windows over 2 buffers (rotation within a call), larger budgets several
    # windows in flight; consecutive streamed calls continue the rotation
    n, r, B = 50_000, 20_001, 11
    nb = (n + 7) // 8
    rng = np.random.default_rng(budget_blocks)
    eng = HashEngine(n, r, max_batch=3)
    budget = budget_blocks * 2 * nb
    firsts = (7, 18, 7)
    xs = [rng.integers(0, 256, size=(B, nb), dtype=np.uint8) for _ in firsts]
    outs = [eng.hash_seeded_host(torch.from_numpy(x).pin_memory(), 5, f, join_in=i == 0,
                                 join_out=False, seed_budget=budget)
            for i, (x, f) in enumerate(zip(xs, firsts))]
    eng.join()
    torch.cuda.synchronize()
    for x, f, o in zip(xs, firsts, outs):
        cs, ds = host_seeds(n, 5, f, B)
        for j in (0, 4, B - 1):
            assert o[j].numpy().tobytes() == oracle.compress(x[j].tobytes(), cs[j], ds[j], n, r)


@pytest.mark.parametrize("exclusive", [True, None])
def test_seed_windows_on_the_hashing_stream(exclusive):
    # the exclusive schedule: each seed window expanded on the hashing stream right
    # before its chunks (one buffer reused in stream order), forced on a small call
    # with ragged windows and chosen by size on a call of >= kExclusiveMin blocks;
    # keys equal the concurrent-window schedule's and the oracle's
    from paper_1910_04429_b200 import batch

    n, r = 4_160, 2_001
    B = 23 if exclusive else batch.kExclusiveMin + 300  # last chunk of 300: hashed in quarters
    nb = (n + 7) // 8
    rng = np.random.default_rng(B)
    x = rng.integers(0, 256, size=(B, nb), dtype=np.uint8)
    px = torch.from_numpy(x).pin_memory()
    eng = HashEngine(n, r, max_batch=4 if exclusive else 512)
    budget = 9 * 2 * nb if exclusive else 4 << 30  # forced: windows of 8 blocks (two chunks)
    outs = [eng.hash_seeded_host(px, 6, f, join_in=i == 0, join_out=False, seed_budget=budget,
                                 exclusive=exclusive) for i, f in enumerate((3, 90))]
    eng.join()
    torch.cuda.synchronize()
    assert eng._xw_win == (8 if exclusive else 4608)  # even windows of whole chunks
    ref = HashEngine(n, r, max_batch=64)
    for f, o in zip((3, 90), outs):
        want = ref.hash_seeded_host(px, 6, f, exclusive=False)
        torch.cuda.synchronize()
        assert torch.equal(o, want)
        cs, ds = host_seeds(n, 6, f, B)
        for j in (0, 7, 8, B - 1):
            assert o[j].numpy().tobytes() == oracle.compress(x[j].tobytes(), cs[j], ds[j], n, r)


def test_bench_protocol_seeds_match_the_reference_workload():
    # pab_seed_expand_bench: block seed s -> gen_seed(n, derive_block_seed(s, n)), the
    # reference benchmark's (c, d) (pkg/src/modpa/bench.py:156; workloads.block_inputs)
    from paper_1910_04429_b200 import workloads

    for n, first, B in ((1_000_000, 0, 3), (4_099, 255, 4), (130_001, 65_534, 3)):
        nb = (n + 7) // 8
        eng = HashEngine(n, n // 2, max_batch=B)
        c = torch.empty((B, nb + 8), dtype=torch.uint8, device="cuda")
        d = torch.empty_like(c)
        eng.seed_device(None, first, B, c, d, protocol="bench")
        torch.cuda.synchronize()
        for j in range(B):
            _, cw, dw = workloads.block_inputs(n, first + j)
            assert c[j, :nb].cpu().numpy().tobytes() == cw, (n, first + j)
            assert d[j, :nb].cpu().numpy().tobytes() == dw, (n, first + j)
    # the seeded engine path on the benchmark protocol equals hashing host (x, c, d)
    n, r, B = 200_000, 99_999, 5
    xs, cs, ds = workloads.batch_inputs(n, range(10, 10 + B))
    eng = HashEngine(n, r, max_batch=2)
    got = eng.hash_seeded_host(torch.from_numpy(xs).pin_memory(), None, 10, protocol="bench")
    torch.cuda.synchronize()
    for j in range(B):
        assert got[j].numpy().tobytes() == oracle.compress(xs[j].tobytes(), cs[j].tobytes(),
                                                           ds[j].tobytes(), n, r)
