"""The C ABI from a plain-C program (examples/capi_demo.c): it compiles with gcc
against include/pa_b200.h, links libpa_b200.so and runs without a GPU (CPU test);
on a B200 it hashes a block end to end, checked against the oracle (GPU test)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1910_04429_b200", "_lib")


def _build(tmp_path):
    exe = str(tmp_path / "capi_demo")
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "capi_demo.c"), "-L", LIBDIR, "-lpa_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_c_program_links_and_queries(tmp_path):
    exe = _build(tmp_path)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stderr
    assert "pa_b200 ABI 102, max block 335544320 bits" in res.stdout


@pytest.mark.gpu
def test_c_program_hashes_a_block(tmp_path):
    import oracle
    from paper_1910_04429_b200 import workloads

    exe = _build(tmp_path)
    n, r = 1_000_003, 333_337
    x, c, d = workloads.block_inputs(n, 9)
    paths = []
    for name, v in (("x", x), ("c", c), ("d", d)):
        p = tmp_path / f"{name}.bin"
        p.write_bytes(v)
        paths.append(str(p))
    out = tmp_path / "out.bin"
    res = subprocess.run([exe, str(n), str(r), *paths, str(out)], capture_output=True, text=True,
                         timeout=300)
    assert res.returncode == 0, res.stderr
    assert out.read_bytes() == oracle.compress(x, c, d, n, r)


@pytest.mark.gpu
def test_c_program_hashes_a_key_file(tmp_path):
    # run_pa's scope from C: one pab_hash_seeded_host call over a key file (several chunks),
    # every sampled key against the oracle on host-derived seeds
    import numpy as np

    import oracle
    from paper_1910_04429_b200 import pa

    exe = _build(tmp_path)
    n, r, blocks, seed = 65_536, 20_000, 1_500, 200
    nb, rb = n // 8, r // 8
    data = np.random.default_rng(1).integers(0, 256, size=blocks * nb, dtype=np.uint8)
    key, out = tmp_path / "key.bin", tmp_path / "keys.bin"
    key.write_bytes(data.tobytes())
    res = subprocess.run([exe, "keyfile", str(n), str(r), str(blocks), str(seed), str(key), str(out)],
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    got = out.read_bytes()
    assert len(got) == blocks * rb
    x = data.reshape(blocks, nb)
    for i in (0, 1, 1023, 1024, blocks - 1):
        s = pa.gen_seed(n, pa.derive_block_seed(seed, i))
        assert got[i * rb:(i + 1) * rb] == oracle.compress(
            x[i].tobytes(), s.c.value.to_bytes(nb, "little"), s.d.value.to_bytes(nb, "little"), n, r), i
