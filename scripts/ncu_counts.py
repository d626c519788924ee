"""Per-launch ncu counters for bench.py's roofline (profiles/ncu_counts.json).

On the GPU box, under ncu (after the same command ran clean without it):
    python scripts/ncu_counts.py run C2        # bench's C2 batch: 1024 blocks per launch
    python scripts/ncu_counts.py run C5        # 64 blocks of n=1e8 per launch
    python scripts/ncu_counts.py run C4        # one n=1e8 block
    python scripts/ncu_counts.py run C3        # 64 blocks of n=1e7 per launch
    python scripts/ncu_counts.py run C1        # one n=1e6 block
Each run hashes the workload's batch twice (the second pass is the one kept).
Here, from the CSVs ncu wrote (--csv --log-file):
    python scripts/ncu_counts.py parse gpurun_out/ncu_counts_C2.csv ... -o profiles/ncu_counts.json
"""
import csv
import json
import sys

METRICS = ("smsp__inst_executed.sum,smsp__thread_inst_executed.sum,"
           "smsp__issue_active.avg.pct_of_peak_sustained_active,"
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,"
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,"
           "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,"
           "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
           "smsp__cycles_elapsed.avg.per_second")
SHAPES = {"C2": (1_000_000, 500_000, 1024), "C5": (100_000_000, 50_000_000, 64),
          "C4": (100_000_000, 50_000_000, 1), "C3": (10_000_000, 2_000_000, 64),
          "C1": (1_000_000, 500_000, 1)}
# CUDA kernel name -> the launcher's profile name (bench.py's kernel table)
FAMILY = (("k_col_fwd", "k_col_fwd"), ("k_colm_fwd", "k_col_fwd"), ("k_col_inv", "k_col_inv"),
          ("k_colm_inv", "k_col_inv"), ("k_carry", "k_carry"), ("k_row", "k_row"),
          ("k_pack", "k_pack"), ("k_unpack", "k_unpack"))


def run(workload):
    sys.path.insert(0, ".")
    import torch
    from paper_1910_04429_b200.batch import HashEngine

    n, r, B = SHAPES[workload]
    nb = (n + 7) // 8
    g = torch.Generator(device="cuda").manual_seed(0)
    x, c, d = (torch.randint(0, 256, (B, nb), dtype=torch.uint8, device="cuda", generator=g)
               for _ in range(3))
    c[:, 0] |= 1
    eng = HashEngine(n, r, max_batch=B, max_workspace=12 << 30)
    assert eng.chunk == B
    out = eng.hash_device(x, c, d)
    eng.hash_device(x, c, d, out)
    torch.cuda.synchronize()
    print("ran", workload, n, r, B)


def family(name):
    base = name.split("(")[0].split("<")[0].strip()
    if base.startswith("void "):
        base = base[5:]
    for pre, fam in FAMILY:
        if base.startswith(pre):
            return fam
    return base


def parse(paths, out_path):
    res = {"metrics": METRICS, "workloads": {}}
    try:
        with open(out_path) as f:
            res["workloads"] = json.load(f).get("workloads", {})
    except FileNotFoundError:
        pass
    for path in paths:
        wl = path.rsplit("_", 1)[-1].split(".")[0]
        n, r, B = SHAPES[wl]
        rows = {}
        with open(path) as f:
            lines = [ln for ln in f if ln.startswith('"')]
        for row in csv.DictReader(lines):
            key = int(row["ID"])
            rec = rows.setdefault(key, {"name": row["Kernel Name"]})
            rec[row["Metric Name"]] = float(row["Metric Value"].replace(",", ""))
        kern = {}
        for key in sorted(rows):  # later launches overwrite: the second pass is kept
            rec = rows[key]
            fam = family(rec["name"])
            kern[fam] = {
                "cuda_kernel": rec["name"].split("(")[0].replace("void ", ""),
                "inst": int(rec["smsp__inst_executed.sum"]),
                "thread_inst": int(rec["smsp__thread_inst_executed.sum"]),
                "issue_active": round(rec["smsp__issue_active.avg.pct_of_peak_sustained_active"] / 100, 4),
                "pipe_alu": round(rec["sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"] / 100, 4),
                "pipe_fma": round(rec["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"] / 100, 4),
                "pipe_fmaheavy": round(rec.get("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", -100) / 100, 4),
                "dram_bytes": int(rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"]),
                "duration_ms": round(rec["gpu__time_duration.sum"] / 1e6, 4),
                "sm_mhz": round(rec["smsp__cycles_elapsed.avg.per_second"] / 1e6, 1),
            }
        res["workloads"][wl] = {"n": n, "r": r, "batch": B, "source": path.split("/")[-1],
                                "kernels": kern}
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        args = sys.argv[2:]
        out = args[args.index("-o") + 1]
        parse([a for a in args if a.endswith(".csv")], out)
