"""Summarise ncu --set full captures (.ncu-rep) into the text kept under profiles/:
python scripts/ncu_full_summary.py rep1 rep2 ... > profiles/rN/ncu_full_TAG.txt"""
import csv
import io
import subprocess
import sys

WANT = (("gpu__time_duration.sum", "duration"),
        ("launch__registers_per_thread", "registers/thread"),
        ("launch__occupancy_limit_registers", "CTAs/SM by registers"),
        ("launch__occupancy_limit_shared_mem", "CTAs/SM by shared memory"),
        ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active"),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe"),
        ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "FMA-heavy pipe"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe"),
        ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("smsp__inst_executed.sum", "warp instructions"),
        ("smsp__cycles_elapsed.avg.per_second", "SM clock"))

for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = [r for r in csv.reader(io.StringIO(raw)) if r]
    hdr, units, vals = rows[0], rows[1], rows[2]
    H = {h: i for i, h in enumerate(hdr)}
    name = vals[H["Kernel Name"]]
    print(f"== {name}   ({rep.split('/')[-1]})")
    for key, label in WANT:
        if key in H:
            print(f"  {label:26s} {float(vals[H[key]]):.6g} {units[H[key]]}")
    src = subprocess.run([sys.executable, "scripts/ncu_source_summary.py", rep, name.replace("void ", "").split("<")[0].split("(")[0]],
                         capture_output=True, text=True).stdout
    print("  " + src.strip().replace("\n", "\n  "))
    print()
