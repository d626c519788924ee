"""Summarise an ncu --page source CSV export: stall reasons, hot SASS, smem excess, opcode mix."""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = [r for r in csv.reader(io.StringIO(txt)) if r]
hdr = next(r for r in rows if r[0] == "Address")
body = [r for r in rows if r[0] not in ("Address", "Kernel Name") and len(r) >= len(hdr) - 1]
body = [r + [""] * (len(hdr) - len(r)) for r in body]
H = {h: i for i, h in enumerate(hdr)}
num = lambda r, k: float(r[H[k]] or 0) if r[H[k]] not in ("-", "") else 0.0
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
ops = collections.Counter()
for r in body:
    for s in stalls:
        tot[s] += num(r, s)
    op = r[H["Source"]].strip().split()[0] if r[H["Source"]].strip() else "?"
    if op.startswith("@"):
        op = r[H["Source"]].strip().split()[1]
    ops[op.split(".")[0]] += num(r, "Instructions Executed")
S = sum(tot.values()) or 1
print("stall samples:", ", ".join(f"{k[6:]} {v / S:.1%}" for k, v in tot.most_common(8)))
I = sum(ops.values()) or 1
print("warp-inst mix:", ", ".join(f"{k} {v / I:.1%}" for k, v in ops.most_common(14)))
print(f"total warp instructions: {I:.3e}")
hot = sorted(body, key=lambda r: -num(r, "# Samples"))[:12]
print("hot instructions (samples):")
for r in hot:
    print(f"  {num(r, '# Samples'):7.0f}  {r[H['Source']].strip()[:70]}")
exc = sorted(body, key=lambda r: -num(r, "L1 Wavefronts Shared Excessive"))[:8]
print("smem excessive wavefronts:")
for r in exc:
    if num(r, "L1 Wavefronts Shared Excessive") > 0:
        print(f"  {num(r, 'L1 Wavefronts Shared Excessive'):10.0f} / {num(r, 'L1 Wavefronts Shared'):10.0f}  {r[H['Source']].strip()[:60]}")
