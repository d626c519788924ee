"""Per-source-line stall samples and instruction counts of one kernel from an ncu report
(--page source --print-source cuda,sass; compile with -lineinfo).  Development aid."""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
path, hdr = None, None
samples = collections.Counter()
insts = collections.Counter()
text = {}
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 8 or not r[0].isdigit():
        continue
    key = (path, int(r[0]))
    text[key] = r[1]
    s = r[hdr["Warp Stall Sampling (All Samples)"]]
    n = r[hdr["Instructions Executed"]]
    try:
        samples[key] += float(s or 0)
        insts[key] += float(n or 0)
    except ValueError:
        continue
tot = sum(samples.values()) or 1
itot = sum(insts.values()) or 1
print(f"total samples {tot:.0f}, warp instructions {itot:.3e}")
for key, v in samples.most_common(top):
    print(f"{100 * v / tot:5.1f}% smp {100 * insts[key] / itot:5.1f}% inst  {key[0]}:{key[1]}: "
          f"{text[key].strip()[:100]}")
