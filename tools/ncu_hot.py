"""Top stall locations (SASS) of an ncu report: python tools/ncu_hot.py <rep> [n]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
k = idx["Warp Stall Sampling (All Samples)"]
data = []
for r in rows[2:]:
    if len(r) <= k:
        continue
    try:
        data.append((float(r[k] or 0), r[idx["Address"]], r[idx["Source"]]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
for d in sorted(data, reverse=True)[:n]:
    print(f"{100 * d[0] / tot:5.1f}%  {d[1]}  {d[2][:120]}")
