"""Top SASS instructions of an ncu report by warp-stall samples (source page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
ia, isrc, isamp = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[1:] if len(r) > isamp and r[isamp].isdigit()]
tot = sum(int(r[isamp]) for r in body) or 1
for i, r in enumerate(body):
    r.append(i)
for r in sorted(body, key=lambda r: -int(r[isamp]))[:n]:
    print(f"{int(r[isamp]) / tot * 100:5.1f}%  #{r[-1]:4d}  {r[isrc].strip()}")
