"""Top warp-stall reasons, duration and L1 / DRAM utilisation from an `ncu --csv --page raw` file."""
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if r]
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[i], [r for r in rows[i + 2:] if len(r) == len(rows[i])]
    for r in data:
        g = lambda k: float(r[hdr.index(k)].replace(",", "") or 0) if k in hdr else float("nan")
        st = {k.split("stalled_")[1].split("_per")[0]: g(k) for k in hdr
              if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")}
        top = sorted(st.items(), key=lambda x: -x[1])[:6]
        print(f, r[hdr.index("Kernel Name")][:60])
        print("   duration", g("gpu__time_duration.sum"), "dram %", g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
              "l1 %", g("l1tex__throughput.avg.pct_of_peak_sustained_active"),
              "issue active %", g("smsp__issue_active.avg.pct_of_peak_sustained_active"))
        print("   stalls per issue:", [(k, round(v, 2)) for k, v in top])
