"""Summaries of ncu output for profiles/: launch-list shares and key raw metrics."""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    k = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = (d["ID"], d["Kernel Name"])
            k.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for (i, name), ms in k.items():
        t = ms.get("gpu__time_duration.sum", 0.0)
        b = ms.get("dram__bytes_read.sum", 0.0) + ms.get("dram__bytes_write.sum", 0.0)
        a = agg[name]
        a[0] += 1
        a[1] += t
        a[2] += b
        tot += t
    out = [f"launches: {len(k)}, total device time {tot / 1e3:.1f} us (ncu, serialised, cold-ish caches)"]
    out.append(f"{'count':>5} {'time_us':>10} {'share':>6} {'dram_MB':>9} {'GB/s':>7}  kernel")
    for name, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{c:5d} {t / 1e3:10.1f} {100 * t / tot:5.1f}% {b / 1e6:9.1f} {b / t:7.0f}  {name[:100]}")
    return "\n".join(out)


RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
       "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
       "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    out = []
    for w in RAW:
        if w in hdr:
            i = hdr.index(w)
            out.append(f"{w:60s} {units[i]:14s} " + " ".join(v[i] for v in vals))
    # stall reasons (warp state)
    st = [(h, i) for i, h in enumerate(hdr) if h.startswith("smsp__average_warp_latency_issue_stalled")
          or h.startswith("smsp__pcsamp_warps_issue_stalled")]
    samp = []
    for h, i in st:
        try:
            v = float(vals[0][i])
        except Exception:
            continue
        if v > 0:
            samp.append((v, h))
    samp.sort(reverse=True)
    out.append("top stall counters (first launch):")
    for v, h in samp[:10]:
        out.append(f"  {h:80s} {v:.0f}")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else raw(path))
