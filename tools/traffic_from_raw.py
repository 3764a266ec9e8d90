"""profiles/r02_traffic.json from the `ncu --set full` raw CSVs of the half-storage
residual pass (tools/ncu_sym_r02.sh): DRAM bytes (read + write) and duration of the
first phase-1 + merge pair, beside the pass's algorithmic bytes printed by
tools/profile_sym.py.  usage: python tools/traffic_from_raw.py KEY=raw.csv:plain.log ..."""
import csv
import json
import sys

out = {}
for spec in sys.argv[1:]:
    key, rest = spec.split("=", 1)
    raw, plain = rest.split(":")
    rows = [r for r in csv.reader(open(raw)) if r]
    i = next(k for k, r in enumerate(rows) if r[0] == "ID")
    hdr, units, data = rows[i], rows[i + 1], [r for r in rows[i + 2:] if len(r) == len(rows[i])]
    alg = json.loads([ln for ln in open(plain) if ln.startswith("{")][-1])["algorithmic_bytes"]

    def val(r, k):
        v = float(r[hdr.index(k)].replace(",", ""))
        u = units[hdr.index(k)]
        return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0), u

    kern, tot = [], 0.0
    for r in data[:2]:  # phase 1 + merge of the first captured pass
        b = val(r, "dram__bytes_read.sum")[0] + val(r, "dram__bytes_write.sum")[0]
        t, tu = val(r, "gpu__time_duration.sum")
        kern.append([r[hdr.index("Kernel Name")][:60], b, f"{t:.6f} {tu}"])
        tot += b
    out[key] = {"dram_bytes_per_launch": int(tot), "algorithmic_bytes": alg, "kernels": kern,
                "source": f"{raw.replace('gpurun_out/', 'profiles/')} (ncu --set full, finest residual pass in the "
                          f"symmetric-half form: bsr_stream_kernel<..., EpiStore, 0, 1> + sym_merge_kernel, "
                          f"dram__bytes_read.sum + dram__bytes_write.sum of both launches)"}
print(json.dumps(out, indent=1))
