"""Summarise tools/gpu_levels.sh output (per-level tile-kernel launches)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/levels_c3.csv")))
hdr = None
agg = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        if unit == "ms":
            v *= 1e6
        elif unit == "us":
            v *= 1e3
        agg.setdefault(int(d["ID"]), {})[d["Metric Name"]] = v
for k in sorted(agg):
    m = agg[k]
    g = m["launch__grid_size"]
    print(f"{k:3d} blocks {int(g):6d}  {m['gpu__time_duration.sum'] / 1e3:9.1f} us  "
          f"inst/block {m['smsp__inst_executed.sum'] / g:8.0f}  dram_read {m['dram__bytes_read.sum'] / 1e6:8.2f} MB")
