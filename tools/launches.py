"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = defaultdict(lambda: defaultdict(float))
order = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    k = d["Kernel Name"][:90]
    key = (d["ID"], k)
    if key not in agg:
        order.append(key)
    v = float(d["Metric Value"].replace(",", ""))
    agg[key][d["Metric Name"]] = v
print(f"{'id':>4} {'us':>9} {'MB_read':>9} {'MB_write':>9}  kernel")
for key in order:
    m = agg[key]
    t = m.get("gpu__time_duration.sum", 0.0)
    print(f"{key[0]:>4} {t / 1e3:9.1f} {m.get('dram__bytes_read.sum', 0) / 1e6:9.2f} "
          f"{m.get('dram__bytes_write.sum', 0) / 1e6:9.2f}  {key[1]}")
