"""Write profiles/<round>/traffic.json from ncu --csv dram captures.

usage: python tools/traffic.py <round> key=path.csv [key=path.csv ...]
Each csv holds ONE conv pass (all k_conv_tile / k_conv launches of it); the
value stored under key is the sum of dram__bytes_read.sum + dram__bytes_write.sum.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def dram_bytes(path):
    rows = list(csv.reader(open(path)))
    hdr, tot, n = None, 0.0, 0
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                v = float(d["Metric Value"].replace(",", ""))
                unit = d["Metric Unit"]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
                tot += v * scale.get(unit, 1)
                n += 1
    return int(tot) if n else None


rnd = sys.argv[1]
out_path = os.path.join(ROOT, "profiles", rnd, "traffic.json")
os.makedirs(os.path.dirname(out_path), exist_ok=True)
data = {}
if os.path.exists(out_path):
    data = json.load(open(out_path))
for kv in sys.argv[2:]:
    k, p = kv.split("=", 1)
    if os.path.exists(p):
        v = dram_bytes(p)
        if v is not None:
            data[k] = v
json.dump(data, open(out_path, "w"), indent=1, sort_keys=True)
print(json.dumps(data))
