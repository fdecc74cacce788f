"""Per-CUDA-source-line instruction counts and stall samples from
`ncu -i rep --page source --print-source cuda,sass --csv` output."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None
hdr = None
agg = {}
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        ws = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None:
        continue
    if r[0]:
        if not r[0].isdigit():
            continue
        cur = (fname, int(r[0]), r[1][:80])
        agg.setdefault(cur, [0, 0])
        continue
    if cur is None:
        continue
    try:
        agg[cur][0] += int(r[ie])
        agg[cur][1] += int(r[ws])
    except (ValueError, IndexError):
        pass
tot = sum(v[0] for v in agg.values())
tots = sum(v[1] for v in agg.values())
print(f"total warp instructions {tot}, stall samples {tots}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / tot * 100:5.1f}% {v[1] / max(tots, 1) * 100:5.1f}%  {k[0]}:{k[1]}  {k[2]}")
