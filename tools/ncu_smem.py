"""Per-CUDA-source-line shared-memory wavefronts (total / excessive) and
global sectors from `ncu -i rep --page source --print-source cuda,sass --csv`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[2]
col = {k: hdr.index(k) for k in ("L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive",
                                  "Warp Stall Sampling (All Samples)", "Instructions Executed")}
agg = {}
cur = None
for r in rows[3:]:
    if not r or len(r) < 4:
        continue
    if r[0] and r[0].isdigit():
        cur = (int(r[0]), r[1][:70])
        continue
    if r[2][:2] != "0x" or cur is None:
        continue
    a = agg.setdefault(cur, [0.0] * 4)
    for i, k in enumerate(col):
        try:
            a[i] += float(r[col[k]] or 0)
        except ValueError:
            pass
tot = [sum(v[i] for v in agg.values()) or 1 for i in range(4)]
print("wavefronts shared %.0f, excessive %.0f" % (tot[0], tot[1]))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
    print("%6.1f%% exc %6.1f%% wf  %5d  %s" % (100 * v[1] / tot[1], 100 * v[0] / tot[0], k[0], k[1]))
