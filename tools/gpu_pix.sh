# pixel-kernel A/B: ncu kernel durations of tools/pix_ab.py under env variants; parity first
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pixels.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pix.log
i=0
for v in ${PIX_VARIANTS:-"X=0"}; do
  i=$((i+1))
  env $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:convolve_pixels --csv --log-file gpurun_out/pix_$i.csv python tools/pix_ab.py > /dev/null 2>&1
  python - gpurun_out/pix_$i.csv "$v" >> gpurun_out/pix.log <<'PY'
import csv, sys
rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))]
names = ["k3 exact", "k3 fast", "k5 exact", "k5 fast"]
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
out = []
for i, nm in enumerate(names):
    rs = rows[4 * i:4 * i + 4]
    t = min(float(r["Metric Value"]) * scale[r["Metric Unit"]] for r in rs[1:])
    out.append(f"{nm} {t:.3f} ms ({8 * 1024 ** 3 / (t / 1e3) / 1e9 / 6377.7:.3f})")
print(sys.argv[2], " | ".join(out))
PY
done
cat gpurun_out/pix.log
