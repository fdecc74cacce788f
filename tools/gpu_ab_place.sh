# A/B of the bank-aware chunk placement (APRGPU_MAP_PLACE): parity subset, then bench conv lines
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_maps_gpu.py tests/test_fullsize_gpu.py tests/test_reference_fullsize_gpu.py -q -x -rf 2>&1 | tail -4 > $O/ab_tests.log
for r in 1; do
for p in 1 0; do
APRGPU_MAP_PLACE=$p timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $O/ab_bench_$p.json 2> $O/ab_bench_$p.err
python - $p <<'PY' >> $O/ab_tests.log
import json, sys
d = json.load(open(f"gpurun_out/ab_bench_{sys.argv[1]}.json"))
print("place", sys.argv[1], "k3_exact", d["ms_per_step"], d["roofline"]["frac"], " ".join(f"{k} {v['ms_per_step']}" for k, v in d["variants"].items()), "cold", d.get("cold_call", {}).get("ms"))
PY
done
done
cat $O/ab_tests.log
