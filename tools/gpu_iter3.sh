# quick iteration on the hot kernel: parity subset + the bench's conv lines (+ A/B env passed through)
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_slab.py tests/test_multi_gpu.py -m gpu -q -x -rf 2>&1 | tail -5 > $O/iter_tests.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $O/iter_bench.json 2> $O/iter_bench.err
APRGPU_MAP_COMPACT=0 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $O/iter_bench_full.json 2>> $O/iter_bench.err
python - <<'PY' >> $O/iter_tests.log
import json
for f in ("gpurun_out/iter_bench.json", "gpurun_out/iter_bench_full.json"):
    d = json.load(open(f))
    print(f, "k3_exact", d["ms_per_step"], d["roofline"]["frac"], "traffic", d["roofline"].get("traffic"))
    for k, v in d["variants"].items():
        print("  ", k, v["ms_per_step"], v["roofline"]["frac"])
    print("  paper", d["paper_protocol"]["ms_per_step"], "cold", d.get("cold_call", {}).get("ms"))
PY
cat $O/iter_tests.log
