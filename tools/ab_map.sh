# A/B of k_conv_map variants (env knobs) on the bench's C3 lines; parity subset under the first variant
mkdir -p gpurun_out
O=gpurun_out
: > $O/ab.log
APRGPU_MAP_THREADS=64 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -m gpu -q -x 2>&1 | tail -2 >> $O/ab.log
for v in "APRGPU_MAP_THREADS=128 APRGPU_MAP_COMPACT=1" "APRGPU_MAP_THREADS=64 APRGPU_MAP_COMPACT=1" "APRGPU_MAP_THREADS=64 APRGPU_MAP_COMPACT=0" "APRGPU_MAP_THREADS=128 APRGPU_MAP_COMPACT=0"; do
  env $v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $O/ab_bench.json 2>> $O/ab.err
  python -c "
import json; d = json.load(open('$O/ab_bench.json')); v = d['variants']
print('$v', 'k3_exact', d['ms_per_step'], 'k3_fast', v['k3_fast']['ms_per_step'])" >> $O/ab.log
done
cat $O/ab.log
