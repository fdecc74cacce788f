# A/B of k_conv_map variants (env knobs, AB_VARIANTS) on the bench's C3 lines; parity subset under AB_PARITY_ENV
mkdir -p gpurun_out
O=gpurun_out
: > $O/ab.log
env ${AB_PARITY_ENV:-X=0} timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -m gpu -q -x 2>&1 | tail -2 >> $O/ab.log
for v in ${AB_VARIANTS:-X=0}; do
  env $(echo $v | tr ',' ' ') timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $O/ab_bench.json 2>> $O/ab.err
  python -c "
import json; d = json.load(open('$O/ab_bench.json')); v = d['variants']
print('$v', 'k3_exact', d['ms_per_step'], 'k3_fast', v['k3_fast']['ms_per_step'], 'k5_exact', v['k5_exact']['ms_per_step'], 'k5_fast', v['k5_fast']['ms_per_step'])" >> $O/ab.log
done
cat $O/ab.log
