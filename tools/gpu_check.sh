# parity subset + sanitizers + bench lines on the default build
mkdir -p gpurun_out
O=gpurun_out
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_sanitizer_gpu.py tests/test_concurrency_gpu.py tests/test_slab.py tests/test_multi_gpu.py tests/test_pipeline_gpu.py tests/test_reference_fullsize_gpu.py -m gpu -q -x -rf 2>&1 | tail -4 > $O/check.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $O/check_bench.json 2>> $O/check.err
python -c "
import json; d = json.load(open('$O/check_bench.json')); v = d['variants']
print('k3_exact', d['ms_per_step'], d['roofline']['frac'], 'k3_fast', v['k3_fast']['ms_per_step'], 'k5_exact', v['k5_exact']['ms_per_step'], 'k5_fast', v['k5_fast']['ms_per_step'], 'e2e', d['e2e'], 'launches', d.get('gpu_launches'))" >> $O/check.log
cat $O/check.log
