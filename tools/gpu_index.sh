mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_concurrency_gpu.py -m gpu -q -x -k "rebuild_index or concurrent or index_step" 2>&1 | tail -3 > gpurun_out/index.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/index_bench.json 2>> gpurun_out/index.log
python -c "
import json; d = json.load(open('gpurun_out/index_bench.json')); print('paper', d['paper_protocol']['ms_per_step'], 'k3', d['ms_per_step'])" >> gpurun_out/index.log
cat gpurun_out/index.log
