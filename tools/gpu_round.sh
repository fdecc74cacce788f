set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | tail -60 > gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --config c1 --cpu-seconds 5 > gpurun_out/bench_c1.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --config c3 --cpu-seconds 10 > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --config c3 --accum fast --no-cpu-baseline > gpurun_out/bench_c3_fast.log 2>&1
tail -3 gpurun_out/*.log
