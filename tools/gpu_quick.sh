# quick pass: parity suite, C3 fast/exact bench, per-level tile-kernel launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -30 > gpurun_out/gputests.log
timeout 600 python bench.py --steps 10 --warmup 3 --config c3 --accum fast --no-cpu-baseline > gpurun_out/bench_c3_fast.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --config c3 --accum exact --no-cpu-baseline > gpurun_out/bench_c3_exact.log 2>&1
bash tools/gpu_levels.sh
