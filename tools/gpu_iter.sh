# iteration pass on the GPU box: parity suite, C3 bench (fast + exact), launch list, optional ncu --set full
# usage: bash tools/gpu_iter.sh [full]
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -30 > gpurun_out/gputests.log
timeout 600 python bench.py --steps 10 --warmup 3 --config c3 --accum fast --no-cpu-baseline > gpurun_out/bench_c3_fast.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --config c3 --accum exact --no-cpu-baseline > gpurun_out/bench_c3_exact.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --config c3 --accum fast --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
if [ "$1" = "full" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-k_conv_map} -s 1 -c 1 -o gpurun_out/tile_full python bench.py --steps 1 --warmup 3 --config c3 --accum fast --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
fi
echo done
