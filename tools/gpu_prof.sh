# profile pass: GPU tests, rows-vs-tile bench, ncu --set full of the finest-level tile launch
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | tail -30 > gpurun_out/gputests.log
APRGPU_CONV_KERNEL=rows timeout 600 python bench.py --steps 10 --warmup 3 --config c3 --accum fast --no-cpu-baseline > gpurun_out/bench_c3_rows_fast.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --config c3 --accum fast --no-cpu-baseline > gpurun_out/bench_c3_tile_fast.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_tile -c 1 -o gpurun_out/tile_l10 python bench.py --steps 1 --warmup 3 --config c3 --accum fast --no-cpu-baseline > gpurun_out/ncu_tile.log 2>&1
echo done
