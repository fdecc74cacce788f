# quick map-kernel timing: C3 5^3 FAST/EXACT and 3^3 FAST bench lines + per-launch list (5^3)
mkdir -p gpurun_out
for a in fast exact; do timeout 600 python bench.py --steps 30 --warmup 3 --stencil 5 --accum $a --no-cpu-baseline > gpurun_out/p5$a.json 2>gpurun_out/p.err; done
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/p3fast.json 2>>gpurun_out/p.err
timeout 600 ncu --metrics gpu__time_duration.sum,launch__occupancy_limit_shared_mem,launch__shared_mem_per_block_dynamic --clock-control none -k regex:"k_conv_map" -s 4 -c 4 --csv --log-file gpurun_out/l5.csv python bench.py --steps 2 --warmup 3 --stencil 5 --no-cpu-baseline > /dev/null 2>&1
