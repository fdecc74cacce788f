# per-level launch list of the tile kernel (time + instructions) on C3
mkdir -p gpurun_out
APRGPU_TILE_SPLIT=1 timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,launch__grid_size -k regex:${KREGEX:-k_conv_map} --clock-control none -c 24 --csv --log-file gpurun_out/levels_c3.csv python bench.py --steps 1 --warmup 3 --config c3 --accum fast --no-cpu-baseline > gpurun_out/ncu_levels.log 2>&1
echo done
