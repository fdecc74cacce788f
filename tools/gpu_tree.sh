# launch list of the tree fill + conv kernels (times per launch, dram bytes)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_fill_tree|k_tree_finalize|k_conv_map|k_rl|k_mean" -c 120 --csv --log-file gpurun_out/tree_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --rl-iters 2 > gpurun_out/tree_ncu.log 2>&1
echo done
