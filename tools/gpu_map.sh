# map-path profile: per-level launch list + one ncu --set full of the fused (all-level) map launch
mkdir -p gpurun_out
bash tools/gpu_levels.sh
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_map -s 1 -c 1 -o gpurun_out/map_full python bench.py --steps 1 --warmup 3 --config c3 --accum fast --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
