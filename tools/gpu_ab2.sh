mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_maps_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/ab_pre.log
bash tools/ab_map.sh > /dev/null 2>&1
cat gpurun_out/ab_pre.log gpurun_out/ab.log
