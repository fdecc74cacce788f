mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_reconstruct.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/recon.log
for v in X=0 APRGPU_RECON_SMEM=0; do
env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/recon_bench.json 2>/dev/null
python -c "
import json; d = json.load(open('gpurun_out/recon_bench.json')); print('$v', d['reconstruct_full'])" >> gpurun_out/recon.log
done
cat gpurun_out/recon.log
