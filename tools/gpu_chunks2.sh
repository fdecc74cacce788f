# e2e vs APRGPU_HOST_CHUNKS on one box (two rounds)
for r in 1 2; do for c in 8 6 5; do
APRGPU_HOST_CHUNKS=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/chunks_$c.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/chunks_$c.json')); print('chunks', $c, 'e2e ms', d['e2e']['ms_per_step'])"
done; done
