for c in 58 72 86 100; do
  APRGPU_CARVEOUT_EXACT=$c timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --rl-iters 1 > gpurun_out/ab_$c.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_$c.json')); print('carve $c', d['ms_per_step'], d['variants']['k5_exact']['ms_per_step'])"
done
