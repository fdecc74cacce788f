# one-box A/B of an environment knob: bash tools/gpu_ab_env.sh VAR v1 v2 [rounds]
V=$1; A=$2; B=$3; R=${4:-2}
mkdir -p gpurun_out
for r in $(seq $R); do for x in $A $B; do
env $V=$x timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abenv_$x.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/abenv_$x.json')); print('$V=$x', d['ms_per_step'], ' '.join(f'{k} {v[\"ms_per_step\"]}' for k, v in d['variants'].items()))"
done; done
