# EXPERIMENT: timing upper bound of a smaller F (tiles beyond the cap skipped -> wrong results, timing only)
for c in 0 768 640 512; do
if [ $c = 0 ]; then unset APRGPU_EXP_NGCAP; else export APRGPU_EXP_NGCAP=$c; fi
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ngcap_$c.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ngcap_$c.json')); print('cap', $c, d['ms_per_step'], d['variants']['k3_fast']['ms_per_step'])"
done
