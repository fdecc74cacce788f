# one-box A/B of two builds of the library: bash tools/gpu_ab_so.sh nameA nameB [rounds]
# (build/ab/libaprgpu_<name>.so, swapped into paper_2112_03592_b200/_lib/ before each run)
A=$1; B=$2; R=${3:-2}
mkdir -p gpurun_out
cp paper_2112_03592_b200/_lib/libaprgpu.so build/ab/libaprgpu_current.so
for r in $(seq $R); do for x in $A $B; do
cp build/ab/libaprgpu_$x.so paper_2112_03592_b200/_lib/libaprgpu.so
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abso_$x.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/abso_$x.json')); print('$x', d['ms_per_step'], ' '.join(f'{k} {v[\"ms_per_step\"]}' for k, v in d['variants'].items()))"
done; done
cp build/ab/libaprgpu_current.so paper_2112_03592_b200/_lib/libaprgpu.so
