# Evidence pass for a round (one GPU): parity suite + smoke, bench lines, launch
# list and dram traffic of the bench command, ncu --set full of the top kernel.
#   bash tools/gpu_round.sh [quick]
mkdir -p gpurun_out
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf 2>&1 | tail -30 > $O/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --accum exact --no-cpu-baseline > $O/bench_c3_k3_exact.json 2>&1
timeout 900 python bench.py --stencil 5 --no-cpu-baseline > $O/bench_c3_k5_fast.json 2>&1
timeout 900 python bench.py --stencil 5 --accum exact --no-cpu-baseline > $O/bench_c3_k5_exact.json 2>&1
timeout 600 python bench.py --config c1 --no-cpu-baseline > $O/bench_c1_k3_fast.json 2>&1
timeout 1200 python bench.py --config c4 --steps 10 --no-cpu-baseline > $O/bench_c4_k3_fast.json 2>&1
timeout 1200 python bench.py --config c4 --steps 10 --stencil 5 --no-cpu-baseline > $O/bench_c4_k5_fast.json 2>&1
[ "$1" = "quick" ] && exit 0
timeout 1200 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2>&1
# launch list of the bench command (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_conv|k_fill_tree|k_tree_finalize|k_mean" -c 300 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
# dram traffic of one warm conv pass per variant (the 3rd conv launch: after the two warm-up passes)
for st in 3 5; do for acc in fast exact; do
if [ $st = 3 ]; then SK=2; CN=1; else SK=4; CN=2; fi   # 5^3 restricted: one 3^3 launch + one 5^3 launch per pass
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_conv" -s $SK -c $CN --csv --log-file $O/traffic_c3_k${st}_${acc}.csv python bench.py --steps 1 --warmup 3 --stencil $st --accum $acc --no-cpu-baseline > /dev/null 2>&1
done; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_map -s 1 -c 1 -o $O/conv_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
echo done
