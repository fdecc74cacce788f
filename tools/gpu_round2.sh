# Evidence pass for round 2 (one GPU): parity suite + smoke, bench lines, the
# launch list of the bench command, per-variant dram traffic of one conv pass,
# ncu --set full of the 3^3 EXACT map kernel.   bash tools/gpu_round2.sh
mkdir -p gpurun_out
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf 2>&1 | tail -30 > $O/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_c3_k3_exact.json 2> $O/bench_default.err
timeout 900 python bench.py --accum fast --no-cpu-baseline > $O/bench_c3_k3_fast.json 2>&1
timeout 900 python bench.py --stencil 5 --no-cpu-baseline > $O/bench_c3_k5_exact.json 2>&1
timeout 900 python bench.py --config c1 --no-cpu-baseline > $O/bench_c1_k3_exact.json 2>&1
timeout 1200 python bench.py --config c4 --steps 10 --no-cpu-baseline > $O/bench_c4_k3_exact.json 2>&1
timeout 1200 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_conv|k_fill_tree|k_mark|k_mean|k_clamp|DeviceSelect|DeviceScan" -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --rl-iters 1 > $O/ncu_launches.log 2>&1
for st in 3 5; do for acc in exact fast; do
if [ $st = 3 ]; then SK=2; CN=1; else SK=4; CN=2; fi
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_conv_map -s $SK -c $CN --csv --log-file $O/traffic_c3_k${st}_${acc}.csv python tools/one_pass.py $st $acc > /dev/null 2>&1
done; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_map -s 2 -c 1 -o $O/conv_full python tools/one_pass.py 3 exact > $O/ncu_full.log 2>&1
echo done
