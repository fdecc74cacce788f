cp build/ab/libaprgpu_head.so paper_2112_03592_b200/_lib/libaprgpu.so
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_maps_gpu.py tests/test_slab.py -q -x 2>&1 | tail -1
bash tools/gpu_ab_so.sh full head 2
for v in full head; do
cp build/ab/libaprgpu_$v.so paper_2112_03592_b200/_lib/libaprgpu.so
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_conv_map -s 2 -c 1 --csv --log-file gpurun_out/tr_$v.csv python tools/one_pass.py 3 exact > /dev/null 2>&1
python - $v <<'PY'
import csv, sys
rows=[r for r in csv.reader(open(f"gpurun_out/tr_{sys.argv[1]}.csv")) if len(r)>10]
h=rows[0]
print(sys.argv[1], [(dict(zip(h,r))["Metric Name"], dict(zip(h,r))["Metric Value"]) for r in rows[1:]])
PY
done
cp build/ab/libaprgpu_head.so paper_2112_03592_b200/_lib/libaprgpu.so
