# one ncu --set full capture of the first finest-level conv launch (C3, fast)
mkdir -p gpurun_out
APRGPU_TILE_SPLIT=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-k_conv_map} -s 7 -c 1 -o gpurun_out/seg_full python bench.py --steps 1 --warmup 3 --config c3 --accum ${ACCUM:-fast} --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
