mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pixels_zreg -s 1 -c 1 -o gpurun_out/pix_zreg python tools/pix_one.py ${ACC:-fast} > gpurun_out/pixncu.log 2>&1
tail -2 gpurun_out/pixncu.log
