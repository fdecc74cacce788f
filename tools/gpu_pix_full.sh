# one ncu --set full capture of the streamed pixel convolution (C3 image, 3^3 FAST)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_convolve_pixels -s 1 -c 1 -o gpurun_out/pix_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --rl-iters 1 > gpurun_out/ncu_pix.log 2>&1
echo done
