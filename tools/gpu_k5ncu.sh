# ncu --set full of the 5^3 launch (k_conv_map<Acc, 2>) of one warm C3 pass
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_map -s 5 -c 1 -o gpurun_out/k5_${ACC:-exact} python tools/one_pass.py 5 ${ACC:-exact} > gpurun_out/k5ncu.log 2>&1
tail -2 gpurun_out/k5ncu.log
