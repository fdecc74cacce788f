# k_map_place / build kernel durations on C3 (3^3 EXACT and 5^3 FAST map builds)
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_map_place|k_conv_tile" --csv --log-file gpurun_out/place_t3.csv python tools/one_pass.py 3 exact > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_map_place|k_conv_tile" --csv --log-file gpurun_out/place_t5.csv python tools/one_pass.py 5 fast > /dev/null 2>&1
