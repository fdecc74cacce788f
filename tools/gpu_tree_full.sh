# one ncu --set full capture of the finest tree-fill level (C3; k_fill_tree_flat, the node-parallel fill)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fill_tree_flat -s 4 -c 1 -o gpurun_out/tree_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --rl-iters 1 > gpurun_out/ncu_tree.log 2>&1
echo done
