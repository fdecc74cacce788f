# debugging pass: sanitizer on the first failing parity case, rows-kernel run of the suite, ncu launch list of C3
mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -x -q "tests/test_parity_gpu.py::test_convolve_exact_bit_identical_to_reference[random_apr_00]" > gpurun_out/san.log 2>&1
APRGPU_CONV_KERNEL=rows timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | tail -40 > gpurun_out/gputests_rows.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --config c3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
echo done
