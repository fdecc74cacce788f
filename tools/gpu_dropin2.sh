# drop-in after the overlapped result vector: the reference's unit tests + acceptance, drop-in timing, pipeline tests
mkdir -p gpurun_out /tmp/fx
timeout 900 python -m pytest tests/test_pipeline_gpu.py tests/test_dropin_gpu.py -q -x -rf 2>&1 | tail -4 > gpurun_out/dropin2.log
for i in 1 2; do timeout 300 ./tests/cpp/_build/dropin_time 1024 10 >> gpurun_out/dropin2.log 2>&1; done
cat gpurun_out/dropin2.log
