# drop-in pass: the reference's own tests against the C++ drop-in, full GPU suite
mkdir -p gpurun_out
timeout 1200 ./tests/cpp/_build/unit_tests > gpurun_out/dropin_unit.log 2>&1; echo "unit rc=$?" >> gpurun_out/dropin_unit.log
timeout 1800 ./tests/cpp/_build/acceptance /tmp/fx 1 2 3 4 5 8 9 > gpurun_out/dropin_accept.log 2>&1; echo "acceptance rc=$?" >> gpurun_out/dropin_accept.log
timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | tail -30 > gpurun_out/gputests.log
echo done
