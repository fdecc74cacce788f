# drop-in pass: the reference's own tests against the C++ drop-in (all ten
# acceptance criteria; 10 with its fixtures written first, then read back)
mkdir -p gpurun_out /tmp/fx
timeout 1200 ./tests/cpp/_build/unit_tests > gpurun_out/dropin_unit.log 2>&1; echo "unit rc=$?" >> gpurun_out/dropin_unit.log
timeout 600 ./tests/cpp/_build/acceptance /tmp/fx --write-fixtures 10 > /dev/null 2>&1
timeout 1800 ./tests/cpp/_build/acceptance /tmp/fx > gpurun_out/dropin_accept.log 2>&1; echo "acceptance rc=$?" >> gpurun_out/dropin_accept.log
echo done
