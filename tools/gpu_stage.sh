mkdir -p gpurun_out
O=gpurun_out
timeout 600 ./tests/cpp/_build/dropin_time 1024 10 > $O/stage.log 2>&1
cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag >> $O/stage.log 2>&1
cat $O/stage.log
