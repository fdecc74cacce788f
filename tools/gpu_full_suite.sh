# the whole GPU suite + smoke (checkpoint)
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/suite.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/suite.log 2>&1
cat gpurun_out/suite.log
