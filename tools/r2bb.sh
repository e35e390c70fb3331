#!/bin/bash
# end-of-round check: the driver's GPU test command, smoke, and the default bench
O=gpurun_out; mkdir -p $O; rm -f $O/*.ncu-rep
start=$(date +%s)
timeout 2400 python -m pytest tests/ -x -q -m gpu > $O/r2bb_pytest_gpu_all.log 2>&1; echo "rc=$? elapsed=$(( $(date +%s) - start ))s" >> $O/r2bb_pytest_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2bb_smoke.log 2>&1; echo "rc=$?" >> $O/r2bb_smoke.log
timeout 1200 python bench.py > $O/r2bb_bench.json 2> $O/r2bb_bench.err
echo done
