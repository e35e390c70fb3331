#!/bin/bash
# the driver's round-end GPU test command, as is (slow tests included)
O=gpurun_out; mkdir -p $O
start=$(date +%s)
timeout 3000 python -m pytest tests/ -x -q -m gpu --durations=15 > $O/r2w_pytest_gpu_all.log 2>&1; echo "rc=$? elapsed=$(( $(date +%s) - start ))s" >> $O/r2w_pytest_gpu_all.log
echo done
