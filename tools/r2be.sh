#!/bin/bash
# the opt-in C5 stepwise parity test (whole-graph oracle checks of sweeps 1-4, 25, 50, 100,
# the merge, the level-0 contraction and every level's Q)
O=gpurun_out; mkdir -p $O; rm -f $O/*.ncu-rep
free -g > $O/r2be_mem.txt
start=$(date +%s)
LV_STEPWISE_C5=1 timeout 2400 python -m pytest tests/test_gpu_fullsize_stepwise.py -m "gpu and slow" -x -q -s -k c5 > $O/r2be_stepwise_c5.log 2>&1; echo "rc=$? elapsed=$(( $(date +%s) - start ))s" >> $O/r2be_stepwise_c5.log
echo done
