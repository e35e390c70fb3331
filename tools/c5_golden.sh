#!/bin/bash
# C5 (R-MAT scale 27) golden on the GPU box's host (196 GB RAM, 16 cores): the oracle's
# full run (tools/oracle_golden.py: oracle/ + seeded generators only).  A gpurun call is
# limited to 60 min, so the GPU's full-run comparison (tests/test_gpu_fullsize_golden.py,
# slow) runs in a later call (tools/c5_compare.sh) once tests/golden/rmat27.json is in.
O=gpurun_out; mkdir -p $O
free -g > $O/c5_mem.txt; nproc >> $O/c5_mem.txt; lscpu | grep "Model name" >> $O/c5_mem.txt
( while true; do free -g | sed -n 2p >> $O/c5_mem_trace.txt; sleep 60; done ) &
MON=$!
start=$(date +%s)
timeout ${ORACLE_TIMEOUT:-3450} python tools/oracle_golden.py rmat27 --out $O > $O/c5_golden.log 2>&1
echo "rc=$? elapsed=$(( $(date +%s) - start ))s" >> $O/c5_golden.log
kill $MON
echo done
