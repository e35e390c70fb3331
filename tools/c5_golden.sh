#!/bin/bash
# C5 (R-MAT scale 27) golden on the GPU box's host (196 GB RAM, 16 cores): the oracle's
# full run (tools/oracle_golden.py: oracle/ + seeded generators only), then the GPU's
# full run compared level by level (tests/test_gpu_fullsize_golden.py, slow).
# Afterwards compute-sanitizer memcheck / racecheck / synccheck of small full runs.
O=gpurun_out; mkdir -p $O
free -g > $O/c5_mem.txt; nproc >> $O/c5_mem.txt; lscpu | grep "Model name" >> $O/c5_mem.txt
( while true; do free -g | sed -n 2p >> $O/c5_mem_trace.txt; sleep 60; done ) &
MON=$!
/usr/bin/time -v timeout ${ORACLE_TIMEOUT:-7800} python tools/oracle_golden.py rmat27 --out tests/golden > $O/c5_golden.log 2>&1
kill $MON
cp tests/golden/rmat27.json $O/ 2>/dev/null
timeout 1200 python -m pytest tests/test_gpu_fullsize_golden.py -m slow -x -q > $O/c5_pytest.log 2>&1; echo "rc=$?" >> $O/c5_pytest.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py > $O/sanitize_$tool.log 2>&1
  echo "rc=$?" >> $O/sanitize_$tool.log
done
echo done
