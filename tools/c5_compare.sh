#!/bin/bash
# C5 GPU full run vs the committed oracle golden (tests/golden/rmat27.json), then
# compute-sanitizer memcheck / racecheck / synccheck of small full runs.
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_fullsize_golden.py -m slow -x -q > $O/c5_pytest.log 2>&1; echo "rc=$?" >> $O/c5_pytest.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py > $O/sanitize_$tool.log 2>&1
  echo "rc=$?" >> $O/sanitize_$tool.log
done
echo done
