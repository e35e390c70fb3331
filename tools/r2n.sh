#!/bin/bash
# batched-insert tab kernel + F3: parity, C5 full-run golden, sweep variants, stepwise C4,
# compute-sanitizer
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_reorder.py tests/test_gpu_parity.py -m "gpu and not slow" -x -q > $O/r2n_pytest.log 2>&1; echo "rc=$?" >> $O/r2n_pytest.log
timeout 1200 python -m pytest tests/test_gpu_fullsize_golden.py -m "gpu" -x -q > $O/r2n_golden.log 2>&1; echo "rc=$?" >> $O/r2n_golden.log
bash tools/variants.sh "base:LV_SO=paper_1805_10904_b200/csrc/liblouvain_base.so" "cur:" "u8big:LV_TAB_U8=1536" "u8all:LV_TAB_U8=2032" "fullcap:LV_TAB_FULLCAP=1" > $O/r2n_variants.txt 2>&1
python tools/profile_sweep.py --warm 3 --reps 5 --reorder > $O/var_reorder.json 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize_stepwise.py -m "gpu and slow" -x -q -k c4 -s > $O/r2n_stepwise_c4.log 2>&1; echo "rc=$?" >> $O/r2n_stepwise_c4.log
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py > $O/sanitize_$tool.log 2>&1
  echo "rc=$?" >> $O/sanitize_$tool.log
done
echo done
