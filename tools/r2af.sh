#!/bin/bash
# two-pass bucketed raw fill vs the atomic scatter (LV_FILL_ONEPASS=1)
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_real.py -m "gpu and not slow" -x -q > $O/r2af_pytest.log 2>&1; echo "rc=$?" >> $O/r2af_pytest.log
timeout 600 python -m pytest tests/test_gpu_fullsize_golden.py -m gpu -x -q -k "c4 or c3_cooc_full_run_equals" > $O/r2af_golden.log 2>&1; echo "rc=$?" >> $O/r2af_golden.log
for v in two one; do
  if [ $v = one ]; then export LV_FILL_ONEPASS=1; else unset LV_FILL_ONEPASS; fi
  timeout 300 python tools/time_create.py > $O/r2af_create_$v.txt 2>&1
done
unset LV_FILL_ONEPASS
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --coloring-steps 0 --reorder-steps 0 --e2e-steps 1 > $O/r2af_bench.json 2>&1
echo done
