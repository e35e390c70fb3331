#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_real.py tests/test_gpu_coloring.py tests/test_gpu_reorder.py -m "gpu and not slow" -x -q > $O/r2ac_pytest.log 2>&1; echo "rc=$?" >> $O/r2ac_pytest.log
timeout 600 python -m pytest tests/test_gpu_fullsize_golden.py -m gpu -x -q -k "c4 or c3_cooc_full_run_equals" > $O/r2ac_golden.log 2>&1; echo "rc=$?" >> $O/r2ac_golden.log
LV_SHARD_SIM=4 timeout 600 python tools/level_probe.py --workload rmat24 --runs 1 > $O/r2ac_sim4_rmat24.json 2>&1
echo done
