#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_real.py tests/test_gpu_sharded.py -m "gpu and not slow" -x -q > $O/r2ax_pytest.log 2>&1; echo "rc=$?" >> $O/r2ax_pytest.log
timeout 600 python -m pytest tests/test_gpu_fullsize_golden.py -m gpu -x -q -k "c4 or c3_cooc_full_run_equals" > $O/r2ax_golden.log 2>&1; echo "rc=$?" >> $O/r2ax_golden.log
bash tools/variants.sh "old:LV_TAB_U2=32 LV_TAB_U1=0" "cur:" "old2:LV_TAB_U2=32 LV_TAB_U1=0" "cur2:" > $O/r2ax_variants.txt 2>&1
python tools/level_probe.py --workload rmat24 --runs 2 > $O/r2ax_levels.json 2>&1
LV_TAB_U2=32 LV_TAB_U1=0 python tools/level_probe.py --workload rmat24 --runs 2 > $O/r2ax_levels_old.json 2>&1
echo done
