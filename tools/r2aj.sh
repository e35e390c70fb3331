#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_coloring.py -m "gpu and not slow" -x -q > $O/r2aj_pytest.log 2>&1; echo "rc=$?" >> $O/r2aj_pytest.log
timeout 600 python -m pytest tests/test_gpu_fullsize_golden.py -m gpu -x -q -k "c4 or c3_cooc_full_run_equals" > $O/r2aj_golden.log 2>&1; echo "rc=$?" >> $O/r2aj_golden.log
python tools/level_probe.py --workload rmat24 --runs 2 > $O/r2aj_rmat24.json 2>&1
LV_CONC_NNZ=0 python tools/level_probe.py --workload rmat24 --runs 2 > $O/r2aj_rmat24_off.json 2>&1
timeout 300 python bench.py --workload sbm --steps 10 --warmup 3 --no-cpu-baseline --coloring-steps 0 --reorder-steps 0 > $O/r2aj_sbm.json 2>&1
LV_CONC_NNZ=0 timeout 300 python bench.py --workload sbm --steps 10 --warmup 3 --no-cpu-baseline --coloring-steps 0 --reorder-steps 0 > $O/r2aj_sbm_off.json 2>&1
echo done
