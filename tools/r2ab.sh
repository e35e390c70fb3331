#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_real.py -m "gpu and not slow" -x -q > $O/r2ab_pytest.log 2>&1; echo "rc=$?" >> $O/r2ab_pytest.log
bash tools/variants.sh "old:LV_HUB_ACC_OLD=1" "new:" "old2:LV_HUB_ACC_OLD=1" "new2:" > $O/r2ab_variants.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize_golden.py -m gpu -x -q -k "c4" > $O/r2ab_golden.log 2>&1; echo "rc=$?" >> $O/r2ab_golden.log
echo done
