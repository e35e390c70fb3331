#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m "gpu and not slow" -x -q > $O/r2l_pytest.log 2>&1; echo "rc=$?" >> $O/r2l_pytest.log
bash tools/variants.sh "cur:LV_HUBCL=0" "l2m3:LV_HUBCL=0 LV_L2MODE=3" "l2m5:LV_HUBCL=0 LV_L2MODE=5" "l2m7:LV_HUBCL=0 LV_L2MODE=7" > $O/r2l_variants.txt 2>&1
echo done
