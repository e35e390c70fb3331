#!/bin/bash
O=gpurun_out; mkdir -p $O; rm -f $O/*.ncu-rep
LV_TAB_B3=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q > $O/r2bd_pytest.log 2>&1; echo "rc=$?" >> $O/r2bd_pytest.log
bash tools/variants.sh "cur:" "t3:LV_TAB_B3=1" "cur2:" "t3b:LV_TAB_B3=1" > $O/r2bd_variants.txt 2>&1
echo done
