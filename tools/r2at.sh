#!/bin/bash
O=gpurun_out; mkdir -p $O
LV_TAB_U2=48 timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q > $O/r2at_pytest.log 2>&1; echo "rc=$?" >> $O/r2at_pytest.log
bash tools/variants.sh "cur:" "u2_128:LV_TAB_U2=16" "u2_256:LV_TAB_U2=32" "cur2:" "u2_128b:LV_TAB_U2=16" > $O/r2at_variants.txt 2>&1
echo done
