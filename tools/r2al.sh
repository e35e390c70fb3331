#!/bin/bash
O=gpurun_out; mkdir -p $O
LV_TAB_NODEG=544 timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q > $O/r2al_pytest.log 2>&1; echo "rc=$?" >> $O/r2al_pytest.log
bash tools/variants.sh "cur:" "nd9:LV_TAB_NODEG=512" "nd5:LV_TAB_NODEG=32" "cur2:" "nd9b:LV_TAB_NODEG=512" > $O/r2al_variants.txt 2>&1
echo done
