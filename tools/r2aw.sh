#!/bin/bash
O=gpurun_out; mkdir -p $O
LV_TAB_U1=2032 timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q > $O/r2aw_pytest.log 2>&1; echo "rc=$?" >> $O/r2aw_pytest.log
bash tools/variants.sh "cur:" "u1all:LV_TAB_U1=2032" "u1_4:LV_TAB_U1=16" "u1_5:LV_TAB_U1=32" "u1_7:LV_TAB_U1=128" "u1_9:LV_TAB_U1=512" "u1_10:LV_TAB_U1=1024" "cur2:" > $O/r2aw_variants.txt 2>&1
LV_TAB_U1=256 python tools/profile_level.py --workload rmat24 --level 1 > $O/r2aw_level1_u1b8.json 2>&1
echo done
