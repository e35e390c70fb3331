#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q > $O/r2au_pytest.log 2>&1; echo "rc=$?" >> $O/r2au_pytest.log
bash tools/variants.sh "cur:" "b6:LV_TAB_U2=96" "b7:LV_TAB_U2=160" "b9:LV_TAB_U2=544" "b10:LV_TAB_U2=1056" "cur2:" > $O/r2au_variants.txt 2>&1
LV_TAB_U2=288 python tools/profile_level.py --workload rmat24 --level 1 > $O/r2au_level1_b8.json 2>&1
python tools/profile_level.py --workload rmat24 --level 1 > $O/r2au_level1.json 2>&1
echo done
