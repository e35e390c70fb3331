#!/bin/bash
# cluster hub kernel: parity + sweep timing variants
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q > $O/r2j_pytest.log 2>&1; echo "rc=$?" >> $O/r2j_pytest.log
bash tools/variants.sh "pool:LV_HUBCL=0" "cl16:" "cl8:LV_HUBCL_CS=8" > $O/r2j_variants.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize_golden.py -m "gpu and not slow" -x -q -k c4 > $O/r2j_golden.log 2>&1; echo "rc=$?" >> $O/r2j_golden.log
echo done
