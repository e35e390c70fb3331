#!/bin/bash
O=gpurun_out; mkdir -p $O
LV_TAB_HALF=56 timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q > $O/r2ae_pytest_half.log 2>&1; echo "rc=$?" >> $O/r2ae_pytest_half.log
bash tools/variants.sh "base:LV_SO=paper_1805_10904_b200/csrc/liblouvain_base.so" "cur:" "h16:LV_TAB_HALF=16" "h8:LV_TAB_HALF=8" "h32:LV_TAB_HALF=32" "h56:LV_TAB_HALF=56" > $O/r2ae_variants.txt 2>&1
echo done
