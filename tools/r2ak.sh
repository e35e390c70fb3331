#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m "gpu and not slow" -x -q > $O/r2ak_pytest.log 2>&1; echo "rc=$?" >> $O/r2ak_pytest.log
bash tools/variants.sh "base:LV_SO=paper_1805_10904_b200/csrc/liblouvain_base.so" "cur:" "base2:LV_SO=paper_1805_10904_b200/csrc/liblouvain_base.so" "cur2:" > $O/r2ak_variants.txt 2>&1
echo done
