#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q > $O/r2ap_pytest.log 2>&1; echo "rc=$?" >> $O/r2ap_pytest.log
bash tools/variants.sh "base:LV_SO=paper_1805_10904_b200/csrc/liblouvain_base.so" "cur:" "c3:LV_SO=paper_1805_10904_b200/csrc/liblouvain_c3.so" "base2:LV_SO=paper_1805_10904_b200/csrc/liblouvain_base.so" "cur2:" > $O/r2ap_variants.txt 2>&1
python tools/profile_level.py --workload rmat24 --level 1 > $O/r2ap_level1.json 2>&1
echo done
