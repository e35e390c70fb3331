#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_real.py tests/test_gpu_coloring.py -m "gpu and not slow" -x -q > $O/r2ar_pytest.log 2>&1; echo "rc=$?" >> $O/r2ar_pytest.log
timeout 600 python -m pytest tests/test_gpu_fullsize_golden.py -m gpu -x -q -k "c4 or c3_cooc_full_run_equals" > $O/r2ar_golden.log 2>&1; echo "rc=$?" >> $O/r2ar_golden.log
bash tools/variants.sh "base:LV_SO=paper_1805_10904_b200/csrc/liblouvain_base.so" "cur:" "base2:LV_SO=paper_1805_10904_b200/csrc/liblouvain_base.so" "cur2:" > $O/r2ar_variants.txt 2>&1
python tools/profile_level.py --workload rmat24 --level 1 > $O/r2ar_level1.json 2>&1
echo done
