#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_real.py -m "gpu and not slow" -x -q > $O/r2s_pytest.log 2>&1; echo "rc=$?" >> $O/r2s_pytest.log
bash tools/variants.sh "base:LV_SO=paper_1805_10904_b200/csrc/liblouvain_base.so" "cur:" > $O/r2s_variants.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --coloring-steps 0 --reorder-steps 0 --e2e-steps 1 > $O/r2s_bench.json 2>&1
echo done
