#!/bin/bash
O=gpurun_out; mkdir -p $O
python tools/run_profile.py --workload rmat24 > $O/r2o_profile_rmat24.json 2>&1
python tools/run_profile.py --workload sbm > $O/r2o_profile_sbm.json 2>&1
python tools/run_profile.py --workload cooc > $O/r2o_profile_cooc.json 2>&1
timeout 300 python bench.py --workload sbm --steps 5 --warmup 3 --no-cpu-baseline --coloring-steps 0 --reorder-steps 0 > $O/r2o_bench_sbm.json 2>&1
timeout 600 python bench.py --workload cooc --steps 3 --warmup 3 --no-cpu-baseline --coloring-steps 0 --reorder-steps 0 > $O/r2o_bench_cooc.json 2>&1
echo done
