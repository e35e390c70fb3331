#!/bin/bash
# Bench lines for the other BASELINE configs (C2 sbm, C3 cooc, C5 rmat27 on one GPU).
TAG=${1:-r1}
mkdir -p gpurun_out
for w in sbm cooc; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err
done
timeout 1500 python bench.py --workload rmat27 --steps 1 --warmup 1 --e2e-steps 1 --coloring-steps 0 > gpurun_out/${TAG}_bench_rmat27.json 2> gpurun_out/${TAG}_bench_rmat27.err
echo done
