#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 1500 python bench.py --workload rmat27 --steps 2 --warmup 3 --coloring-steps 0 --reorder-steps 0 --e2e-steps 1 > $O/r2ag_bench_rmat27.json 2> $O/r2ag_bench_rmat27.err
timeout 600 python bench.py --workload sbm --steps 10 --warmup 3 --coloring-steps 1 --reorder-steps 1 > $O/r2ag_bench_sbm.json 2> $O/r2ag_bench_sbm.err
timeout 900 python bench.py --workload cooc --steps 5 --warmup 3 --coloring-steps 1 --reorder-steps 1 > $O/r2ag_bench_cooc.json 2> $O/r2ag_bench_cooc.err
echo done
