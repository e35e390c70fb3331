#!/bin/bash
O=gpurun_out; mkdir -p $O
TA=1 python tools/steps_probe.py sbm > $O/r2r_sbm_torch.txt 2>&1
timeout 300 python bench.py --workload sbm --steps 10 --warmup 3 --no-cpu-baseline --coloring-steps 0 --reorder-steps 0 > $O/r2r_bench_sbm.json 2>&1
BENCH_CLOCK_MS=1000 timeout 300 python bench.py --workload sbm --steps 10 --warmup 3 --no-cpu-baseline --coloring-steps 0 --reorder-steps 0 > $O/r2r_bench_sbm_clk1000.json 2>&1
timeout 300 python bench.py --workload cooc --steps 5 --warmup 3 --no-cpu-baseline --coloring-steps 0 --reorder-steps 0 > $O/r2r_bench_cooc.json 2>&1
echo done
