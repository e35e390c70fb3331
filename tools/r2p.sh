#!/bin/bash
O=gpurun_out; mkdir -p $O
for w in sbm cooc; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --coloring-steps 0 --reorder-steps 0 > $O/r2p_bench_${w}_pool.json 2>&1
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --coloring-steps 0 --reorder-steps 0 --torch-allocator > $O/r2p_bench_${w}_torch.json 2>&1
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --coloring-steps 0 --reorder-steps 0 > $O/r2p_bench_rmat24_pool.json 2>&1
echo done
