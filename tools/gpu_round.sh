#!/bin/bash
# One GPU pass: parity tests, smoke, bench line, launch list of one bench step,
# and one `ncu --set full` capture of the level-0 sweep kernels of C4.
# Usage (from the repo root, on the B200 box): bash tools/gpu_round.sh TAG
TAG=${1:-r1}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/${TAG}_launches.csv python bench.py --steps 1 --warmup 0 --e2e-steps 0 --coloring-steps 0 --no-cpu-baseline > $O/${TAG}_ncu_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
    --profile-from-start off -o $O/${TAG}_sweep_full -f \
    env LV_PROFILE_RANGE=1 python tools/profile_sweep.py --workload rmat24 --warm 3 --reps 1 > $O/${TAG}_ncu_full.log 2>&1
ncu -i $O/${TAG}_sweep_full.ncu-rep --page raw --csv > $O/${TAG}_sweep_full_raw.csv 2>/dev/null
echo done
