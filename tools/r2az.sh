#!/bin/bash
# round-2 final measurement: GPU tests, smoke, bench (all legs), reference arm, launch list
# of one bench step, ncu --set full of a level-0 sweep
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $O/r2az_smi.txt 2>&1
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > $O/r2az_pytest.log 2>&1; echo "rc=$?" >> $O/r2az_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2az_smoke.log 2>&1; echo "rc=$?" >> $O/r2az_smoke.log
timeout 1200 python bench.py > $O/r2az_bench.json 2> $O/r2az_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/r2az_bench_reference.json 2> $O/r2az_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2az_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --coloring-steps 0 --reorder-steps 0 > $O/r2az_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"sweep_tab|hub_acc|hub_fin" -o $O/r2az_full -f env LV_PROFILE_RANGE=1 python tools/profile_sweep.py --workload rmat24 --warm 3 --reps 1 > $O/r2az_ncu.log 2>&1
python tools/profile_sweep.py --workload rmat24 --warm 3 --reps 1 > $O/r2az_sweep_alg_bytes.json 2>&1
echo done
