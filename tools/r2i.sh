#!/bin/bash
# Round-2 re-entry measurement: parity (not slow), smoke, bench (C4, default), per-kernel
# sweep times, launch list of the bench step, ncu --set full of the level-0 sweep kernels.
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $O/r2i_smi.txt 2>&1
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > $O/r2i_pytest.log 2>&1; echo "rc=$?" >> $O/r2i_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2i_smoke.log 2>&1; echo "rc=$?" >> $O/r2i_smoke.log
bash tools/variants.sh "cur:" > $O/r2i_variants.txt 2>&1
timeout 900 python bench.py > $O/r2i_bench.json 2> $O/r2i_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2i_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --coloring-steps 0 > $O/r2i_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"apply_moves|sweep_tab|sweep_thr|sweep_reg|agg_reg|hub_acc|hub_fin|hub_decide" -o $O/r2i_full -f env LV_PROFILE_RANGE=1 python tools/profile_sweep.py --workload rmat24 --warm 3 --reps 1 > $O/r2i_ncu.log 2>&1
echo done
