O=gpurun_out; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"apply_moves|sweep_tab|agg_reg|hub_acc|hub_fin" -o $O/r2h_full -f env LV_PROFILE_RANGE=1 python tools/profile_sweep.py --workload rmat24 --warm 3 --reps 1 > $O/r2h_ncu.log 2>&1
echo done
