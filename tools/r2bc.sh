#!/bin/bash
O=gpurun_out; mkdir -p $O; rm -f $O/*.ncu-rep
for v in cur au4 au2; do
  if [ $v = cur ]; then unset LV_SO; else export LV_SO=paper_1805_10904_b200/csrc/liblouvain_$v.so; fi
  python tools/level_probe.py --workload rmat24 --runs 2 > $O/r2bc_levels_$v.json 2>&1
  timeout 300 python tools/time_create.py > $O/r2bc_create_$v.txt 2>&1
done
unset LV_SO
python tools/level_probe.py --workload rmat24 --runs 2 > $O/r2bc_levels_cur2.json 2>&1
echo done
