#!/bin/bash
O=gpurun_out; mkdir -p $O
python tools/profile_level.py --workload rmat24 --level 1 > $O/r2t_level1.json 2>&1
python tools/profile_level.py --workload rmat24 --level 2 > $O/r2t_level2.json 2>&1
echo done
