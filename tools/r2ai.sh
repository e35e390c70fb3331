#!/bin/bash
O=gpurun_out; mkdir -p $O
python tools/level_probe.py --workload rmat24 --runs 2 > $O/r2ai_default.json 2>&1
LV_CONCURRENT=1 python tools/level_probe.py --workload rmat24 --runs 2 > $O/r2ai_conc.json 2>&1
python tools/level_probe.py --workload rmat24 --runs 2 > $O/r2ai_default2.json 2>&1
LV_CONCURRENT=1 python tools/level_probe.py --workload rmat24 --runs 2 > $O/r2ai_conc2.json 2>&1
echo done
