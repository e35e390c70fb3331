"""Target for ncu: build a workload's graph, run `warm` sweeps, then `reps` more.

    ncu --set full --clock-control none --import-source on \
        -k regex:"k_agg_smem|k_hub" -s <skip> -c <count> -o gpurun_out/prof \
        python tools/profile_sweep.py --workload rmat24 --warm 3 --reps 1

Prints the time_sweeps JSON (CUDA-event timing; not a bench value when under ncu).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1805_10904_b200 import Louvain, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="rmat24")
ap.add_argument("--warm", type=int, default=3)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--reorder", action="store_true", help="F3 degree-class relabel (louvain_config.reorder)")
args = ap.parse_args()
r = inputs.make(args.workload)
lv = Louvain(r.n, r.src, r.dst, r.w, reorder=args.reorder)
print(json.dumps(lv.time_sweeps(args.warm, args.reps)), flush=True)
lv.close()
