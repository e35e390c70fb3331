"""Whole-run per-kernel profile (cfg.profile: CUDA events per kernel on its launching
stream) plus the per-level phase times of one full run.

    python tools/run_profile.py --workload rmat24
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1805_10904_b200 import Louvain, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="rmat24")
args = ap.parse_args()
r = inputs.make(args.workload)
with Louvain(r.n, r.src, r.dst, r.w) as lv:
    lv.run()
with Louvain(r.n, r.src, r.dst, r.w, profile=True) as lv:
    lv.run()
    levels = []
    for l in range(lv.num_levels):
        sw, t = lv.level_stats(l)
        levels.append(dict(level=l, n=lv.level_size(l), sweeps=sw, **{k: round(v, 2) for k, v in t.items()}))
    prof = lv.profile()
print(json.dumps(dict(workload=args.workload, levels=levels, profile=prof)), flush=True)
