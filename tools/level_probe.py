"""Per-level breakdown of one full run: level sizes, sweeps and phase times (ms).

    python tools/level_probe.py --workload rmat24
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1805_10904_b200 import Louvain, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="rmat24")
ap.add_argument("--runs", type=int, default=2)
args = ap.parse_args()
r = inputs.make(args.workload)
lv = Louvain(r.n, r.src, r.dst, r.w)
for _ in range(args.runs):
    lv.run()
out = []
for l in range(lv.num_levels):
    sw, t = lv.level_stats(l)
    out.append(dict(level=l, n=lv.level_size(l), sweeps=sw, **{k: round(v, 2) for k, v in t.items()}))
print(json.dumps(dict(workload=args.workload, q=lv.modularity(), levels=out, run=lv.run_stats())), flush=True)
lv.close()
