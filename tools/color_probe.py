"""Timing probe of the colouring heuristic (D29) on a workload (not a bench value)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1805_10904_b200 import Louvain, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="rmat24")
ap.add_argument("--caps", default="32,0,16,64")
args = ap.parse_args()
r = inputs.make(args.workload)
dev = torch.device("cuda", 0)
s = torch.cuda.Stream(dev)
torch.cuda.set_stream(s)
src, dst = torch.from_numpy(r.src).to(dev), torch.from_numpy(r.dst).to(dev)
w = None if r.w is None else torch.from_numpy(r.w).to(dev)
for cap in [int(x) for x in args.caps.split(",")]:
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with Louvain(r.n, src, dst, w, stream=s, coloring=cap >= 0, color_classes=max(cap, 0)) as g:
            g.run()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            info = dict(cap=cap, s=round(dt, 4), q=g.modularity(-1),
                        sweeps=[g.level_stats(l)[0] for l in range(g.num_levels)],
                        colors=[g.level_colors(l) for l in range(g.num_levels)],
                        phases=[{k: round(v, 1) for k, v in g.level_stats(l)[1].items()} for l in range(g.num_levels)])
    print(json.dumps(info), flush=True)
