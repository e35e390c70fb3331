"""Per-kernel sweep times (CUDA events) of a HIGHER level's graph: run the workload once,
contract level l-1's partition (louvain_contract), feed the contracted graph back as
records (u < v entries + loops), and time its sweeps from singletons like level l's.

    python tools/profile_level.py --workload rmat24 --level 1
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1805_10904_b200 import Louvain, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="rmat24")
ap.add_argument("--level", type=int, default=1)
ap.add_argument("--warm", type=int, default=3)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
r = inputs.make(args.workload)
n, src, dst, w = r.n, r.src, r.dst, r.w
for lev in range(args.level):
    with Louvain(n, src, dst, w) as lv:
        lv.run()
        p = lv.partition(0)
        k = int(p.max()) + 1
        g = lv.contract(p, k)
    rp, col, wt, loop = g["row_ptr"], g["col"], g["w"], g["loop"]
    row = np.repeat(np.arange(k, dtype=np.int64), np.diff(rp))
    keep = row < col
    lp = np.nonzero(loop)[0]
    src = np.concatenate([row[keep], lp]).astype(np.int32)
    dst = np.concatenate([col[keep], lp]).astype(np.int32)
    w = np.concatenate([wt[keep], loop[lp]]).astype(np.int64)
    n = k
with Louvain(n, src, dst, w) as lv:
    out = lv.time_sweeps(args.warm, args.reps)
out["graph"] = dict(level=args.level, n=n, records=len(src))
print(json.dumps(out), flush=True)
