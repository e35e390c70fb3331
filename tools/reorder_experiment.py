"""Locality experiment: C4 with ids relabeled by descending degree vs the generator's
random permutation (different graph labels -> different results; timing only)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1805_10904_b200 import Louvain, inputs
r = inputs.rmat(24, 16, seed=4)
deg = np.bincount(r.src, minlength=r.n) + np.bincount(r.dst, minlength=r.n)
order = np.argsort(-deg, kind="stable")
rank = np.empty(r.n, np.int32); rank[order] = np.arange(r.n, dtype=np.int32)
for name, s, d in (("random_ids", r.src, r.dst), ("degree_sorted_ids", rank[r.src], rank[r.dst])):
    lv = Louvain(r.n, s, d, r.w)
    t = lv.time_sweeps(3, 3)
    print(json.dumps({"ids": name, "ms_sweep": t["ms_sweep"], "kernels": [(k["name"], round(k["ms"], 2)) for k in t["kernels"]]}), flush=True)
    lv.close()
