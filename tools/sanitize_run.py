"""Target for compute-sanitizer (memcheck / racecheck / initcheck): small full runs of the
GPU path through the C ABI — karate (C1), R-MAT 12, SBM 5k, co-occurrence 2k docs, with
the colouring heuristic and float weights once each — every result checked against the
oracle (test infrastructure).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
from paper_1805_10904_b200 import Louvain, inputs  # noqa: E402

cases = [("karate", inputs.karate(), {}),
         ("rmat12", inputs.rmat(12, 16, seed=7), {}),
         ("sbm5k", inputs.sbm(n=5000, blocks=50, avg_deg=16, seed=3), {}),
         ("cooc", inputs.cooc(topics=20, topic_size=100, docs=2000, seed=5), {}),
         ("rmat12_color", inputs.rmat(12, 16, seed=7), {"coloring": True})]
only = sys.argv[1:]
for name, r, kw in cases:
    if only and name not in only:
        continue
    with Louvain(r.n, r.src, r.dst, r.w, torch_allocator=False, **kw) as lv:
        lv.run()
        got = [lv.partition(l) for l in range(lv.num_levels)]
        q = lv.modularity(-1)
    want = oracle.run(oracle.Graph.from_edges(r.n, r.src, r.dst, r.w), **kw)
    ok = len(got) == len(want.levels) and all(np.array_equal(a, b) for a, b in zip(got, want.levels))
    print(f"{name}: levels={len(got)} Q={q:.10f} oracle_equal={ok}", flush=True)
    assert ok and q == want.final_q, name
print("sanitize_run ok")
