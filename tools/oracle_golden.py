"""Write full-size golden results of the CPU oracle (tests/golden/<config>.json).

Calls only ``oracle/`` and the seeded input generators (``paper_1805_10904_b200.inputs``,
the one module both sides share; it holds no method arithmetic).  Nothing here touches
the CUDA path, so the stored values are the oracle's: the full multi-level run of
Algorithm 2 around Algorithm 1 with the DESIGN.md
readings, default configuration (alg1_abs, θ = Θ = 1e-6, 100 sweeps, merge on).

Per level: vertices n, communities k, sweeps, Q (hex float, bit-exact) and the SHA-256 of
the dense int32 label array (little-endian bytes); also the SHA-256 and Q of the final
composed partition, the per-sweep trace (moved, Q hex) and the oracle's CSR summary.

    python tools/oracle_golden.py cooc rmat24            # dev box (8 cores, 62 GB)
    python tools/oracle_golden.py rmat27 --out gpurun_out # GPU box host (196 GB)
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1805_10904_b200 import inputs  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i4").tobytes()).hexdigest()


def golden(name: str, threads: int) -> dict:
    oracle.set_threads(threads)
    t0 = time.time()
    r = inputs.make(name)
    t_gen = time.time() - t0
    n, m, recipe = r.n, r.m, r.name
    t0 = time.time()
    g = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w)
    t_build = time.time() - t0
    del r  # the COO is not needed any more (C5 memory)
    t0 = time.time()
    res = oracle.run(g)
    t_run = time.time() - t0
    levels = []
    for l, lab in enumerate(res.levels):
        mv, qs = res.traces[l]
        levels.append(dict(
            n=int(len(lab)), k=int(lab.max()) + 1 if len(lab) else 0, sweeps=int(res.sweeps[l]),
            q=float(res.q[l]), q_hex=float(res.q[l]).hex(), labels_sha256=sha(lab),
            trace_moved=[int(x) for x in mv], trace_q_hex=[float(x).hex() for x in qs]))
    return dict(
        config=name, recipe=recipe, n=int(n), records=int(m), nnz=int(g.nnz), W=int(g.W),
        levels=levels, final_sha256=sha(res.final), final_q=float(res.final_q),
        final_q_hex=float(res.final_q).hex(), edge_visits=int(res.edge_visits),
        oracle=dict(threads=oracle.get_threads(), cpu=os.cpu_count(), gen_s=round(t_gen, 1),
                    build_s=round(t_build, 1), run_s=round(t_run, 1)),
        generated_by="tools/oracle_golden.py (oracle/ + paper_1805_10904_b200.inputs only)",
        settings=dict(stop_rule="alg1_abs", theta=1e-6, big_theta=1e-6, max_sweeps=100, merge_isolated=True))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    for name in a.configs:
        d = golden(name, a.threads)
        path = os.path.join(a.out, f"{name}.json")
        with open(path, "w") as f:
            json.dump(d, f, indent=1)
        print(name, json.dumps({k: d[k] for k in ("n", "nnz", "W", "final_q", "edge_visits", "oracle")}),
              [(L["n"], L["k"], L["sweeps"]) for L in d["levels"]], flush=True)


if __name__ == "__main__":
    main()
