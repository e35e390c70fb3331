"""Full-size stepwise parity: every compared step over the WHOLE graph, bit for bit, each
against the oracle's own implementation of that step (oracle/, never the CUDA path).

The full multi-level runs of C3, C4 and C5 are compared with the oracle's committed
golden results (tests/test_gpu_fullsize_golden.py).  This file checks the same runs step
by step, which localises a disagreement to one step and covers what a per-level hash
does not (the sweep-by-sweep Eq. 3 numerators, the contraction, every level's Q against
the oracle's own level graphs):

  * the CSR build: nnz, W, δ;
  * Algorithm 1's Jacobi sweeps along the GPU's own level-0 trajectory: the
    GPU runs sweeps 1..S through the step-level entry point louvain_sweep (the same
    pass as louvain_run), and at the sweeps in CHECK the oracle re-decides every vertex
    from the same snapshot (og_sweep) — labels, moved count and the exact Eq. 3
    numerators (I2, S2) of the snapshot must be equal;
  * the isolated-merge batch from the last swept state;
  * the GPU's full run (louvain_run): Q of every level equals the oracle's exact Eq. 3 on
    that level's graph (og_modularity), each level graph induced by the oracle from the
    GPU's partition of the level below (og_induce), the level-0 contraction
    itself equal to the oracle's (CSR, loops, δ'), and the final partition equal to the
    composition of the levels.
Not compared: the unchecked sweeps of the trajectory (GPU only) and the levels' sweep
counts (compared by the golden test).

C5 runs on the GPU box's host (196 GB): the oracle's C5 CSR alone is ~51 GB.
"""
import os

import numpy as np
import pytest

import oracle
from paper_1805_10904_b200 import Louvain, inputs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _canon(rp, col, w):
    row = np.repeat(np.arange(len(rp) - 1, dtype=np.int64), np.diff(rp))
    o = np.lexsort((col, row))
    return col[o], w[o]


def _stepwise(name, check, sweeps, threads=None, compare_contraction=True):
    import torch

    psutil = pytest.importorskip("psutil")
    need = {"rmat27": 150 << 30, "rmat24": 24 << 30}.get(name, 8 << 30)
    if psutil.virtual_memory().available < need:
        pytest.skip(f"{name}: needs ~{need >> 30} GB of free host memory")
    oracle.set_threads(threads or os.cpu_count() or 1)
    r = inputs.make(name)
    og = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    args = [torch.from_numpy(r.src).to(dev), torch.from_numpy(r.dst).to(dev),
            None if r.w is None else torch.from_numpy(r.w).to(dev)]
    torch.cuda.synchronize()
    n = r.n
    del r
    report = {}
    with Louvain(n, *args, stream=stream) as lv:
        del args
        torch.cuda.empty_cache()
        assert lv.nnz() == og.nnz
        # ---- level-0 sweeps along the GPU trajectory
        lab = np.arange(n, dtype=np.int32)
        checked = []
        for s in range(1, sweeps + 1):
            got, moved, i2, s2 = lv.sweep(lab, 0)
            if s in check:
                want, wmoved = og.sweep(lab, 0)
                assert np.array_equal(got, want), (name, s, np.nonzero(got != want)[0][:10])
                assert moved == wmoved, (name, s)
                m = og.modularity(lab)
                assert (i2, s2) == (m["I2"], m["S2"]), (name, s)
                checked.append(s)
            lab = got
        got, moved, _, _ = lv.sweep(lab, 1)
        want, wmoved = og.sweep(lab, 1)
        assert np.array_equal(got, want) and moved == wmoved, (name, "merge")
        report["sweeps_checked"] = checked
        # ---- the full run: every level's Q on the oracle's own level graphs
        lv.run()
        L = lv.num_levels
        parts = [lv.partition(l) for l in range(L)]
        qs = [lv.modularity(l) for l in range(L)]
        final = lv.partition(-1)
        g = og
        del og  # (C5: the level graphs are dropped as soon as the next one is built)
        for l in range(L):
            p = parts[l]
            assert len(p) == g.n
            k = int(p.max()) + 1
            assert np.array_equal(np.unique(p), np.arange(k))  # dense, order-preserving ids
            m = g.modularity(p)
            assert m["Q"] == qs[l], (name, l, m["Q"], qs[l])
            if l + 1 < L:
                h = g.induce(p, k)
                if l == 0 and compare_contraction:
                    a = lv.contract(p, k)
                    b = h.arrays()
                    assert np.array_equal(a["row_ptr"], b["row_ptr"])
                    assert np.array_equal(a["loop"], b["loop"])
                    assert np.array_equal(a["delta"], b["delta"])
                    ca, wa = _canon(a["row_ptr"], a["col"], a["w"])
                    assert np.array_equal(ca, b["col"]) and np.array_equal(wa, b["w"])
                    del a, b, ca, wa
                g = h
        comp = parts[0].copy()
        for l in range(1, L):
            comp = parts[l][comp]
        assert np.array_equal(comp, final)
        report["levels"] = [(len(p), int(p.max()) + 1, float(q)) for p, q in zip(parts, qs)]
    return report


def test_c5_rmat27_stepwise_equals_oracle():
    """C5 on one B200: sweeps 1-4, 25, 50 and 100 of level 0 (every vertex), the merge
    batch, the level-0 contraction and the exact Q of every level of the full run.
    ~25 min and ~150 GB of host memory: opt-in (LV_STEPWISE_C5=1); the full C5 run is
    compared with the oracle's golden in test_gpu_fullsize_golden.py."""
    if os.environ.get("LV_STEPWISE_C5") != "1":
        pytest.skip("opt-in: LV_STEPWISE_C5=1 (C5 is covered by the golden full-run test)")
    # the level-0 contraction's CSR is compared at C4 only: its host copies and the
    # canonicalising sort on top of the oracle's 51 GB CSR exceeded the box's 196 GB
    # (r2be: killed after 760 s); at C5 the levels' exact Q on the oracle's own induced
    # graphs covers the contraction
    rep = _stepwise("rmat27", check={1, 2, 3, 4, 25, 50, 100}, sweeps=100, compare_contraction=False)
    print(rep)


def test_c4_rmat24_stepwise_equals_oracle():
    """The same protocol on C4 (whose full run is also compared with the committed
    golden): validates the stepwise harness where the oracle's whole run is available."""
    rep = _stepwise("rmat24", check={1, 2, 3, 50, 100}, sweeps=100)
    print(rep)
