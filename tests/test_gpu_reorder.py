"""F3 — degree-class vertex relabel before the CSR build (louvain_config.reorder; SURVEY
F3).  The method then runs on the relabelled graph, so the oracle runs on the same
relabelled records (tests/reorder_ref.py, written from the header's definition): every
level, sweep count and Q must be equal; level-0 and final partitions are compared through
perm (the library returns them indexed by the original ids)."""
import numpy as np
import pytest

import oracle
from paper_1805_10904_b200 import Louvain, inputs
from reorder_ref import degree_perm, relabel
from test_gpu_parity import _random_records, _star_plus


def test_degree_perm_definition():
    # hand example: d = [3, 1, 0, 2, 1, 1] (records (0,1) (0,3) (0,3) (3,4)... see below)
    src = np.array([0, 0, 0, 3, 5, 2], np.int32)
    dst = np.array([1, 3, 3, 4, 5, 2], np.int32)  # (5,5) and (2,2) are loops
    perm, key = degree_perm(6, src, dst)
    # d = [3, 1, 0, 3, 1, 0] -> key = [30, 31, 32, 30, 31, 32]
    assert key.tolist() == [30, 31, 32, 30, 31, 32]
    assert perm.tolist() == [0, 2, 4, 1, 3, 5]
    r = inputs.rmat(12, 16, seed=3)
    perm, key = degree_perm(r.n, r.src, r.dst)
    assert np.array_equal(np.sort(perm), np.arange(r.n))
    inv = np.argsort(perm)
    assert np.all(np.diff(key[inv]) >= 0)
    same = np.diff(key[inv]) == 0
    assert np.all(np.diff(inv)[same] > 0)  # old ids ascending within a class


CASES = {
    "karate": lambda: inputs.karate(),
    "rmat12": lambda: inputs.rmat(12, 16, seed=4),
    "rmat14": lambda: inputs.rmat(14, 16, seed=9),
    "sbm": lambda: inputs.sbm(20_000, 20, 32, 0.3, seed=2),
    "cooc": lambda: inputs.cooc(topics=40, topic_size=500, docs=60_000, seed=3),
    "random_loops_dups": lambda: _random_records(1, 500, 4000),
    "star_plus": lambda: _star_plus(seed=2),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_reorder_full_run_equals_oracle_on_relabelled_graph(name):
    r = CASES[name]()
    perm, s2, d2 = relabel(r.n, r.src, r.dst)
    want = oracle.run(oracle.Graph.from_edges(r.n, s2, d2, r.w))
    with Louvain(r.n, r.src, r.dst, r.w, reorder=True) as g:
        g.run()
        assert g.num_levels == len(want.levels)
        assert [g.level_stats(l)[0] for l in range(g.num_levels)] == list(want.sweeps)
        lev0 = g.partition(0)
        assert np.array_equal(lev0, want.levels[0][perm]), name
        for l in range(1, g.num_levels):
            assert np.array_equal(g.partition(l), want.levels[l]), (name, l)
        assert np.array_equal(g.partition(-1), want.final[perm])
        assert g.modularity() == want.final_q


@pytest.mark.gpu
def test_reorder_device_inputs_and_identity_on_sorted_input():
    import torch

    r = inputs.rmat(13, 16, seed=5)
    perm, s2, d2 = relabel(r.n, r.src, r.dst)
    dev = torch.device("cuda", 0)
    args = [torch.from_numpy(r.src).to(dev), torch.from_numpy(r.dst).to(dev), torch.from_numpy(r.w).to(dev)]
    torch.cuda.synchronize()
    with Louvain(r.n, *args, reorder=True) as g:
        g.run()
        a = g.partition(-1)
    # the relabelled graph is already in degree-class order: relabelling it again is the
    # identity, so reorder on it equals the plain run on it
    perm2, _ = degree_perm(r.n, s2, d2)
    assert np.array_equal(perm2, np.arange(r.n))
    with Louvain(r.n, s2, d2, r.w) as g:
        g.run()
        b = g.partition(-1)
    assert np.array_equal(a, b[perm])
