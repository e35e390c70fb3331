"""GPU parity of the colouring heuristic (reading D29) through the C ABI.

The Jones–Plassmann colouring (k_jp_round) must equal the oracle's sequential greedy
colouring in decreasing-priority order exactly, and full runs with colour-class sweeps
must reproduce the oracle's levels, sweep counts and Q exactly (integer weights: every
decision is a function of the input; the per-class ΔI2 bookkeeping is exact).
"""
import numpy as np
import pytest

import oracle
from paper_1805_10904_b200 import Louvain, LouvainError, inputs
from test_gpu_parity import _random_records, _star_plus

pytestmark = pytest.mark.gpu

GRAPHS = {
    "karate": lambda: inputs.karate(),
    "ring": lambda: inputs.ring_of_cliques(10, 6),
    "random_loops_dups": lambda: _random_records(1, 500, 4000),
    "rmat12": lambda: inputs.rmat(12, 16, seed=4),
    "sbm": lambda: inputs.sbm(20_000, 20, 32, 0.3, seed=2),
    "cooc": lambda: inputs.cooc(topics=40, topic_size=500, docs=60_000, seed=3),
    "star_plus": lambda: _star_plus(),
}


@pytest.mark.parametrize("name", list(GRAPHS))
def test_coloring_parity(name):
    r = GRAPHS[name]()
    want, K = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w).color()
    with Louvain(r.n, r.src, r.dst, r.w) as g:
        got, Kg = g.color()
    assert Kg == K
    assert np.array_equal(got, want)


@pytest.mark.parametrize("cap", [32, 0, 3])
@pytest.mark.parametrize("name", list(GRAPHS))
def test_colored_full_run_parity(name, cap):
    r = GRAPHS[name]()
    og = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w)
    # color_cap_min_n=0: cap every level, so the synchronous last class (k_delta_i2) runs
    want = oracle.run(og, coloring=True, color_classes=cap, color_cap_min_n=0)
    with Louvain(r.n, r.src, r.dst, r.w, coloring=True, color_classes=cap, color_cap_min_n=0) as g:
        g.run()
        assert g.num_levels == len(want.levels)
        for l in range(g.num_levels):
            assert np.array_equal(g.partition(l), want.levels[l]), (name, l)
            assert g.modularity(l) == want.q[l]
            assert g.level_stats(l)[0] == want.sweeps[l]
        assert np.array_equal(g.partition(-1), want.final)
        assert g.modularity(-1) == want.final_q
        assert g.level_colors(0)[0] >= 1


def test_colored_default_cap_threshold():
    """Default D29 cap: levels of <= 65536 vertices keep one class per colour."""
    r = inputs.sbm(20_000, 20, 32, 0.3, seed=2)
    want = oracle.run(oracle.Graph.from_edges(r.n, r.src, r.dst), coloring=True)
    with Louvain(r.n, r.src, r.dst, coloring=True) as g:
        g.run()
        assert [g.level_stats(l)[0] for l in range(g.num_levels)] == want.sweeps
        assert np.array_equal(g.partition(-1), want.final) and g.modularity(-1) == want.final_q


@pytest.mark.parametrize("stop_rule", [0, 1])
def test_colored_rmat16_and_real_weights(stop_rule):
    for r in (inputs.rmat(16, 16, seed=4),
              inputs.Records(4096, *(lambda x: (x.src, x.dst, inputs.real_weights(x.m, 3)))(inputs.rmat(12, 16, seed=6)))):
        og = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w if r.w.dtype.kind != "f" else r.w.astype(np.float64))
        want = oracle.run(og, coloring=True, stop_rule=stop_rule)
        with Louvain(r.n, r.src, r.dst, r.w, coloring=True, stop_rule=stop_rule) as g:
            g.run()
            assert [g.level_stats(l)[0] for l in range(g.num_levels)] == want.sweeps
            for l in range(g.num_levels):
                assert np.array_equal(g.partition(l), want.levels[l])
            assert g.modularity(-1) == want.final_q


def test_coloring_not_in_sharded_mode():
    r = inputs.karate()
    with pytest.raises(LouvainError, match="LV_EINVAL"):
        Louvain(r.n, r.src, r.dst, coloring=True, nccl_comm=1)


def test_colored_full_size_rmat24_properties():
    """C4 with colouring: the Q of the final partition against an independent exact numpy
    Eq. 3, fewer sweeps than the synchronous run (3 levels at the 100-sweep cap), higher Q, and
    bit-identical repeated runs."""
    r = inputs.rmat(24, 16, seed=4)
    with Louvain(r.n, r.src, r.dst, r.w, coloring=True) as g:
        csr = g.csr()
        g.run()
        final, q = g.partition(-1), g.modularity(-1)
        sweeps = [g.level_stats(l)[0] for l in range(g.num_levels)]
        g.run()
        assert np.array_equal(final, g.partition(-1)) and q == g.modularity(-1)
    assert sum(sweeps) < 300  # the synchronous run: 3 levels x the 100-sweep cap
    rp, col, w = csr["row_ptr"], csr["col"], csr["w"]
    row = np.repeat(np.arange(r.n), np.diff(rp))
    intra = int(w[final[row] == final[col]].sum(dtype=np.int64)) + 2 * int(csr["loop"].sum())
    deg = np.bincount(final, weights=csr["delta"].astype(np.float64), minlength=r.n)  # < 2^53: exact
    S2 = sum(int(x) * int(x) for x in deg[deg > 0].astype(np.int64))
    W = int(csr["W"])
    assert abs((2 * W * intra - S2) / (4 * W * W) - q) <= 1e-12
    assert q > 0.0459  # the synchronous run's final Q at C4 (profiles/r1b_bench_rmat24.json)
