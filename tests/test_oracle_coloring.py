"""Pins of the oracle's colouring heuristic (reading D29) — CPU only.

Lu et al.'s distance-1 colouring heuristic (the "other heuristics" of P:L89 / P:L441):
vertices are coloured greedily in decreasing priority π(v) = fmix64(v ^ 0x9E37...),
and one sweep processes the colour classes in turn, each class deciding in parallel
against the state the previous class committed.  Pinned against: an independent
Python fmix64, networkx's greedy colouring with the same vertex order, colouring
validity, the rational brute-force decisions of tests/brute.py applied class by class,
and the textbook sequential (Gauss–Seidel) Louvain sweep on complete graphs, where every
vertex is its own class.
"""
import networkx as nx
import numpy as np
import pytest

import brute
import oracle
from paper_1805_10904_b200 import inputs

M64 = (1 << 64) - 1


def fmix64(v):
    k = (v ^ 0x9E3779B97F4A7C15) & M64
    k ^= k >> 33
    k = (k * 0xFF51AFD7ED558CCD) & M64
    k ^= k >> 33
    k = (k * 0xC4CEB9FE1A85EC53) & M64
    k ^= k >> 33
    return k


def test_priority_is_murmur3_fmix64():
    for v in [0, 1, 2, 33, 12345, 2**31 - 1]:
        assert oracle.color_priority(v) == fmix64(v)
    assert len({fmix64(v) for v in range(5000)}) == 5000  # distinct (a bijection)


def _records_graph(r):
    G = nx.Graph()
    G.add_nodes_from(range(r.n))
    G.add_edges_from((int(a), int(b)) for a, b in zip(r.src, r.dst) if a != b)
    return G


@pytest.mark.parametrize("name", ["karate", "rmat10", "ring", "cooc"])
def test_coloring_is_greedy_in_priority_order(name):
    r = {"karate": inputs.karate, "rmat10": lambda: inputs.rmat(10, 8, seed=3),
         "ring": lambda: inputs.ring_of_cliques(6, 5),
         "cooc": lambda: inputs.cooc(topics=10, topic_size=100, docs=3000, seed=3)}[name]()
    g = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w)
    colors, K = g.color()
    G = _records_graph(r)
    order = sorted(range(r.n), key=lambda v: -fmix64(v))
    want = nx.greedy_color(G, strategy=lambda G_, c_: iter(order))
    assert [want[v] for v in range(r.n)] == colors.tolist()
    assert K == max(want.values()) + 1
    for a, b in G.edges():  # a proper distance-1 colouring
        assert colors[a] != colors[b]
    assert K <= max(dict(G.degree()).values()) + 1


def _rand_graph(seed, n, p):
    rng = np.random.default_rng(seed)
    e = [(i, j, int(rng.integers(1, 5))) for i in range(n) for j in range(i + 1, n) if rng.random() < p]
    e += [(i, i, 2) for i in range(0, n, 5)]
    a = np.array(e, dtype=np.int64)
    return n, a[:, 0], a[:, 1], a[:, 2]


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
@pytest.mark.parametrize("cap", [0, 2, 3])
def test_colored_sweep_equals_brute_force_class_by_class(seed, cap):
    """Each class decides by exact Eq. 3 re-evaluation (brute.decide) against the labels
    the previous classes committed; colours >= cap-1 share the last class (D29)."""
    n, s, d, w = _rand_graph(seed, 11, 0.35)
    g = oracle.Graph.from_edges(n, s, d, w)
    bg = brute.G(n, s, d, w)
    colors, K = g.color()
    if cap and K > cap:
        colors, K = np.minimum(colors, cap - 1), cap
    rng = np.random.default_rng(seed)
    for start in (list(range(n)), [int(x) for x in rng.integers(0, n, n)], [int(x) for x in rng.integers(0, 3, n)]):
        got, moved = g.sweep_colored(np.array(start, np.int32), colors, K)
        lab = list(start)
        for c in range(K):
            lab = [brute.decide(bg, lab, i) if colors[i] == c else lab[i] for i in range(n)]
        assert got.tolist() == lab
        assert moved == sum(a != b for a, b in zip(start, lab))


def _sequential_sweep(bg, labels, order):
    """Textbook sequential Louvain sweep (Blondel et al.): vertices in `order`,
    each decision against the live state."""
    lab = list(labels)
    for i in order:
        lab[i] = brute.decide(bg, lab, i)
    return lab


@pytest.mark.parametrize("seed", [5, 6, 7])
def test_complete_graph_colored_sweep_is_the_sequential_sweep(seed):
    """On a complete graph every vertex gets its own colour, in decreasing priority order,
    so a coloured sweep is the sequential sweep in that order."""
    n = 9
    rng = np.random.default_rng(seed)
    e = [(i, j, int(rng.integers(1, 9))) for i in range(n) for j in range(i + 1, n)]
    a = np.array(e, dtype=np.int64)
    g = oracle.Graph.from_edges(n, a[:, 0], a[:, 1], a[:, 2])
    bg = brute.G(n, a[:, 0], a[:, 1], a[:, 2])
    colors, K = g.color()
    order = sorted(range(n), key=lambda v: -fmix64(v))
    assert K == n and [colors[v] for v in order] == list(range(n))
    lab = list(range(n))
    for _ in range(3):
        got, _ = g.sweep_colored(np.array(lab, np.int32), colors, K)
        lab = _sequential_sweep(bg, lab, order)
        assert got.tolist() == lab


def test_coloring_run_properties():
    """Full runs with colouring: Q of every level recomputed by exact Eq. 3 (brute), Q
    non-decreasing across levels, fewer sweeps than the Jacobi run on R-MAT (where the
    synchronous sweeps oscillate up to the cap), and the karate Q band."""
    r = inputs.rmat(10, 8, seed=5)
    g = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w)
    res = oracle.run(g, coloring=True)
    jac = oracle.run(g)
    assert sum(res.sweeps) < sum(jac.sweeps)
    assert all(b >= a for a, b in zip(res.q, res.q[1:]))
    bg = brute.G(r.n, r.src, r.dst, r.w)
    assert abs(float(brute.q_exact(bg, list(res.final))) - res.final_q) < 1e-12
    k = inputs.karate()
    kq = oracle.run(oracle.Graph.from_edges(k.n, k.src, k.dst), coloring=True).final_q
    assert 0.40 <= kq <= 0.42
