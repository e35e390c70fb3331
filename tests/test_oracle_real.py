"""Pins of the oracle's real-weight mode (reading D28) — CPU only.

The paper stores float weights.  Reading D28 maps them to fixed-point integers
ω~ = rint(ω·2^s), s the largest integer with Σ ω~ <= 2^52, and runs the integer method.
These pins check the mapping against exact rational arithmetic (Python Fractions,
independent of oracle.c), and the integration against properties the mathematics fixes:
modularity is invariant under a common scaling of all weights (Eq. 3 is homogeneous of
degree 0 in ω), so integer-valued and power-of-two-scaled weights must reproduce the
integer run exactly.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_1805_10904_b200 import inputs

LIM = 1 << 52


def _T_exact(w, s):
    """Σ round-half-even(ω·2^s) with exact rationals (Python's round() on a Fraction
    rounds half to even)."""
    sc = Fraction(2) ** s
    return sum(round(Fraction(float(x)) * sc) for x in w)


def _graph(seed, n=40, p=0.15):
    rng = np.random.default_rng(seed)
    iu = np.triu_indices(n, 1)
    keep = rng.random(iu[0].size) < p
    src, dst = iu[0][keep].astype(np.int32), iu[1][keep].astype(np.int32)
    loops = np.arange(0, n, 7, dtype=np.int32)
    return n, np.concatenate([src, loops]), np.concatenate([dst, loops])


@pytest.mark.parametrize("case", ["lognormal", "tiny", "huge", "dyadic", "ties"])
def test_scale_is_the_largest_s_with_sum_at_most_2_52(case):
    """D28: s = max{s : Σ rint(ω·2^s) <= 2^52}; W of the built graph = T(s)."""
    n, src, dst = _graph(1)
    m = len(src)
    if case == "lognormal":
        w = inputs.real_weights(m, seed=11, sigma=2.0, dtype=np.float64)
    elif case == "tiny":
        w = inputs.real_weights(m, seed=12).astype(np.float64) * 1e-200
    elif case == "huge":
        w = inputs.real_weights(m, seed=13).astype(np.float64) * 1e250
    elif case == "dyadic":
        w = np.arange(1, m + 1, dtype=np.float64) / 8.0
    else:  # many exact .5 ties after scaling: rounding half to even decides them
        w = np.full(m, 0.75) + np.arange(m) % 3
    g = oracle.Graph.from_edges(n, src, dst, w)
    s = g.scale
    assert _T_exact(w, s) <= LIM < _T_exact(w, s + 1)
    assert g.W == _T_exact(w, s)
    assert oracle.fixed_sum(w, s) == _T_exact(w, s)
    # each stored weight is the exact rational rounding of its record (loops in loop[])
    sc = Fraction(2) ** s
    a = g.arrays()
    want = {}
    for u, v, x in zip(src, dst, w):
        q = round(Fraction(float(x)) * sc)
        if u == v:
            assert a["loop"][u] >= q
            continue
        want[(u, v)] = want.get((u, v), 0) + q
        want[(v, u)] = want.get((v, u), 0) + q
    got = {}
    for i in range(n):
        for k in range(a["row_ptr"][i], a["row_ptr"][i + 1]):
            got[(i, int(a["col"][k]))] = int(a["w"][k])
    assert got == want


def test_half_even_rounding_at_the_scale():
    """Ties go to even (D28 rint), checked against exact rationals at and around s."""
    w = np.array([0.5, 1.5, 2.5, 3.5] * 4, dtype=np.float64)
    src = np.arange(16, dtype=np.int32)
    dst = (src + 1) % 16
    s = oracle.Graph.from_edges(16, src, dst, w).scale
    for t in (s - 1, s, s + 1):
        assert oracle.fixed_sum(w, t) == _T_exact(w, t)
    assert oracle.fixed_sum(w[:4], 0) == 0 + 2 + 2 + 4  # rint(.5)=0, rint(1.5)=2, rint(2.5)=2, rint(3.5)=4


def _levels(res):
    return [np.asarray(x) for x in res.levels]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_integer_valued_floats_reproduce_the_integer_run(seed):
    """Eq. 3 is homogeneous of degree 0 in ω: ω·2^s gives the same decisions (every score
    scales by 2^2s) and the same partitions at every level as the integer graph."""
    r = inputs.rmat(scale=9, edge_factor=8, seed=seed)
    gi = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w)
    gf = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w.astype(np.float64))
    assert gf.W == gi.W * 2 ** gf.scale
    ri, rf = oracle.run(gi), oracle.run(gf)
    assert len(ri.levels) == len(rf.levels)
    for a, b in zip(_levels(ri), _levels(rf)):
        assert np.array_equal(a, b)
    assert np.array_equal(ri.final, rf.final)
    assert abs(ri.final_q - rf.final_q) <= 1e-15


@pytest.mark.parametrize("k", [-9, 3])
def test_power_of_two_rescaling_gives_the_same_fixed_point_graph(k):
    n, src, dst = _graph(4)
    w = inputs.real_weights(len(src), seed=5, dtype=np.float64)
    a = oracle.Graph.from_edges(n, src, dst, w)
    b = oracle.Graph.from_edges(n, src, dst, w * 2.0 ** k)
    assert b.scale == a.scale - k
    for key, x in a.arrays().items():
        assert np.array_equal(x, b.arrays()[key]), key


def test_real_q_matches_the_float_graph():
    """The fixed-point graph's Q (Eq. 3) is within m·2^-s-relative of the real-weight Q of
    the same partition (brute-force exact rationals on the original ω)."""
    n, src, dst = _graph(6, n=60, p=0.1)
    w = inputs.real_weights(len(src), seed=7, sigma=1.5, dtype=np.float64)
    g = oracle.Graph.from_edges(n, src, dst, w)
    res = oracle.run(g)
    lab = np.asarray(res.final)
    # exact Eq. 3 on the real weights: Q = Σ_C [in_C / W − (deg_C / 2W)^2]
    W = sum(Fraction(float(x)) for x in w)
    inC, deg = {}, {}
    for u, v, x in zip(src, dst, w):
        x = Fraction(float(x))
        deg[lab[u]] = deg.get(lab[u], 0) + x
        deg[lab[v]] = deg.get(lab[v], 0) + x
        if lab[u] == lab[v]:
            inC[lab[u]] = inC.get(lab[u], 0) + x
    Q = sum(inC.values()) / W - sum(d * d for d in deg.values()) / (4 * W * W)
    assert abs(float(Q) - res.final_q) <= 1e-12
    assert res.final_q > 0.3


@pytest.mark.parametrize("bad", [0.0, -1.0, float("nan"), float("inf")])
def test_real_weight_errors(bad):
    w = np.array([1.0, bad, 2.0])
    with pytest.raises(oracle.OracleError):
        oracle.Graph.from_edges(4, [0, 1, 2], [1, 2, 3], w)


def test_dynamic_range_beyond_52_bits_is_an_error():
    """ω~ = 0 for the smallest weight once the largest fills the 52-bit budget."""
    with pytest.raises(oracle.OracleError):
        oracle.Graph.from_edges(3, [0, 1], [1, 2], np.array([1e-20, 1e20]))
