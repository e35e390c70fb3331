"""Text loaders of the input subsystem: edge lists and MatrixMarket,
integer / real / pattern weights, comments, densification and the error cases.  The
parsed records feed the oracle here (CPU); the same records feed the library in the
GPU tests."""
import numpy as np
import pytest

import oracle
from paper_1805_10904_b200 import inputs

EDGES = """# a comment
% another
10 20
20 30 2
30 10
40 40 3
"""


def test_edge_list_densify_and_weights():
    r, ids = inputs.parse_edge_list(EDGES)
    assert ids.tolist() == [10, 20, 30, 40] and r.n == 4
    assert r.src.tolist() == [0, 1, 2, 3] and r.dst.tolist() == [1, 2, 0, 3]
    assert r.w.dtype == np.int64 and r.w.tolist() == [1, 2, 1, 3]
    g = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w)
    assert g.W == 7 and g.arrays()["loop"].tolist() == [0, 0, 0, 3]


def test_edge_list_unweighted_and_real():
    r, _ = inputs.parse_edge_list("0 1\n1 2\n")
    assert r.w is None
    r, _ = inputs.parse_edge_list("0 1 0.5\n1 2 1.25\n")
    assert r.w.dtype == np.float64 and r.w.tolist() == [0.5, 1.25]
    g = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w)  # real weights: reading D28
    assert g.scale is not None and g.W == int(1.75 * 2 ** g.scale)


@pytest.mark.parametrize("bad", ["0 1 0\n", "0 1 -2\n", "0 1 inf\n", "0\n", "0 1 2 3\n", "-1 2\n", "a b\n", "#\n"])
def test_edge_list_errors(bad):
    with pytest.raises(ValueError):
        inputs.parse_edge_list(bad)


MM_INT = """%%MatrixMarket matrix coordinate integer symmetric
% comment
3 3 3
1 2 4
2 3 1
3 3 2
"""


def test_matrix_market_integer_symmetric():
    r = inputs.parse_matrix_market(MM_INT)
    assert r.n == 3 and r.src.tolist() == [0, 1, 2] and r.dst.tolist() == [1, 2, 2]
    assert r.w.tolist() == [4, 1, 2]
    g = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w)
    assert g.W == 7 and g.arrays()["delta"].tolist() == [4, 5, 5]


def test_matrix_market_pattern_general_duplicates_sum():
    txt = "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n2 1\n"
    r = inputs.parse_matrix_market(txt)
    assert r.w is None
    g = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w)
    a = g.arrays()
    assert g.W == 2 and a["w"].tolist() == [2, 2]  # (1,2) and (2,1): one undirected pair, summed (D25)


def test_matrix_market_real():
    txt = "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 0.25\n"
    r = inputs.parse_matrix_market(txt)
    assert r.w.dtype == np.float64 and r.w.tolist() == [0.25]


@pytest.mark.parametrize("bad", ["", "%%MatrixMarket matrix array real general\n1 1\n1\n",
                                 "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 2 1\n",
                                 "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n3 1 1\n",
                                 "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 0\n"])
def test_matrix_market_errors(bad):
    with pytest.raises(ValueError):
        inputs.parse_matrix_market(bad)
