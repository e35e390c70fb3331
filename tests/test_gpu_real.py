"""GPU parity of the real-weight mode (reading D28) through the C ABI.

Real weights (float32 / float64, as the paper stores them) are mapped to the
fixed point w~ = rint(w·2^s) on both sides independently (oracle.c vs the CUDA
k_fx_sum / k_fx_conv), then the integer method runs, so the bar stays exact equality:
the scale s, the CSR, every level's labels, sweep counts and Q.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_1805_10904_b200 import Louvain, LouvainError, inputs

pytestmark = pytest.mark.gpu


def _with_real(r, seed, dtype, sigma=1.0):
    return inputs.Records(r.n, r.src, r.dst, inputs.real_weights(r.m, seed, sigma=sigma, dtype=dtype),
                          name=r.name + f"+lognormal({sigma},{np.dtype(dtype).name})")


GRAPHS = {
    "karate_f32": lambda: _with_real(inputs.karate(), 1, np.float32),
    "rmat12_f32": lambda: _with_real(inputs.rmat(12, 16, seed=4), 2, np.float32),
    "rmat14_f64": lambda: _with_real(inputs.rmat(14, 16, seed=4), 3, np.float64, sigma=2.0),
    "sbm_f32": lambda: _with_real(inputs.sbm(20_000, 20, 32, 0.3, seed=2), 4, np.float32, sigma=0.5),
    "cooc_f64": lambda: _with_real(inputs.cooc(topics=40, topic_size=500, docs=60_000, seed=3), 5, np.float64),
    "rmat12_intvalued_f64": lambda: inputs.Records(4096, *(lambda r: (r.src, r.dst, r.w.astype(np.float64)))(
        inputs.rmat(12, 16, seed=4)), name="rmat12 integer-valued f64"),
}


@pytest.mark.parametrize("name", list(GRAPHS))
def test_real_weight_full_run_parity(name):
    r = GRAPHS[name]()
    og = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w.astype(np.float64))
    want = oracle.run(og)
    with Louvain(r.n, r.src, r.dst, r.w) as g:
        assert g.weight_scale == og.scale
        c, a = g.csr(), og.arrays()
        assert c["W"] == a["W"]
        assert np.array_equal(c["delta"], a["delta"]) and np.array_equal(c["loop"], a["loop"])
        g.run()
        assert g.num_levels == len(want.levels)
        for l in range(g.num_levels):
            assert np.array_equal(g.partition(l), want.levels[l]), (name, l)
            assert g.modularity(l) == want.q[l]
            assert g.level_stats(l)[0] == want.sweeps[l]
        assert np.array_equal(g.partition(-1), want.final)
        assert g.modularity(-1) == want.final_q


def test_real_weights_from_device_tensors():
    r = _with_real(inputs.rmat(12, 16, seed=7), 8, np.float32)
    want = oracle.run(oracle.Graph.from_edges(r.n, r.src, r.dst, r.w.astype(np.float64)))
    dev = torch.device("cuda", 0)
    with Louvain(r.n, torch.from_numpy(r.src).to(dev), torch.from_numpy(r.dst).to(dev),
                 torch.from_numpy(r.w).to(dev)) as g:
        g.run()
        assert np.array_equal(g.partition(-1), want.final)
        assert g.modularity(-1) == want.final_q


@pytest.mark.parametrize("bad", [0.0, -2.0, float("nan"), float("inf")])
def test_real_weight_errors(bad):
    w = np.array([1.0, bad, 2.0], dtype=np.float64)
    with pytest.raises(LouvainError, match="LV_EGRAPH"):
        Louvain(4, np.array([0, 1, 2], np.int32), np.array([1, 2, 3], np.int32), w)
    with pytest.raises(LouvainError, match="LV_EGRAPH"):  # dynamic range beyond 52 bits
        Louvain(3, np.array([0, 1], np.int32), np.array([1, 2], np.int32), np.array([1e-20, 1e20]))


def test_full_size_c3_real_weights_properties():
    """C3 shape (5M vertices, ~200M edges) with float32 weights: the oracle's scale and W
    from the same records (its quantisation is a linear pass), Q against an exact numpy
    Eq. 3 on the fixed-point CSR, and bit-identical repeated runs."""
    r = inputs.make("cooc")
    w = inputs.real_weights(r.m, 9, sigma=1.0, dtype=np.float32)
    wd = w.astype(np.float64)
    with Louvain(r.n, r.src, r.dst, w) as g:
        s = g.weight_scale
        assert oracle.fixed_sum(wd, s) <= 1 << 52 < oracle.fixed_sum(wd, s + 1)
        c = g.csr()
        assert c["W"] == oracle.fixed_sum(wd, s)
        g.run()
        final, q = g.partition(-1), g.modularity(-1)
        g.run()
        assert np.array_equal(final, g.partition(-1)) and q == g.modularity(-1)
    rp, col, ww, loop = c["row_ptr"], c["col"], c["w"], c["loop"]
    row = np.repeat(np.arange(r.n), np.diff(rp))
    intra = int(ww[final[row] == final[col]].sum(dtype=np.int64)) + 2 * int(loop.sum())
    dsum = np.zeros(r.n, dtype=object)
    np.add.at(dsum, final, c["delta"].astype(object))
    W = int(c["W"])
    num = 2 * W * intra - int(sum(int(x) * int(x) for x in dsum if x))
    assert abs(num / (4 * W * W) - q) <= 1e-12
    assert q > 0.3
