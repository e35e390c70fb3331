"""Sweep-sharded path on one GPU.

The partition (edge-balanced vertex ranges, per-range bins, exact counter combination,
replicated move application, the CSR build and the contraction computed in row parts —
SURVEY F4) runs with P virtual ranks in one process (LV_SHARD_SIM=P);
the NCCL exchange runs over a real world-1 NCCL communicator.  Jacobi semantics make the
result independent of the rank count, so every configuration must equal the oracle.
"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_1805_10904_b200 import Louvain, _lib, inputs

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

CODE = """
import numpy as np, oracle
from test_gpu_parity import _star_plus, _canon_fast
from paper_1805_10904_b200 import Louvain, inputs
for r in (inputs.karate(), inputs.rmat(14, 16, seed=3), _star_plus(seed=1), inputs.sbm(20000, 20, 32, 0.3, seed=2)):
    og = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w)
    # the CSR built in row parts (sharded build) and the level-0 contraction in community
    # parts equal the oracle's
    b = og.arrays()
    with Louvain(r.n, r.src, r.dst, r.w) as g:
        a = g.csr()
        assert a["W"] == b["W"] and np.array_equal(a["row_ptr"], b["row_ptr"]), r.name
        assert np.array_equal(a["loop"], b["loop"]) and np.array_equal(a["delta"], b["delta"]), r.name
        ca, wa = _canon_fast(a["row_ptr"], a["col"], a["w"])
        assert np.array_equal(ca, b["col"]) and np.array_equal(wa, b["w"]), r.name
    for rule in (0, 1):
        want = oracle.run(og, stop_rule=rule)
        with Louvain(r.n, r.src, r.dst, r.w, stop_rule=rule) as g:
            g.run()
            assert [g.level_stats(l)[0] for l in range(g.num_levels)] == want.sweeps, r.name
            for l in range(g.num_levels):
                assert np.array_equal(g.partition(l), want.levels[l]), (r.name, l)
            assert g.modularity() == want.final_q
print('ok')
"""


@pytest.mark.parametrize("P", [2, 3, 7])
def test_simulated_ranks_match_oracle(P):
    env = dict(os.environ, LV_SHARD_SIM=str(P),
               PYTHONPATH=os.pathsep.join([HERE, os.path.dirname(HERE), os.environ.get("PYTHONPATH", "")]))
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


def test_nccl_world1_matches_oracle():
    lib = _lib.load()
    uid = (C.c_uint8 * 128)()
    assert lib.louvain_nccl_unique_id(uid) == 0
    comm = C.c_void_p()
    assert lib.louvain_nccl_init(uid, 1, 0, 0, C.byref(comm)) == 0
    try:
        for r in (inputs.rmat(13, 16, seed=5), inputs.karate()):
            og = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w)
            want = oracle.run(og)
            with Louvain(r.n, r.src, r.dst, r.w, nccl_comm=comm.value, rank=0, world=1) as g:
                g.run()
                assert [g.level_stats(l)[0] for l in range(g.num_levels)] == want.sweeps
                assert np.array_equal(g.partition(-1), want.final)
                assert g.modularity() == want.final_q
    finally:
        lib.louvain_nccl_destroy(comm)


@pytest.mark.parametrize("cs", ["16", "8"])
def test_cluster_hub_path_matches_oracle(cs):
    """The opt-in thread-block-cluster hub kernel (lv_hubcl.cuh, LV_HUBCL=1): hub rows'
    e_{i->C} tables sharded over the cluster's shared memory — same decisions as the
    oracle (_star_plus has a 20k-entry hub row, R-MAT 14 several)."""
    env = dict(os.environ, LV_HUBCL="1", LV_HUBCL_CS=cs,
               PYTHONPATH=os.pathsep.join([HERE, os.path.dirname(HERE), os.environ.get("PYTHONPATH", "")]))
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
