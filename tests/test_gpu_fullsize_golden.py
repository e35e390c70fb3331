"""Full-size parity: the whole multi-level run on the GPU against the oracle's committed
golden results (tests/golden/<config>.json, written by tools/oracle_golden.py, which calls
only oracle/ and the seeded generators).

The north_star's agreement criterion: per-level label arrays bit-identical
(compared here by SHA-256 of the dense int32 arrays), Q per level bit-identical (hex
float), the same sweep counts, and the same final composed partition.  The run is
Algorithm 2 around Algorithm 1 with the default
configuration, launched exactly as bench.py launches it (device-resident records on a
dedicated stream).
"""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_1805_10904_b200 import Louvain, inputs

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i4").tobytes()).hexdigest()


def _gold(name):
    p = os.path.join(GOLD, f"{name}.json")
    if not os.path.exists(p):
        pytest.skip(f"tests/golden/{name}.json not committed (tools/oracle_golden.py {name})")
    return json.load(open(p))


def _compare(name, device_inputs=True):
    import torch

    gold = _gold(name)
    r = inputs.make(name)
    assert (r.n, r.m) == (gold["n"], gold["records"])
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    if device_inputs:
        args = [torch.from_numpy(r.src).to(dev), torch.from_numpy(r.dst).to(dev),
                None if r.w is None else torch.from_numpy(r.w).to(dev)]
        torch.cuda.synchronize()
    else:
        args = [r.src, r.dst, r.w]
    del r
    with Louvain(gold["n"], *args, stream=stream) as lv:
        assert lv.nnz() == gold["nnz"]
        lv.run()
        got = []
        for l in range(lv.num_levels):
            lab = lv.partition(l)
            got.append(dict(n=int(len(lab)), k=int(lab.max()) + 1 if len(lab) else 0,
                            sweeps=int(lv.level_stats(l)[0]), q_hex=float(lv.modularity(l)).hex(),
                            labels_sha256=_sha(lab)))
        final = lv.partition(-1)
        fq = lv.modularity(-1)
    want = [{k: L[k] for k in ("n", "k", "sweeps", "q_hex", "labels_sha256")} for L in gold["levels"]]
    assert len(got) == len(want)
    for l, (g, w) in enumerate(zip(got, want)):
        assert g == w, f"level {l}: {g} != {w}"
    assert _sha(final) == gold["final_sha256"]
    assert float(fq).hex() == gold["final_q_hex"]


@pytest.mark.gpu
def test_c4_rmat24_full_run_equals_oracle():
    """C4 (R-MAT scale 24, 520.8M directed entries, the bench workload): every level."""
    _compare("rmat24")


@pytest.mark.gpu
def test_c3_cooc_full_run_equals_oracle():
    """C3 (5M-vertex Collaboration-Spotting-shaped co-occurrence graph): every level."""
    _compare("cooc")


@pytest.mark.gpu
def test_c3_cooc_full_run_host_inputs_equals_oracle():
    """C3 again through the e2e path (host records copied by louvain_create)."""
    _compare("cooc", device_inputs=False)


@pytest.mark.gpu
@pytest.mark.slow
def test_c5_rmat27_full_run_equals_oracle():
    """C5 (R-MAT scale 27, 4.2G directed entries > 2^31: int64 offsets) on one B200,
    every level compared by SHA-256.  Host memory: ~40 GB of records."""
    psutil = pytest.importorskip("psutil")
    if psutil.virtual_memory().available < 64 << 30:
        pytest.skip("C5 records need more host memory than this machine has free")
    _compare("rmat27")
