"""C-ABI boundary checks that need no GPU: the library builds for sm_100a, loads, and
exports every function include/louvain.h declares; the binding raises (never falls
back) when the device is unavailable."""
import os
import re
import subprocess

import pytest

from paper_1805_10904_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "louvain.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(louvain_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    build.build_louvain()
    return _lib.load()


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == names


def test_sm100a_only(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.SO_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    assert "sm_90" not in out.stdout and "sm_80" not in out.stdout


def test_config_default(lib):
    import ctypes as C

    cfg = _lib.Config()
    assert lib.louvain_config_default(C.byref(cfg)) == 0
    assert cfg.theta == 1e-6 and cfg.big_theta == 1e-6
    assert cfg.max_sweeps == 100 and cfg.max_levels == 64
    assert cfg.stop_rule == 0 and cfg.merge_isolated == 1


def test_invalid_arguments_rejected_without_gpu(lib):
    import ctypes as C

    h = C.c_void_p()
    assert lib.louvain_create(None, None, C.byref(h)) == _lib.LV_EINVAL
    g = _lib.Graph()
    g.n = 0
    assert lib.louvain_create(C.byref(g), None, C.byref(h)) == _lib.LV_EINVAL
    assert not h.value
    assert lib.louvain_run(None) == _lib.LV_EINVAL


def test_no_cpu_fallback():
    """Without a device the product path raises; it never computes on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1805_10904_b200 import Louvain, LouvainError, inputs

    r = inputs.karate()
    with pytest.raises(LouvainError):
        Louvain(r.n, r.src, r.dst).run()


def test_package_does_not_import_oracle():
    """The product package never imports the oracle (test infrastructure only)."""
    pkg = os.path.join(ROOT, "paper_1805_10904_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".c", ".h")):
                src = open(os.path.join(dp, f), errors="ignore").read()
                assert "import oracle" not in src and "from oracle" not in src and "oracle.h" not in src, f
