"""Build the in-tree shared libraries.

* ``csrc/liblouvain.so`` — the product: CUDA sources compiled for sm_100a only
  (``-gencode arch=compute_100a,code=sm_100a``), C ABI declared in include/louvain.h.
* ``inputs/liblvgen.so`` — seeded input generators (gcc, OpenMP).

nvcc cross-compiles without a GPU, so this runs on the CPU dev box.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(CSRC, "liblouvain.so")
SOURCES = ["lv_api.cu"]
# every header in csrc/ is a dependency (a header edited alone must rebuild the .so)
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_louvain(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "louvain.h"), __file__]
    if not force and not _stale(SO, deps):
        return SO
    tmp = SO + f".tmp{os.getpid()}"
    cmd = [NVCC, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           "-o", tmp, *[os.path.join(CSRC, s) for s in SOURCES], "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, SO)
    return SO


def build_all(force: bool = False, verbose: bool = False) -> None:
    from . import inputs

    inputs.build(force)
    build_louvain(force, verbose)


if __name__ == "__main__":
    sys.path.insert(0, ROOT)
    from paper_1805_10904_b200 import build as b

    b.build_all(force="--force" in sys.argv, verbose=True)
    print(SO)
