"""Seeded synthetic inputs and text loaders (binding over ``lvgen.c``).

Inputs only — none of the method's arithmetic lives here.  Both the CUDA path's
callers (tests, bench.py) and the oracle's tests draw their graphs from this module,
which is the one piece of code the two sides share.

Workload recipes:
  C1 karate        : Zachary's 78 unit edges (networkx order).
  C2 sbm           : n=1,000,000, 1000 blocks, avg degree 32, mu=0.3, seed 2.
  C3 cooc          : 5000 topics x 1000 entities, 17.5M documents, Zipf(2.0) sizes
                     capped at 40, p_in 0.8, popularity exponent 1.1, seed 3.
  C4 rmat24        : scale 24, edge factor 16, (0.57,0.19,0.19), weights U{1..16}, seed 4.
  C5 rmat27        : scale 27, same parameters, seed 5.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(os.path.dirname(_HERE))
_SRC = os.path.join(_HERE, "lvgen.c")
_SO = os.path.join(_HERE, "liblvgen.so")
_HDR = os.path.join(_ROOT, "include", "lvgen.h")

GCC_FLAGS = ["-O3", "-std=c11", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(_HDR)
    ):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *GCC_FLAGS, "-I", os.path.join(_ROOT, "include"), "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def _L():
    global _lib
    if _lib is None:
        lib = C.CDLL(build())
        P, i64, i32, dbl, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_uint64
        lib.lvgen_karate.argtypes = [P, P]
        lib.lvgen_ring_of_cliques_m.argtypes = [i32, i32]
        lib.lvgen_ring_of_cliques_m.restype = i64
        lib.lvgen_ring_of_cliques.argtypes = [i32, i32, P, P]
        lib.lvgen_sbm.argtypes = [i64, i64, i64, dbl, u64, P, P, P]
        lib.lvgen_cooc_count.argtypes = [i64, i64, i64, dbl, i32, dbl, dbl, u64]
        lib.lvgen_cooc_count.restype = i64
        lib.lvgen_cooc_fill.argtypes = [i64, i64, i64, dbl, i32, dbl, dbl, u64, P, P]
        lib.lvgen_rmat.argtypes = [i32, i64, dbl, dbl, dbl, i32, u64, P, P, P]
        lib.lvgen_permutation.argtypes = [i64, u64, C.c_uint32, P]
        lib.lvgen_philox.argtypes = [C.c_uint32] * 6 + [P]
        lib.lvgen_set_threads.argtypes = [i32]
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class Records:
    """Undirected COO records on vertices [0,n).  ``w is None`` = unweighted (1)."""

    n: int
    src: np.ndarray
    dst: np.ndarray
    w: np.ndarray | None = None
    truth: np.ndarray | None = None
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.src.shape[0])


def philox(k0, k1, c0, c1, c2, c3):
    out = np.zeros(4, dtype=np.uint32)
    _L().lvgen_philox(k0, k1, c0, c1, c2, c3, _p(out))
    return out


def permutation(n, seed, stream=0):
    out = np.empty(n, dtype=np.int32)
    _L().lvgen_permutation(n, seed, stream, _p(out))
    return out


def karate() -> Records:
    s, d = np.empty(78, np.int32), np.empty(78, np.int32)
    _L().lvgen_karate(_p(s), _p(d))
    return Records(34, s, d, None, name="karate")


def ring_of_cliques(k: int, c: int) -> Records:
    m = _L().lvgen_ring_of_cliques_m(k, c)
    if m < 0:
        raise ValueError("ring_of_cliques needs k>=3, c>=3")
    s, d = np.empty(m, np.int32), np.empty(m, np.int32)
    _L().lvgen_ring_of_cliques(k, c, _p(s), _p(d))
    return Records(k * c, s, d, None, truth=np.repeat(np.arange(k, dtype=np.int32), c),
                   name=f"ring_of_cliques({k},{c})")


def sbm(n=1_000_000, blocks=1000, avg_deg=32, mu=0.3, seed=2) -> Records:
    m = n * avg_deg // 2
    s, d, t = np.empty(m, np.int32), np.empty(m, np.int32), np.empty(n, np.int32)
    if _L().lvgen_sbm(n, blocks, avg_deg, mu, seed, _p(s), _p(d), _p(t)):
        raise ValueError("bad sbm arguments")
    return Records(n, s, d, None, truth=t, name=f"sbm(n={n},blocks={blocks},deg={avg_deg},mu={mu})",
                   meta=dict(n=n, blocks=blocks, avg_deg=avg_deg, mu=mu, seed=seed))


def cooc(topics=5000, topic_size=1000, docs=17_500_000, zipf_s=2.0, max_size=40, p_in=0.8,
         pop_exp=1.1, seed=3) -> Records:
    args = (topics, topic_size, docs, zipf_s, max_size, p_in, pop_exp, seed)
    m = _L().lvgen_cooc_count(*args)
    if m < 0:
        raise ValueError("bad cooc arguments")
    s, d = np.empty(m, np.int32), np.empty(m, np.int32)
    if _L().lvgen_cooc_fill(*args, _p(s), _p(d)):
        raise RuntimeError("cooc fill failed")
    return Records(topics * topic_size, s, d, None, name=f"cooc(n={topics * topic_size},docs={docs})",
                   meta=dict(topics=topics, topic_size=topic_size, docs=docs, seed=seed))


def rmat(scale=24, edge_factor=16, a=0.57, b=0.19, c=0.19, wmax=16, seed=4) -> Records:
    n = 1 << scale
    m = edge_factor * n
    s, d = np.empty(m, np.int32), np.empty(m, np.int32)
    w = np.empty(m, np.int32) if wmax > 0 else None
    if _L().lvgen_rmat(scale, edge_factor, a, b, c, wmax, seed, _p(s), _p(d), _p(w)):
        raise ValueError("bad rmat arguments")
    return Records(n, s, d, w, name=f"rmat(scale={scale},ef={edge_factor})",
                   meta=dict(scale=scale, edge_factor=edge_factor, wmax=wmax, seed=seed))


def real_weights(m: int, seed: int, sigma: float = 1.0, dtype=np.float32) -> np.ndarray:
    """Seeded positive real weights (lognormal(0, sigma), numpy's counter-based Philox
    bit generator) for the float-weight mode (the paper stores float
    weights).  Input data only: no method arithmetic."""
    g = np.random.Generator(np.random.Philox(key=int(seed)))
    return g.lognormal(0.0, float(sigma), int(m)).astype(dtype)


# The five BASELINE.json configurations (and the small analogues used by parity tests).
CONFIGS = {
    "karate": lambda: karate(),
    "sbm": lambda: sbm(),
    "cooc": lambda: cooc(),
    "rmat24": lambda: rmat(24, 16, seed=4),
    "rmat27": lambda: rmat(27, 16, seed=5),
}


def make(name: str) -> Records:
    return CONFIGS[name]()


# ------------------------------------------------------------------ text loaders
def _densify(u, v):
    ids, inv = np.unique(np.concatenate([u, v]), return_inverse=True)
    inv = inv.astype(np.int32)
    return len(ids), inv[: len(u)], inv[len(u):], ids


def _weights_out(wa: np.ndarray):
    """None when every weight is 1, int64 when all are integral, else float64 (the
    real-weight mode of reading D28 maps them to exact fixed point in the library)."""
    if not np.all(np.isfinite(wa)) or np.any(wa <= 0):
        raise ValueError("weights must be finite and > 0 (P:L43)")
    if np.all(wa == 1):
        return None
    wi = wa.astype(np.int64)
    if np.all(wi == wa):
        return wi
    return wa.astype(np.float64)


def parse_edge_list(text: str, default_weight=1):
    """Edge list: ``src dst [w]`` per line; ``#``/``%`` comments.

    Returns (Records, original_ids).  Ids are densified (sorted order); weights must be
    finite and > 0 — integral weights come back as int64 (exact integer path), others as
    float64 (fixed-point real-weight path, reading D28), all-ones as None."""
    us, vs, ws = [], [], []
    for ln, line in enumerate(text.splitlines(), 1):
        t = line.strip()
        if not t or t[0] in "#%":
            continue
        f = t.split()
        if len(f) < 2 or len(f) > 3:
            raise ValueError(f"line {ln}: expected 2 or 3 fields")
        try:
            u, v = int(f[0]), int(f[1])
            w = float(f[2]) if len(f) == 3 else float(default_weight)
        except ValueError as e:
            raise ValueError(f"line {ln}: {e}") from None
        if u < 0 or v < 0:
            raise ValueError(f"line {ln}: negative id")
        if not (w > 0) or not np.isfinite(w):
            raise ValueError(f"line {ln}: weight must be finite and > 0")
        us.append(u); vs.append(v); ws.append(w)
    if not us:
        raise ValueError("no edges")
    n, su, sv, ids = _densify(np.array(us, np.int64), np.array(vs, np.int64))
    return Records(n, su, sv, _weights_out(np.array(ws, np.float64)), name="edgelist"), ids


def parse_matrix_market(text: str):
    """MatrixMarket coordinate (pattern|integer|real, symmetric|general).

    Ids are 1-based in the file and kept (n = max(rows, cols)); weights as in
    parse_edge_list.  'general' files may list (i,j) and (j,i): the library sums
    duplicate undirected pairs (reading D25)."""
    lines = text.splitlines()
    if not lines or not lines[0].startswith("%%MatrixMarket"):
        raise ValueError("missing MatrixMarket header")
    h = lines[0].lower().split()
    if len(h) < 5 or h[1] != "matrix" or h[2] != "coordinate" or h[3] not in ("pattern", "integer", "real") \
            or h[4] not in ("symmetric", "general"):
        raise ValueError("unsupported MatrixMarket format")
    body = [ln for ln in lines[1:] if ln.strip() and not ln.startswith("%")]
    if not body:
        raise ValueError("missing size line")
    nr, nc, nz = (int(x) for x in body[0].split()[:3])
    if len(body) - 1 < nz:
        raise ValueError(f"expected {nz} entries, found {len(body) - 1}")
    us, vs, ws = [], [], []
    for ln in body[1:1 + nz]:
        f = ln.split()
        i, j = int(f[0]) - 1, int(f[1]) - 1
        if not (0 <= i < nr and 0 <= j < nc):
            raise ValueError(f"entry ({i + 1},{j + 1}) outside {nr}x{nc}")
        us.append(i); vs.append(j)
        ws.append(1.0 if h[3] == "pattern" else float(f[2]))
    n = max(nr, nc)
    return Records(n, np.array(us, np.int32), np.array(vs, np.int32), _weights_out(np.array(ws, np.float64)),
                   name="matrixmarket")
