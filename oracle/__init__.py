"""CPU oracle for the GPU Louvain hot path of arXiv 1805.10904 — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg
and ``--impl reference``) may import this package.  The product package
``paper_1805_10904_b200`` never imports it, and the two share no code.

This module is a thin ctypes binding over ``oracle.c`` (plain single-threaded C that
follows the paper step by step; see the header of ``oracle.c`` for the citations).
All numerics live in the C file; this file only marshals numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

GCC_FLAGS = ["-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (no FMA contraction, no fast-math; reading D22)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *GCC_FLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class _Graph(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("nnz", C.c_int64),
        ("row_ptr", C.POINTER(C.c_int64)),
        ("col", C.POINTER(C.c_int32)),
        ("w", C.POINTER(C.c_int64)),
        ("loop", C.POINTER(C.c_int64)),
        ("delta", C.POINTER(C.c_int64)),
        ("W", C.c_int64),
    ]


class _Config(C.Structure):
    _fields_ = [
        ("theta", C.c_double),
        ("big_theta", C.c_double),
        ("max_sweeps", C.c_int32),
        ("max_levels", C.c_int32),
        ("stop_rule", C.c_int32),
        ("merge_isolated", C.c_int32),
        ("theta_schedule", C.POINTER(C.c_double)),
        ("theta_schedule_len", C.c_int32),
        ("coloring", C.c_int32),
        ("color_classes", C.c_int32),
        ("color_cap_min_n", C.c_int64),
    ]


_lib = None


def _L():
    global _lib
    if _lib is None:
        lib = C.CDLL(build())
        P = C.c_void_p
        i64, i32, dbl = C.c_int64, C.c_int32, C.c_double
        GP = C.POINTER(_Graph)
        lib.og_graph_build.argtypes = [i64, i64, P, P, P, C.POINTER(GP)]
        lib.og_graph_build.restype = C.c_int
        lib.og_graph_build_real.argtypes = [i64, i64, P, P, P, C.POINTER(i32), C.POINTER(GP)]
        lib.og_graph_build_real.restype = C.c_int
        lib.og_fixed_sum.argtypes = [i64, P, i32]
        lib.og_fixed_sum.restype = i64
        lib.og_graph_free.argtypes = [GP]
        lib.og_modularity.argtypes = [GP, P, P, P, P, P]
        lib.og_modularity.restype = C.c_int
        lib.og_state_new.argtypes = [GP, P]
        lib.og_state_new.restype = P
        lib.og_state_free.argtypes = [P]
        lib.og_decide.argtypes = [P, i64, i32]
        lib.og_decide.restype = i32
        lib.og_sweep.argtypes = [GP, P, P, i32]
        lib.og_sweep.restype = i64
        lib.og_color_priority.argtypes = [i64]
        lib.og_color_priority.restype = C.c_uint64
        lib.og_color.argtypes = [GP, P]
        lib.og_color.restype = i32
        lib.og_sweep_colored.argtypes = [GP, P, i32, P, P]
        lib.og_sweep_colored.restype = i64
        lib.og_renumber.argtypes = [i64, P, P]
        lib.og_renumber.restype = i64
        lib.og_induce.argtypes = [GP, P, i64, C.POINTER(GP)]
        lib.og_induce.restype = C.c_int
        lib.og_run.argtypes = [GP, C.POINTER(_Config), C.POINTER(P)]
        lib.og_run.restype = C.c_int
        lib.og_result_free.argtypes = [P]
        lib.og_result_levels.argtypes = [P]
        lib.og_result_levels.restype = i32
        lib.og_result_level_n.argtypes = [P, i32]
        lib.og_result_level_n.restype = i64
        lib.og_result_level_labels.argtypes = [P, i32, P]
        lib.og_result_level_q.argtypes = [P, i32]
        lib.og_result_level_q.restype = dbl
        lib.og_result_level_sweeps.argtypes = [P, i32]
        lib.og_result_level_sweeps.restype = i32
        lib.og_result_final.argtypes = [P, P]
        lib.og_result_final_q.argtypes = [P]
        lib.og_result_final_q.restype = dbl
        lib.og_result_trace_len.argtypes = [P, i32]
        lib.og_result_trace_len.restype = i32
        lib.og_result_trace.argtypes = [P, i32, P, P]
        lib.og_result_edge_visits.argtypes = [P]
        lib.og_result_edge_visits.restype = i64
        lib.og_config_default.argtypes = [C.POINTER(_Config)]
        lib.og_set_threads.argtypes = [i32]
        lib.og_get_threads.restype = i32
        _lib = lib
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    pass


def set_threads(t: int) -> None:
    """OpenMP threads of the oracle's schedule-independent loops (1 = single-threaded).
    Results are bit-identical for any count (Jacobi sweeps, exact integer sums)."""
    _L().og_set_threads(int(t))


def get_threads() -> int:
    return int(_L().og_get_threads())


class Graph:
    """Oracle CSR (int64 weights).  Built from undirected records (src,dst,w)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def from_edges(cls, n, src, dst, w=None) -> "Graph":
        """Integer weights (or None = 1) build directly; float weights go through the
        fixed-point mapping of reading D28 (``og_graph_build_real``; ``g.scale`` = s)."""
        src = np.ascontiguousarray(src, dtype=np.int32)
        dst = np.ascontiguousarray(dst, dtype=np.int32)
        h = C.POINTER(_Graph)()
        scale = None
        if w is not None and np.asarray(w).dtype.kind == "f":
            wa = np.ascontiguousarray(w, dtype=np.float64)
            s = C.c_int32()
            rc = _L().og_graph_build_real(int(n), len(src), _ptr(src), _ptr(dst), _ptr(wa), C.byref(s), C.byref(h))
            scale = s.value
        else:
            wa = None if w is None else np.ascontiguousarray(w, dtype=np.int64)
            rc = _L().og_graph_build(int(n), len(src), _ptr(src), _ptr(dst), _ptr(wa), C.byref(h))
        if rc not in (0, 3) or not h:
            raise OracleError(f"og_graph_build failed rc={rc}")
        g = cls(h)
        g.rc = rc
        g.scale = scale
        return g

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.og_graph_free(self._h)
            self._h = None

    @property
    def n(self):
        return self._h.contents.n

    @property
    def nnz(self):
        return self._h.contents.nnz

    @property
    def W(self):
        return self._h.contents.W

    def arrays(self):
        g = self._h.contents
        n, nnz = g.n, g.nnz
        return dict(
            row_ptr=np.ctypeslib.as_array(g.row_ptr, (n + 1,)).copy(),
            col=np.ctypeslib.as_array(g.col, (max(nnz, 1),))[:nnz].copy(),
            w=np.ctypeslib.as_array(g.w, (max(nnz, 1),))[:nnz].copy(),
            loop=np.ctypeslib.as_array(g.loop, (n,)).copy(),
            delta=np.ctypeslib.as_array(g.delta, (n,)).copy(),
            W=g.W,
        )

    # ---- single steps (for step-level parity and pins) ----
    def modularity(self, labels):
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        I2, hi, lo, q = C.c_int64(), C.c_int64(), C.c_uint64(), C.c_double()
        rc = _L().og_modularity(self._h, _ptr(lab), C.byref(I2), C.byref(hi), C.byref(lo), C.byref(q))
        if rc:
            raise OracleError(f"og_modularity rc={rc}")
        return dict(I2=I2.value, S2=(hi.value << 64) + lo.value, Q=q.value)

    def sweep(self, labels, mode=0):
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        out = np.empty_like(lab)
        moved = _L().og_sweep(self._h, _ptr(lab), _ptr(out), int(mode))
        return out, int(moved)

    def decide(self, labels, vertices, mode=0):
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        st = _L().og_state_new(self._h, _ptr(lab))
        try:
            return np.array([_L().og_decide(st, int(v), int(mode)) for v in vertices], dtype=np.int32)
        finally:
            _L().og_state_free(st)

    def color(self):
        """Greedy distance-1 colouring by decreasing priority (D29) -> (colors, K)."""
        out = np.empty(self.n, dtype=np.int32)
        K = _L().og_color(self._h, _ptr(out))
        if K < 0:
            raise OracleError("og_color failed")
        return out, int(K)

    def sweep_colored(self, labels, colors, K):
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        col = np.ascontiguousarray(colors, dtype=np.int32)
        out = np.empty_like(lab)
        moved = _L().og_sweep_colored(self._h, _ptr(col), int(K), _ptr(lab), _ptr(out))
        if moved < 0:
            raise OracleError("og_sweep_colored failed")
        return out, int(moved)

    def induce(self, labels, k) -> "Graph":
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        h = C.POINTER(_Graph)()
        rc = _L().og_induce(self._h, _ptr(lab), int(k), C.byref(h))
        if rc:
            raise OracleError(f"og_induce rc={rc}")
        return Graph(h)


def fixed_sum(w, s: int) -> int:
    """T(s) = Σ rint(ω·2^s), saturated at 2^62 (reading D28)."""
    wa = np.ascontiguousarray(w, dtype=np.float64)
    return int(_L().og_fixed_sum(len(wa), _ptr(wa), int(s)))


def renumber(labels):
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    out = np.empty_like(lab)
    k = _L().og_renumber(len(lab), _ptr(lab), _ptr(out))
    return out, int(k)


@dataclass
class Result:
    levels: list = field(default_factory=list)        # per-level dense label arrays
    q: list = field(default_factory=list)             # per-level Q (after merge, D15)
    sweeps: list = field(default_factory=list)
    traces: list = field(default_factory=list)        # per level: (moved[], Q[]) per sweep
    final: np.ndarray | None = None
    final_q: float = 0.0
    edge_visits: int = 0


def color_priority(v: int) -> int:
    return int(_L().og_color_priority(int(v)))


def run(graph: Graph, theta=1e-6, big_theta=1e-6, max_sweeps=100, max_levels=64,
        stop_rule=0, merge_isolated=True, theta_schedule=None, coloring=False,
        color_classes=32, color_cap_min_n=65536) -> Result:
    """Algorithm 2 around Algorithm 1 with the DESIGN.md readings."""
    cfg = _Config()
    _L().og_config_default(C.byref(cfg))
    cfg.theta, cfg.big_theta = float(theta), float(big_theta)
    cfg.max_sweeps, cfg.max_levels = int(max_sweeps), int(max_levels)
    cfg.stop_rule, cfg.merge_isolated = int(stop_rule), int(bool(merge_isolated))
    cfg.coloring = int(bool(coloring))
    cfg.color_classes = int(color_classes)
    cfg.color_cap_min_n = int(color_cap_min_n)
    sched = None
    if theta_schedule:
        sched = (C.c_double * len(theta_schedule))(*theta_schedule)
        cfg.theta_schedule = C.cast(sched, C.POINTER(C.c_double))
        cfg.theta_schedule_len = len(theta_schedule)
    r = C.c_void_p()
    rc = _L().og_run(graph._h, C.byref(cfg), C.byref(r))
    if rc:
        if r:
            _L().og_result_free(r)
        raise OracleError(f"og_run rc={rc}")
    try:
        L = _L()
        res = Result()
        for l in range(L.og_result_levels(r)):
            n = L.og_result_level_n(r, l)
            lab = np.empty(n, dtype=np.int32)
            L.og_result_level_labels(r, l, _ptr(lab))
            res.levels.append(lab)
            res.q.append(L.og_result_level_q(r, l))
            res.sweeps.append(L.og_result_level_sweeps(r, l))
            t = L.og_result_trace_len(r, l)
            mv, qs = np.empty(t, dtype=np.int64), np.empty(t, dtype=np.float64)
            L.og_result_trace(r, l, _ptr(mv), _ptr(qs))
            res.traces.append((mv, qs))
        res.final = np.empty(graph.n, dtype=np.int32)
        L.og_result_final(r, _ptr(res.final))
        res.final_q = L.og_result_final_q(r)
        res.edge_visits = L.og_result_edge_visits(r)
        return res
    finally:
        _L().og_result_free(r)
