"""Python API over the C ABI (include/louvain.h).  Marshalling only.

    from paper_1805_10904_b200 import Louvain, inputs
    g = inputs.karate()
    lv = Louvain(g.n, g.src, g.dst, g.w)          # host numpy arrays, or CUDA tensors
    lv.run()
    lv.partition(), lv.modularity(), lv.num_levels

Device memory comes from PyTorch's caching allocator (through the library's
allocation hooks) when torch with CUDA is available; the work runs on a
library-owned CUDA stream unless ``stream=`` (a ``torch.cuda.Stream`` or raw handle)
is given.
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import _lib
from ._lib import Config, Graph, LouvainError, check

_CAP = 1 << 16


def _torch():
    try:
        import torch

        return torch if torch.cuda.is_available() else None
    except Exception:  # pragma: no cover
        return None


def _is_cuda_tensor(x):
    t = _torch()
    return t is not None and isinstance(x, t.Tensor) and x.is_cuda


class _TorchAllocator:
    """Routes the library's device allocations to torch's caching allocator."""

    def __init__(self, device):
        import torch

        self.device = device
        self._torch = torch

        def _alloc(ctx, nbytes, stream):
            try:
                return int(torch.cuda.caching_allocator_alloc(int(nbytes), device, stream or 0))
            except Exception:
                return 0

        def _free(ctx, ptr, nbytes, stream):
            try:
                torch.cuda.caching_allocator_delete(ptr)
            except Exception:
                pass

        self.alloc = _lib.ALLOC_FN(_alloc)
        self.free = _lib.FREE_FN(_free)


def default_config(**kw) -> Config:
    cfg = Config()
    check(_lib.load().louvain_config_default(C.byref(cfg)))
    for k, v in kw.items():
        if k == "theta_schedule":
            continue
        if not hasattr(cfg, k):
            raise TypeError(f"unknown config field {k}")
        setattr(cfg, k, v)
    return cfg


class Louvain:
    """One graph on one GPU: ``louvain_create`` at construction, ``run()`` = Alg. 2."""

    def __init__(self, n, src, dst, w=None, *, device=0, stream=None, torch_allocator=True,
                 theta=1e-6, big_theta=1e-6, max_sweeps=100, max_levels=64, stop_rule=0,
                 merge_isolated=True, theta_schedule=None, nccl_comm=None, rank=0, world=1, profile=False,
                 coloring=False, color_classes=32, color_cap_min_n=65536, reorder=False):
        self._lib = _lib.load()
        self._h = C.c_void_p()
        self._keep = []
        cfg = default_config(theta=float(theta), big_theta=float(big_theta), max_sweeps=int(max_sweeps),
                             max_levels=int(max_levels), stop_rule=int(stop_rule),
                             merge_isolated=int(bool(merge_isolated)), device=int(device), rank=int(rank),
                             world=int(world), profile=int(bool(profile)), coloring=int(bool(coloring)),
                             color_classes=int(color_classes), color_cap_min_n=int(color_cap_min_n),
                             reorder=int(bool(reorder)))
        if theta_schedule:
            arr = (C.c_double * len(theta_schedule))(*[float(x) for x in theta_schedule])
            self._keep.append(arr)
            cfg.theta_schedule = C.cast(arr, C.POINTER(C.c_double))
            cfg.theta_schedule_len = len(theta_schedule)
        if stream is not None:
            cfg.stream = C.c_void_p(int(getattr(stream, "cuda_stream", stream)))
        if torch_allocator and _torch() is not None:
            self._alloc = _TorchAllocator(device)
            cfg.alloc = self._alloc.alloc
            cfg.free = self._alloc.free
        if nccl_comm is not None:
            cfg.nccl_comm = C.c_void_p(int(nccl_comm))
        g = Graph()
        g.n = int(n)
        if _is_cuda_tensor(src):
            t = _torch()
            s = src.to(t.int32).contiguous()
            d = dst.to(t.int32).contiguous()
            self._keep += [s, d]
            g.src, g.dst, g.on_device = s.data_ptr(), d.data_ptr(), 1
            g.m = s.numel()
            if w is None:
                g.w, g.wtype = None, _lib.LV_W_NONE
            else:
                ww = w.contiguous()
                kinds = {t.int32: _lib.LV_W_I32, t.int64: _lib.LV_W_I64, t.float32: _lib.LV_W_F32,
                         t.float64: _lib.LV_W_F64}
                if ww.dtype not in kinds:
                    raise TypeError("weights must be int32/int64 (exact) or float32/float64 (fixed point, D28)")
                self._keep.append(ww)
                g.w = ww.data_ptr()
                g.wtype = kinds[ww.dtype]
            # the conversions above ran on torch's current stream, while louvain_create
            # reads the buffers on cfg.stream (or a library-owned stream): order them
            t.cuda.current_stream(s.device).synchronize()
        else:
            s = np.ascontiguousarray(src, dtype=np.int32)
            d = np.ascontiguousarray(dst, dtype=np.int32)
            self._keep += [s, d]
            g.src, g.dst, g.on_device = s.ctypes.data, d.ctypes.data, 0
            g.m = s.shape[0]
            if w is None:
                g.w, g.wtype = None, _lib.LV_W_NONE
            else:
                ww = np.ascontiguousarray(w)
                kinds = {np.dtype(np.int32): _lib.LV_W_I32, np.dtype(np.int64): _lib.LV_W_I64,
                         np.dtype(np.float32): _lib.LV_W_F32, np.dtype(np.float64): _lib.LV_W_F64}
                if ww.dtype not in kinds:
                    if ww.dtype.kind in "iu":
                        ww = ww.astype(np.int64)
                    elif ww.dtype.kind == "f":
                        ww = ww.astype(np.float64)
                    else:
                        raise TypeError("weights must be integers (exact) or reals (fixed point, D28)")
                self._keep.append(ww)
                g.w = ww.ctypes.data
                g.wtype = kinds[ww.dtype]
        rc = self._lib.louvain_create(C.byref(g), C.byref(cfg), C.byref(self._h))
        self._keep = [k for k in self._keep if not isinstance(k, np.ndarray)]
        check(rc, None)
        self.n = int(n)
        self.device = device

    # ---------------------------------------------------------------- lifecycle
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.louvain_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---------------------------------------------------------------- Alg. 2
    def run(self):
        check(self._lib.louvain_run(self._h), self._h)
        return self

    @property
    def weight_scale(self) -> int:
        """s of the real-weight fixed point w~ = rint(w·2^s) (reading D28); 0 for integers."""
        x = C.c_int32()
        check(self._lib.louvain_weight_scale(self._h, C.byref(x)), self._h)
        return x.value

    def level_colors(self, level: int):
        """(colours, Jones–Plassmann rounds) of a level under cfg.coloring (D29)."""
        k, r = C.c_int32(), C.c_int32()
        check(self._lib.louvain_level_colors(self._h, int(level), C.byref(k), C.byref(r)), self._h)
        return k.value, r.value

    def color(self):
        """Distance-1 colouring of the level-0 graph (D29) -> (colors int32[n], K)."""
        out = np.empty(self.n, dtype=np.int32)
        k = C.c_int32()
        check(self._lib.louvain_color(self._h, out.ctypes.data, 0, C.byref(k)), self._h)
        return out, k.value

    @property
    def num_levels(self) -> int:
        x = C.c_int32()
        check(self._lib.louvain_num_levels(self._h, C.byref(x)), self._h)
        return x.value

    def level_size(self, level: int) -> int:
        x = C.c_int64()
        check(self._lib.louvain_level_size(self._h, int(level), C.byref(x)), self._h)
        return x.value

    def partition(self, level: int = -1, out=None):
        """Level labels (level >= 0) or the final composed partition (level = -1).
        Returns a numpy array, or fills ``out`` (a CUDA int32 tensor) in place."""
        n = self.n if level < 0 else self.level_size(level)
        if out is not None and _is_cuda_tensor(out):
            check(self._lib.louvain_get_partition(self._h, int(level), C.c_void_p(out.data_ptr()), out.numel(), 1),
                  self._h)
            return out
        a = np.empty(n, dtype=np.int32)
        check(self._lib.louvain_get_partition(self._h, int(level), a.ctypes.data, n, 0), self._h)
        return a

    def modularity(self, level: int = -1) -> float:
        q = C.c_double()
        check(self._lib.louvain_modularity(self._h, int(level), C.byref(q)), self._h)
        return q.value

    def level_stats(self, level: int):
        s = C.c_int32()
        t = (C.c_double * 5)()
        check(self._lib.louvain_level_stats(self._h, int(level), C.byref(s), t), self._h)
        return s.value, dict(zip(["neighbour", "init", "onelevel", "renumber", "induce"], list(t)))

    def run_stats(self):
        e, l = C.c_int64(), C.c_int64()
        check(self._lib.louvain_run_stats(self._h, C.byref(e), C.byref(l)), self._h)
        return dict(edge_visits=e.value, launches=l.value)

    # ---------------------------------------------------------------- step-level API
    def sweep(self, labels, mode: int = 0):
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        out = np.empty_like(lab)
        mv, i2, hi, lo = C.c_int64(), C.c_int64(), C.c_int64(), C.c_uint64()
        check(self._lib.louvain_sweep(self._h, lab.ctypes.data, out.ctypes.data, int(mode), 0, C.byref(mv),
                                      C.byref(i2), C.byref(hi), C.byref(lo)), self._h)
        return out, mv.value, i2.value, (hi.value << 64) + lo.value

    def time_sweeps(self, warm: int = 3, reps: int = 5) -> dict:
        buf = C.create_string_buffer(_CAP)
        check(self._lib.louvain_time_sweeps(self._h, int(warm), int(reps), buf, _CAP), self._h)
        return json.loads(buf.value.decode())

    def profile(self) -> dict:
        buf = C.create_string_buffer(_CAP)
        check(self._lib.louvain_profile_json(self._h, buf, _CAP), self._h)
        return json.loads(buf.value.decode())

    def nnz(self) -> int:
        """Directed non-loop adjacency entries of the level-0 CSR."""
        nnz, W = C.c_int64(), C.c_int64()
        check(self._lib.louvain_get_csr(self._h, C.byref(nnz), None, None, None, None, None, C.byref(W)), self._h)
        return nnz.value

    def csr(self) -> dict:
        nnz, W = C.c_int64(), C.c_int64()
        check(self._lib.louvain_get_csr(self._h, C.byref(nnz), None, None, None, None, None, C.byref(W)), self._h)
        n, m = self.n, nnz.value
        rp = np.empty(n + 1, np.int64)
        col = np.empty(max(m, 1), np.int32)
        w = np.empty(max(m, 1), np.int64)
        loop = np.empty(n, np.int64)
        delta = np.empty(n, np.int64)
        check(self._lib.louvain_get_csr(self._h, C.byref(nnz), rp.ctypes.data, col.ctypes.data, w.ctypes.data,
                                        loop.ctypes.data, delta.ctypes.data, C.byref(W)), self._h)
        return dict(row_ptr=rp, col=col[:m], w=w[:m], loop=loop, delta=delta, W=W.value)

    def contract(self, labels, k: int) -> dict:
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        nnz = C.c_int64()
        check(self._lib.louvain_contract(self._h, lab.ctypes.data, int(k), C.byref(nnz), None, None, None, None,
                                         None), self._h)
        m = nnz.value
        rp = np.empty(k + 1, np.int64)
        col = np.empty(max(m, 1), np.int32)
        w = np.empty(max(m, 1), np.int64)
        loop = np.empty(k, np.int64)
        delta = np.empty(k, np.int64)
        check(self._lib.louvain_contract(self._h, lab.ctypes.data, int(k), C.byref(nnz), rp.ctypes.data,
                                         col.ctypes.data, w.ctypes.data, loop.ctypes.data, delta.ctypes.data),
              self._h)
        return dict(row_ptr=rp, col=col[:m], w=w[:m], loop=loop, delta=delta)


def run(n, src, dst, w=None, **kw):
    """Convenience: create + run + (final partition, per-level labels, per-level Q)."""
    with Louvain(n, src, dst, w, **kw) as lv:
        lv.run()
        L = lv.num_levels
        return dict(final=lv.partition(-1), levels=[lv.partition(l) for l in range(L)],
                    q=[lv.modularity(l) for l in range(L)], sweeps=[lv.level_stats(l)[0] for l in range(L)],
                    final_q=lv.modularity(-1))
