"""ctypes binding of ``csrc/liblouvain.so`` (C ABI in ``include/louvain.h``).

Argument marshalling only: every step of the method runs in the library's CUDA
kernels.  There is no CPU fallback — if the shared library is missing this module
raises ``ImportError``/``LouvainError`` instead of computing anything.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "csrc", "liblouvain.so")

LV_OK, LV_EINVAL, LV_EGRAPH, LV_EZEROW, LV_ENOMEM, LV_ECUDA, LV_ENCCL, LV_ESTATE, LV_ERANGE = range(9)
STATUS_NAMES = ["LV_OK", "LV_EINVAL", "LV_EGRAPH", "LV_EZEROW", "LV_ENOMEM", "LV_ECUDA", "LV_ENCCL",
                "LV_ESTATE", "LV_ERANGE"]
LV_W_NONE, LV_W_I32, LV_W_I64, LV_W_F32, LV_W_F64 = 0, 1, 2, 3, 4

EXPORTS = [
    "louvain_config_default", "louvain_create", "louvain_run", "louvain_num_levels", "louvain_level_size",
    "louvain_get_partition", "louvain_modularity", "louvain_weight_scale", "louvain_level_colors", "louvain_color", "louvain_level_stats", "louvain_run_stats", "louvain_sweep",
    "louvain_time_sweeps", "louvain_profile_json", "louvain_get_csr", "louvain_contract", "louvain_last_error", "louvain_destroy",
    "louvain_nccl_unique_id", "louvain_nccl_init", "louvain_nccl_destroy", "louvain_shard_bounds",
]

ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class Graph(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("m", C.c_int64),
        ("src", C.c_void_p),
        ("dst", C.c_void_p),
        ("w", C.c_void_p),
        ("wtype", C.c_int32),
        ("on_device", C.c_int32),
    ]


class Config(C.Structure):
    _fields_ = [
        ("theta", C.c_double),
        ("big_theta", C.c_double),
        ("max_sweeps", C.c_int32),
        ("max_levels", C.c_int32),
        ("stop_rule", C.c_int32),
        ("merge_isolated", C.c_int32),
        ("theta_schedule", C.POINTER(C.c_double)),
        ("theta_schedule_len", C.c_int32),
        ("device", C.c_int32),
        ("stream", C.c_void_p),
        ("alloc", ALLOC_FN),
        ("free", FREE_FN),
        ("alloc_ctx", C.c_void_p),
        ("nccl_comm", C.c_void_p),
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("profile", C.c_int32),
        ("coloring", C.c_int32),
        ("color_classes", C.c_int32),
        ("color_cap_min_n", C.c_int64),
        ("reorder", C.c_int32),
    ]


class LouvainError(RuntimeError):
    def __init__(self, code, msg=""):
        name = STATUS_NAMES[code] if 0 <= code < len(STATUS_NAMES) else str(code)
        super().__init__(f"{name}: {msg}" if msg else name)
        self.code = code


_lib = None


def load() -> C.CDLL:
    """Load the in-tree CUDA library; raise if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise ImportError(f"liblouvain.so not built ({SO_PATH}); run `python -m paper_1805_10904_b200.build` "
                          "(there is no CPU fallback)")
    # LV_SO: an alternative in-tree build of the same library (tuning experiments)
    lib = C.CDLL(os.environ.get("LV_SO", SO_PATH), mode=C.RTLD_GLOBAL)
    P, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    sig = {
        "louvain_config_default": ([C.POINTER(Config)], C.c_int),
        "louvain_create": ([C.POINTER(Graph), C.POINTER(Config), C.POINTER(P)], C.c_int),
        "louvain_run": ([P], C.c_int),
        "louvain_num_levels": ([P, C.POINTER(i32)], C.c_int),
        "louvain_weight_scale": ([P, C.POINTER(i32)], C.c_int),
        "louvain_level_colors": ([P, i32, C.POINTER(i32), C.POINTER(i32)], C.c_int),
        "louvain_color": ([P, P, i32, C.POINTER(i32)], C.c_int),
        "louvain_level_size": ([P, i32, C.POINTER(i64)], C.c_int),
        "louvain_get_partition": ([P, i32, P, i64, i32], C.c_int),
        "louvain_modularity": ([P, i32, C.POINTER(dbl)], C.c_int),
        "louvain_level_stats": ([P, i32, C.POINTER(i32), P], C.c_int),
        "louvain_run_stats": ([P, C.POINTER(i64), C.POINTER(i64)], C.c_int),
        "louvain_sweep": ([P, P, P, i32, i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.POINTER(u64)], C.c_int),
        "louvain_time_sweeps": ([P, i32, i32, C.c_char_p, i64], C.c_int),
        "louvain_profile_json": ([P, C.c_char_p, i64], C.c_int),
        "louvain_get_csr": ([P, C.POINTER(i64), P, P, P, P, P, C.POINTER(i64)], C.c_int),
        "louvain_contract": ([P, P, i64, C.POINTER(i64), P, P, P, P, P], C.c_int),
        "louvain_last_error": ([P], C.c_char_p),
        "louvain_destroy": ([P], None),
        "louvain_nccl_unique_id": ([P], C.c_int),
        "louvain_nccl_init": ([P, i32, i32, i32, C.POINTER(P)], C.c_int),
        "louvain_nccl_destroy": ([P], C.c_int),
        "louvain_shard_bounds": ([P, i64, i32, P], C.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def check(rc: int, handle=None):
    if rc != LV_OK:
        msg = load().louvain_last_error(handle)
        raise LouvainError(rc, msg.decode() if msg else "")
