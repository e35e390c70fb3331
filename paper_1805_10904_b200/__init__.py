"""B200-native (sm_100a) GPU Louvain hot path of arXiv 1805.10904 (Forster 2018).

The compute runs in ``csrc/liblouvain.so`` (hand-written CUDA, C ABI in
``include/louvain.h``); this package only marshals arguments.  ``inputs`` holds the
seeded synthetic-graph generators and text loaders.
"""
from . import inputs  # noqa: F401
from ._lib import LouvainError  # noqa: F401
from .louvain import Louvain, run  # noqa: F401

__all__ = ["Louvain", "LouvainError", "run", "inputs"]
