"""Reference of the F3 input relabel ("divergence ... could be reduced by
ordering the vertices by degree"), written from include/louvain.h's definition of
louvain_config.reorder — test infrastructure, independent of the CUDA path:

    d(v)   = number of non-loop records incident to v (duplicates counted)
    key(v) = 31 - floor(log2 d(v))  (d >= 1),  32  (d = 0)
    new id = position of v in the stable order of key (ascending key, then old id)

so vertices are grouped by decreasing degree class.  `relabel` returns the records with
both endpoints mapped and perm (perm[old] = new); the oracle runs on the relabelled
records, and the GPU's level-0 / final partitions (indexed by old ids) must equal the
oracle's at perm[v].
"""
import numpy as np


def degree_perm(n, src, dst):
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    nl = src != dst
    d = np.bincount(src[nl], minlength=n) + np.bincount(dst[nl], minlength=n)
    key = np.full(n, 32, dtype=np.int64)
    pos = d > 0
    key[pos] = 31 - np.floor(np.log2(d[pos])).astype(np.int64)
    inv = np.argsort(key, kind="stable")  # new -> old
    perm = np.empty(n, dtype=np.int64)
    perm[inv] = np.arange(n)
    return perm, key


def relabel(n, src, dst):
    perm, _ = degree_perm(n, src, dst)
    return perm, perm[np.asarray(src)].astype(np.int32), perm[np.asarray(dst)].astype(np.int32)
