"""Independent brute-force definitions used to PIN the oracle (tests only).

Nothing here is shared with ``oracle/`` or with the CUDA path; every quantity is
recomputed from the paper's definitions by a different route than the oracle takes:

* ``q_exact``   — Eq. 3 as the textbook pair sum
                  Q = 1/(2W) Σ_ij [A_ij − δ_i δ_j / 2W] [C_i = C_j],  A_ii = 2·loop_i,
                  in exact rationals (the oracle uses I2/S2 aggregates and int128).
* ``decide``    — Eq. 5 with §3.1.1/§3.1.2 heuristics, where the gain of every
                  candidate is obtained by RE-EVALUATING Eq. 3 after the move (the
                  oracle uses the closed-form Eq. 4 score, reading D4).
* ``optimum``   — exhaustive search over all set partitions (restricted growth strings).
"""
from __future__ import annotations

from fractions import Fraction
from itertools import product

import numpy as np


class G:
    """Small undirected weighted graph with loops, from undirected records."""

    def __init__(self, n, src, dst, w=None):
        self.n = n
        self.adj = [dict() for _ in range(n)]
        self.loop = [0] * n
        self.W = 0
        for k in range(len(src)):
            u, v = int(src[k]), int(dst[k])
            wk = 1 if w is None else int(w[k])
            self.W += wk
            if u == v:
                self.loop[u] += wk
            else:
                self.adj[u][v] = self.adj[u].get(v, 0) + wk
                self.adj[v][u] = self.adj[v].get(u, 0) + wk
        self.delta = [sum(self.adj[i].values()) + 2 * self.loop[i] for i in range(n)]

    def A(self, i, j):
        return 2 * self.loop[i] if i == j else self.adj[i].get(j, 0)


def q_exact(g: G, labels) -> Fraction:
    """Eq. 3 as the pair sum (1/2W) Σ_ij [A_ij − δ_iδ_j/2W] [C_i = C_j]."""
    twoW = 2 * g.W
    tot = Fraction(0)
    for i in range(g.n):
        for j in range(g.n):
            if labels[i] == labels[j]:
                tot += Fraction(g.A(i, j)) - Fraction(g.delta[i] * g.delta[j], twoW)
    return tot / twoW


def decide(g: G, labels, i, mode=0) -> int:
    """One vertex's decision against the snapshot ``labels`` (Jacobi)."""
    own = labels[i]
    nbr = sorted({labels[j] for j in g.adj[i]})
    if not nbr:
        return own
    size = {}
    for c in labels:
        size[c] = size.get(c, 0) + 1
    if mode == 1:  # isolated merge: singlet with exactly one neighbour community
        if size[own] != 1:
            return own
        others = [c for c in nbr if c != own]
        if len(others) != 1:
            return own
        T = others[0]
        return own if (size[T] == 1 and T > own) else T
    base = q_exact(g, labels)
    best, best_q = None, None
    for c in nbr:
        if c == own:
            continue
        moved = list(labels)
        moved[i] = c
        q = q_exact(g, moved)
        if best is None or q > best_q or (q == best_q and c < best):
            best, best_q = c, q
    if best is None or not (best_q > base):
        return own
    if size[own] == 1 and size[best] == 1 and best > own:
        return own
    return best


def sweep(g: G, labels, mode=0):
    return [decide(g, labels, i, mode) for i in range(g.n)]


def rgs(n):
    """All set partitions of range(n) as restricted growth strings (numpy array)."""
    out = []

    def rec(prefix, mx):
        if len(prefix) == n:
            out.append(list(prefix))
            return
        for c in range(mx + 2):
            prefix.append(c)
            rec(prefix, max(mx, c))
            prefix.pop()

    rec([0], 0)
    return np.array(out, dtype=np.int64)


def optimum(g: G) -> Fraction:
    """max over all partitions of Eq. 3, via exact integer numerators."""
    P = rgs(g.n)
    twoW = 2 * g.W
    I2 = np.full(len(P), 2 * sum(g.loop), dtype=np.int64)
    for i in range(g.n):
        for j, wij in g.adj[i].items():
            I2 += wij * (P[:, i] == P[:, j])
    S2 = np.zeros(len(P), dtype=np.int64)
    delta = np.array(g.delta, dtype=np.int64)
    for c in range(g.n):
        dc = ((P == c) * delta[None, :]).sum(axis=1)
        S2 += dc * dc
    num = twoW * I2 - S2
    return Fraction(int(num.max()), twoW * twoW)
