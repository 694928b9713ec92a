"""Independent brute-force checker for the oracle (pin P1).

Eq. 1 taken literally as a recursion over Parent(i), on 4x4
homogeneous fp64 matrices with numpy's matmul — no topological order, no 3x4
compose, nothing shared with oracle/oracle.c.
"""
from __future__ import annotations

import numpy as np


def homog(m34) -> np.ndarray:
    h = np.zeros((4, 4), np.float64)
    h[:3, :] = np.asarray(m34, np.float64).reshape(3, 4)
    h[3, 3] = 1.0
    return h


def is_forest(parents) -> bool:
    n = len(parents)
    for i in range(n):
        v, steps = i, 0
        while v != -1:
            if not (-1 <= parents[v] < n):
                return False
            v = parents[v]
            steps += 1
            if steps > n:
                return False
    return True


def global_pose(parents, local) -> np.ndarray:
    """G(i) = G(Parent(i)) @ L(i) by memoised recursion; returns [n,4,4]."""
    n = len(parents)
    memo: dict[int, np.ndarray] = {}

    def g(i):
        if i in memo:
            return memo[i]
        h = homog(local[i])
        r = h if parents[i] == -1 else g(parents[i]) @ h
        memo[i] = r
        return r

    return np.stack([g(i) for i in range(n)]) if n else np.zeros((0, 4, 4))


def root_path_product(parents, local, i) -> np.ndarray:
    """Eq. 1 literally: multiply the matrices along the root path of i (root first)."""
    path = []
    v = i
    while v != -1:
        path.append(v)
        v = parents[v]
    h = np.eye(4)
    for v in reversed(path):
        h = h @ homog(local[v])
    return h
