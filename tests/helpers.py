"""Test helpers: small random graded trees, dense assembly, brute-force tree tables."""
from __future__ import annotations

import numpy as np

from octgen import canonical_order, grade_repair, uniform_tiles


def random_graded_tree(rng, l0=1, lmax=3, p_refine=0.3, ext=(1, 1, 1)):
    tiles = uniform_tiles(l0, ext)
    for _ in range(lmax - l0):
        sel = (tiles[:, 0] < lmax) & (rng.random(len(tiles)) < p_refine)
        if not np.any(sel):
            continue
        par = tiles[sel]
        kids = []
        for d in range(8):
            c = par.copy()
            c[:, 0] += 1
            c[:, 1] = 2 * par[:, 1] + (d & 1)
            c[:, 2] = 2 * par[:, 2] + ((d >> 1) & 1)
            c[:, 3] = 2 * par[:, 3] + (d >> 2)
            kids.append(c)
        tiles = np.concatenate([tiles[~sel]] + kids)
    tiles = grade_repair(tiles, ext)
    return tiles[canonical_order(tiles)]


def morton_py(i, j, k):
    m = 0
    for b in range(21):
        m |= ((i >> b) & 1) << (3 * b)
        m |= ((j >> b) & 1) << (3 * b + 1)
        m |= ((k >> b) & 1) << (3 * b + 2)
    return m


def brute_force_tables(tiles, ext=(1, 1, 1)):
    """Independent plain-Python construction of the canonical tile order and tables
    (definitions in include/octmg.h / SURVEY c-1)."""
    leaves = {tuple(int(v) for v in t) for t in tiles}
    inners = set()
    for (l, i, j, k) in leaves:
        while l > 0:
            l, i, j, k = l - 1, i // 2, j // 2, k // 2
            inners.add((l, i, j, k))
    key = lambda t: (-t[0], morton_py(t[1], t[2], t[3]))
    order = sorted(leaves, key=key) + sorted(inners, key=key)
    index = {t: n for n, t in enumerate(order)}
    NL = len(leaves)
    nbr = np.full((len(order), 6), -1, dtype=np.int64)
    parent = np.full(len(order), -1, dtype=np.int64)
    child = np.full((len(inners), 8), -1, dtype=np.int64)
    for n, (l, i, j, k) in enumerate(order):
        for f in range(6):
            q = [i, j, k]
            q[f // 2] += 1 if f & 1 else -1
            if q[f // 2] < 0 or q[f // 2] >= (ext[f // 2] << l):
                continue
            t = (l, *q)
            if t in index:
                nbr[n, f] = index[t]
            else:
                c = (l - 1, q[0] // 2, q[1] // 2, q[2] // 2)
                assert c in leaves and n < NL
                nbr[n, f] = -2 - index[c]
        if l > 0:
            parent[n] = index[(l - 1, i // 2, j // 2, k // 2)]
        if n >= NL:
            for d in range(8):
                child[n - NL, d] = index[(l + 1, 2 * i + (d & 1), 2 * j + ((d >> 1) & 1), 2 * k + (d >> 2))]
    return np.array(order, dtype=np.int64), nbr, parent, child


def dense_composite(orc):
    N = orc.N
    A = np.zeros((N, N))
    e = np.zeros(N)
    for j in range(N):
        e[j] = 1.0
        A[:, j] = orc.apply(e)
        e[j] = 0.0
    return A


def dense_level(orc, level, cells):
    """Dense A^level restricted to the given all-tile cell indices."""
    n = len(cells)
    A = np.zeros((n, n))
    u = np.zeros(orc.T * orc.B3)
    for jj, j in enumerate(cells):
        u[j] = 1.0
        y = orc.apply_level(level, u)
        A[:, jj] = y[cells]
        u[j] = 0.0
    return A
