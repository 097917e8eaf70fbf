"""Leaf-tile list generators (workload shapes only; no solver arithmetic).

Tiles are ``(level, i, j, k)`` int64 rows.  At level ``l`` there are ``ext*2^l``
tiles per axis, each 8^3 cells of edge ``h_l = 2^-l / 8`` (P:L385, P:L873,
P:L1229: l0 = 3 gives a 64-cell base).  All tile lists returned here are graded
across faces ("two face-neighboring leaf cells may differ by at most one
level") when ``repair=True``.
"""
from __future__ import annotations

import numpy as np

B = 8  # tile edge in cells


def _spread3(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
    v = (v | (v << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    v = (v | (v << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
    return v


def morton3(i, j, k) -> np.ndarray:
    """Bit-interleave (x in the lowest bit of each triple), 21 bits per axis."""
    i = np.asarray(i); j = np.asarray(j); k = np.asarray(k)
    return _spread3(i) | (_spread3(j) << np.uint64(1)) | (_spread3(k) << np.uint64(2))


def canonical_order(tiles: np.ndarray) -> np.ndarray:
    """Permutation that sorts leaf tiles by (level descending, Morton ascending).

    This is the documented leaf-slot order of the C ABI (include/octmg.h)."""
    tiles = np.asarray(tiles, dtype=np.int64)
    m = morton3(tiles[:, 1], tiles[:, 2], tiles[:, 3])
    return np.lexsort((m, -tiles[:, 0]))


def tile_counts_by_level(tiles: np.ndarray) -> dict:
    lv, cnt = np.unique(np.asarray(tiles)[:, 0], return_counts=True)
    return {int(a): int(b) for a, b in zip(lv, cnt)}


def uniform_tiles(level: int, ext=(1, 1, 1)) -> np.ndarray:
    n = [e << level for e in ext]
    i, j, k = np.meshgrid(np.arange(n[0]), np.arange(n[1]), np.arange(n[2]), indexing="ij")
    t = np.stack([np.full(i.size, level), i.ravel(), j.ravel(), k.ravel()], axis=1)
    return t.astype(np.int64)


def _children(t: np.ndarray) -> np.ndarray:
    out = []
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                c = t.copy()
                c[:, 0] += 1
                c[:, 1] = 2 * t[:, 1] + dx
                c[:, 2] = 2 * t[:, 2] + dy
                c[:, 3] = 2 * t[:, 3] + dz
                out.append(c)
    return np.concatenate(out, axis=0) if out else t[:0]


def octant_tiles(base_level: int = 1, refine=((0, 0, 0),), ext=(1, 1, 1)) -> np.ndarray:
    """BASELINE config 1: a level-1 base (16^3 cells) with tile (1,0,0,0) refined once
    -> 7 leaf tiles at level 1 and 8 at level 2 (7680 leaf cells)."""
    base = uniform_tiles(base_level, ext)
    ref = np.array([[base_level, *r] for r in refine], dtype=np.int64)
    keep = ~np.any(np.all(base[:, None, :] == ref[None, :, :], axis=2), axis=1)
    return np.concatenate([base[keep], _children(ref)], axis=0)


def _box_sphere_strict(t: np.ndarray, center, r) -> np.ndarray:
    """Strict box-vs-sphere-surface test d_min < r < d_max (SURVEY c-1 pin reading of
    P:L1224 "If a tile intersects the zero level set")."""
    size = np.ldexp(1.0, -t[:, 0].astype(np.int64))
    lo = t[:, 1:4] * size[:, None]
    hi = lo + size[:, None]
    c = np.asarray(center, dtype=np.float64)[None, :]
    nearest = np.clip(c, lo, hi)
    dmin = np.sqrt(((nearest - c) ** 2).sum(1))
    far = np.maximum(np.abs(c - lo), np.abs(c - hi))
    dmax = np.sqrt((far ** 2).sum(1))
    return (dmin < r) & (r < dmax)


def sphere_band_tiles(l0: int, extra: int = 2, center=(0.5, 0.5, 0.5), r: float = 0.25,
                      ext=(1, 1, 1), repair: bool = True) -> np.ndarray:
    """Narrow-band grid of P:L1224: tiles intersecting the sphere surface get target
    level l0+extra (paper: extra=2), others l0.  Refinement is top-down; then grading
    repair to fixpoint (refine the coarser side)."""
    leaves = []
    cur = uniform_tiles(l0, ext)
    for _ in range(extra):
        hit = _box_sphere_strict(cur, center, r)
        leaves.append(cur[~hit])
        cur = _children(cur[hit])
    leaves.append(cur)
    tiles = np.concatenate(leaves, axis=0)
    if repair:
        tiles = grade_repair(tiles, ext)
    return tiles


def _level_sets(tiles):
    sets = {}
    for l in np.unique(tiles[:, 0]):
        t = tiles[tiles[:, 0] == l]
        sets[int(l)] = np.sort(morton3(t[:, 1], t[:, 2], t[:, 3]))
    return sets


def _find_violations(tiles: np.ndarray, ext):
    """Return list of (level m, indices into tiles-at-level-m) of leaves covering a
    face-neighbour position of a leaf two or more levels finer."""
    ext = np.asarray(ext, dtype=np.int64)
    levels = sorted(int(l) for l in np.unique(tiles[:, 0]))
    sets = _level_sets(tiles)
    marks = {m: np.zeros(len(sets[m]), dtype=bool) for m in levels}
    any_v = False
    for l in levels:
        t = tiles[tiles[:, 0] == l]
        for axis in range(3):
            for sgn in (-1, 1):
                q = t[:, 1:4].copy()
                q[:, axis] += sgn
                lim = ext << l
                inside = np.all((q >= 0) & (q < lim[None, :]), axis=1)
                q = q[inside]
                for m in levels:
                    if m > l - 2:
                        continue
                    qm = q >> (l - m)
                    key = morton3(qm[:, 0], qm[:, 1], qm[:, 2])
                    s = sets[m]
                    pos = np.searchsorted(s, key)
                    pos_c = np.minimum(pos, len(s) - 1)
                    found = (len(s) > 0) & (s[pos_c] == key)
                    if np.any(found):
                        marks[m][pos_c[found]] = True
                        any_v = True
    return any_v, marks, sets


def grade_repair(tiles: np.ndarray, ext=(1, 1, 1)) -> np.ndarray:
    """Refine coarse leaves that face-neighbour a leaf >= 2 levels finer, to fixpoint."""
    tiles = np.asarray(tiles, dtype=np.int64)
    while True:
        any_v, marks, sets = _find_violations(tiles, ext)
        if not any_v:
            return tiles
        out = []
        for m, s in sets.items():
            t = tiles[tiles[:, 0] == m]
            key = morton3(t[:, 1], t[:, 2], t[:, 3])
            order = np.argsort(key)
            t = t[order]
            mk = marks[m]
            out.append(t[~mk])
            if np.any(mk):
                out.append(_children(t[mk]))
        tiles = np.concatenate(out, axis=0)


def is_graded(tiles: np.ndarray, ext=(1, 1, 1)) -> bool:
    any_v, _, _ = _find_violations(np.asarray(tiles, dtype=np.int64), ext)
    return not any_v


def leaf_cell_geometry(tiles_sorted: np.ndarray, t0: int = 0, t1: int | None = None):
    """Cell centres (n,3) and edges h (n,) for tiles[t0:t1] (already in canonical order),
    cells ordered x + 8y + 64z within a tile."""
    t = np.asarray(tiles_sorted, dtype=np.int64)[t0:t1]
    h = np.ldexp(1.0, -t[:, 0].astype(np.int64)) / B
    z, y, x = np.meshgrid(np.arange(B), np.arange(B), np.arange(B), indexing="ij")
    loc = np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1).astype(np.float64)  # (512,3)
    base = t[:, 1:4].astype(np.float64) * B
    cen = (base[:, None, :] + loc[None, :, :] + 0.5) * h[:, None, None]
    hh = np.repeat(h, B * B * B)
    return cen.reshape(-1, 3), hh
