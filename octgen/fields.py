"""Per-leaf-cell input fields (kinds, face weights, right-hand sides).

Workload recipe only:

* kinds: fluid / Dirichlet / Neumann (ghost-fluid classification);
  Neumann where the solid SDF is negative at the cell centre (SPEC S:L124 reading).
* face weights ``w in [0,1]``: fluid area fraction of each cell face from corner SDF
  samples by marching squares ("signed distance values are evaluated at cell
  corners"), times beta.
* RHS in the volume-integrated SPD convention ``A p = b``, ``A ~ -div(beta grad) * V``
  (P:L290-299).

Face order everywhere: x-, x+, y-, y+, z-, z+.
"""
from __future__ import annotations

import numpy as np

from .trees import B, leaf_cell_geometry

FLUID, DIRICHLET, NEUMANN = 0, 1, 2

_M64 = (1 << 64) - 1


def splitmix64_uniform(seed: int, slots: np.ndarray) -> np.ndarray:
    """U(-1,1) from splitmix64(seed ^ slot) — counter-based, so any side can regenerate it."""
    z = (np.asarray(slots, dtype=np.uint64) ^ np.uint64(seed & _M64))
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))
    return (2.0 * u - 1.0)


def random_rhs(n: int, seed: int = 0) -> np.ndarray:
    return splitmix64_uniform(seed, np.arange(n, dtype=np.uint64)).astype(np.float32)


def _sin_exact(p):
    # f = -sin(2 pi x) sin(2 pi y) sin(2 pi z) / (3 pi)   (P:L1341 with G=A=1, L=1)
    s = np.sin(2 * np.pi * p[..., 0]) * np.sin(2 * np.pi * p[..., 1]) * np.sin(2 * np.pi * p[..., 2])
    return -s / (3 * np.pi)


def _sin_source(p):
    # g = -lap f = -4 pi sin sin sin
    s = np.sin(2 * np.pi * p[..., 0]) * np.sin(2 * np.pi * p[..., 1]) * np.sin(2 * np.pi * p[..., 2])
    return -4 * np.pi * s


def sinusoid_exact(centres: np.ndarray) -> np.ndarray:
    return _sin_exact(centres)


def sinusoid_rhs(tiles_sorted: np.ndarray, ext=(1, 1, 1), wall_bc=(1, 1, 1, 1, 1, 1),
                 chunk_tiles: int = 8192) -> np.ndarray:
    """b_i = V_i * g(x_i) + sum over Dirichlet wall faces of kappa * f(x_ext), kappa = h
    (w = 1), x_ext = centre of the virtual wall cell at distance h (SURVEY c-9 'BC-folded
    sinusoid').  All cells fluid."""
    t = np.asarray(tiles_sorted, dtype=np.int64)
    out = np.empty(len(t) * B ** 3, dtype=np.float32)
    ext = np.asarray(ext, dtype=np.float64)
    for t0 in range(0, len(t), chunk_tiles):
        t1 = min(len(t), t0 + chunk_tiles)
        cen, h = leaf_cell_geometry(t, t0, t1)
        b = h ** 3 * _sin_source(cen)
        for axis in range(3):
            for side in (0, 1):
                f = 2 * axis + side
                if not wall_bc[f]:
                    continue
                if side == 0:
                    at = cen[:, axis] - 0.5 * h <= 0.0
                else:
                    at = cen[:, axis] + 0.5 * h >= ext[axis]
                if np.any(at):
                    pe = cen[at].copy()
                    pe[:, axis] += (h[at] if side else -h[at])
                    b[at] += h[at] * _sin_exact(pe)
        out[t0 * 512:t1 * 512] = b
    return out


def neumann_layer_kind(tiles_sorted: np.ndarray, ext=(1, 1, 1)) -> np.ndarray:
    """Paper Sec. 5.2/5.3 setup: "the outermost layer of cells in the grid [is set] to
    Neumann boundary conditions and all other cells [are] interior cells" (P:L1343,
    P:L1315).  Returns kind u8[N] with the domain-boundary cell layer Neumann."""
    t = np.asarray(tiles_sorted, dtype=np.int64)
    out = np.empty(len(t) * B ** 3, dtype=np.uint8)
    ext = np.asarray(ext, dtype=np.float64)
    for t0 in range(0, len(t), 8192):
        t1 = min(len(t), t0 + 8192)
        cen, h = leaf_cell_geometry(t, t0, t1)
        edge = np.any((cen - 0.5 * h[:, None] <= 0.0) | (cen + 0.5 * h[:, None] >= ext[None, :]), axis=1)
        out[t0 * 512:t1 * 512] = np.where(edge, NEUMANN, FLUID)
    return out


# ---------------------------------------------------------------------------------------
# Cut cells (tank scene) -------------------------------------------------


def face_fraction_marching_squares(phi: np.ndarray, phi_centre: np.ndarray | None = None) -> np.ndarray:
    """Fluid (phi >= 0) area fraction of a square face from its 4 corner samples given in
    cyclic order (0,0),(1,0),(1,1),(0,1).  Edge crossings by linear interpolation; the
    ambiguous saddle is resolved by the sign of the face-centre sample."""
    phi = np.asarray(phi, dtype=np.float64)
    P = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], dtype=np.float64)
    n = phi.shape[0]
    pts = np.zeros((n, 8, 2))
    valid = np.zeros((n, 8), dtype=bool)
    fl = phi >= 0
    for e in range(4):
        a, b = e, (e + 1) % 4
        pts[:, 2 * e] = P[a]
        valid[:, 2 * e] = fl[:, a]
        cross = fl[:, a] != fl[:, b]
        den = phi[:, a] - phi[:, b]
        tt = np.where(cross, phi[:, a] / np.where(den == 0, 1, den), 0.0)
        pts[:, 2 * e + 1] = P[a][None, :] + tt[:, None] * (P[b] - P[a])[None, :]
        valid[:, 2 * e + 1] = cross
    # shoelace over the valid points in walk order: compact valid points to the front
    area = np.zeros(n)
    order_pts = np.where(valid[..., None], pts, np.nan)
    idx = np.argsort(~valid, axis=1, kind="stable")
    cp = np.take_along_axis(order_pts, idx[..., None], axis=1)
    cnt = valid.sum(1)
    for k in range(8):
        k1 = (k + 1)
        p0 = cp[:, k]
        nxt = np.where((k1 < cnt)[:, None], cp[:, min(k1, 7)], cp[:, 0])
        use = k < cnt
        term = p0[:, 0] * nxt[:, 1] - nxt[:, 0] * p0[:, 1]
        area += np.where(use, term, 0.0)
    area = 0.5 * np.abs(area)
    # saddle with solid centre: two separate corner triangles
    sad = (fl[:, 0] == fl[:, 2]) & (fl[:, 1] == fl[:, 3]) & (fl[:, 0] != fl[:, 1])
    if phi_centre is None:
        phi_centre = phi.mean(1)
    split = sad & (phi_centre < 0)
    if np.any(split):
        s = np.where(split)[0]
        tri = np.zeros(len(s))
        for c in range(4):
            isf = fl[s, c]
            nxt, prv = (c + 1) % 4, (c + 3) % 4
            a = phi[s, c] / (phi[s, c] - phi[s, nxt])
            bb = phi[s, c] / (phi[s, c] - phi[s, prv])
            tri += np.where(isf, 0.5 * a * bb, 0.0)
        area[s] = tri
    return np.clip(area, 0.0, 1.0)


def _sphere_phi(p, centre, r):
    c = np.asarray(centre, dtype=np.float64)
    return np.sqrt(((p - c) ** 2).sum(-1)) - r


def tank_fields(tiles_sorted: np.ndarray, ext=(1, 1, 1), centre=(0.5, 0.5, 0.5), radius=0.3,
                beta_jump: float | None = None, chunk_tiles: int = 4096):
    """Static cut-cell projection scene: tank with solid bottom and sides,
    open (Dirichlet) top at y = ext_y, a solid sphere obstacle, unit downward velocity.

    Returns kind u8[N], w f32[6][N], b f32[N] with b_i = h_i^2 (w_{y+} - w_{y-}) for fluid
    cells and 0 elsewhere.  w is 0 on solid tank walls and 1 on the
    open top.  ``radius <= 0`` means no obstacle.  ``beta_jump`` multiplies w by that
    factor inside |x-0.5| < 0.1 (discontinuous-beta variant)."""
    t = np.asarray(tiles_sorted, dtype=np.int64)
    N = len(t) * 512
    kind = np.zeros(N, dtype=np.uint8)
    w = np.zeros((6, N), dtype=np.float32)
    b = np.zeros(N, dtype=np.float32)
    ext = np.asarray(ext, dtype=np.float64)
    # face corner offsets in cell units, per face: fixed axis + cyclic corners over the
    # two other axes
    for t0 in range(0, len(t), chunk_tiles):
        t1 = min(len(t), t0 + chunk_tiles)
        cen, h = leaf_cell_geometry(t, t0, t1)
        sl = slice(t0 * 512, t1 * 512)
        if radius > 0:
            inside = _sphere_phi(cen, centre, radius) < 0
        else:
            inside = np.zeros(len(cen), dtype=bool)
        kind[sl] = np.where(inside, NEUMANN, FLUID)
        for axis in range(3):
            o1, o2 = [a for a in range(3) if a != axis]
            for side in (0, 1):
                f = 2 * axis + side
                pc = cen.copy()
                pc[:, axis] += (side - 0.5) * h
                if radius > 0:
                    phic = _sphere_phi(pc, centre, radius)
                    frac = (phic >= 0).astype(np.float64)
                    # only faces within a half-diagonal of the surface can be cut (SDF is
                    # 1-Lipschitz); others are entirely fluid or solid
                    near = np.abs(phic) <= 0.75 * h
                    if np.any(near):
                        corners = []
                        for (u, v) in ((-1, -1), (1, -1), (1, 1), (-1, 1)):
                            q = pc[near].copy()
                            q[:, o1] += 0.5 * u * h[near]
                            q[:, o2] += 0.5 * v * h[near]
                            corners.append(_sphere_phi(q, centre, radius))
                        phi = np.stack(corners, axis=1)
                        frac[near] = face_fraction_marching_squares(phi, phic[near])
                else:
                    frac = np.ones(len(cen))
                # tank walls: solid except the open top (y+ at y = ext_y)
                lo_wall = pc[:, axis] <= 0.0
                hi_wall = pc[:, axis] >= ext[axis]
                if axis == 1:
                    frac = np.where(lo_wall, 0.0, frac)
                    frac = np.where(hi_wall, 1.0, frac)
                else:
                    frac = np.where(lo_wall | hi_wall, 0.0, frac)
                if beta_jump is not None:
                    frac = np.where(np.abs(cen[:, 0] - 0.5) < 0.1, beta_jump * frac, frac)
                w[f, sl] = frac.astype(np.float32)
        fluid = kind[sl] == FLUID
        bb = (h ** 2) * (w[3, sl].astype(np.float64) - w[2, sl].astype(np.float64))
        b[sl] = np.where(fluid, bb, 0.0).astype(np.float32)
    return kind, w, b


def tank_exact_pressure(centres: np.ndarray, h_top: float, ext_y: float = 1.0) -> np.ndarray:
    """Exact discrete solution of the obstacle-free tank: p = ext_y + h_top/2 - y
    (SURVEY c-9 'Linear exactness'; derivation in DESIGN.md)."""
    return ext_y + 0.5 * h_top - centres[:, 1]
