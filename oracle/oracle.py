"""ctypes wrapper of the fp64 CPU oracle (oracle/octmg_oracle.cpp).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs are the only permitted users.  The product path
(paper_2604_18886_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "octmg_oracle.cpp")
_LIB = os.path.join(_HERE, "liboctmg_oracle.so")

STATUS = {0: "OK", 1: "INVALID", 2: "OVERLAP", 3: "GAP", 4: "NOT_GRADED", 9: "BREAKDOWN", 10: "MAXITER"}


def build_oracle(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["g++", "-O2", "-fopenmp", "-std=c++17", "-shared", "-fPIC",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build_oracle())
        P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        _lib.orc_create.restype = P
        _lib.orc_create.argtypes = [C.c_int, P, P, P, I64, P]
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_destroy.argtypes = [P]
        _lib.orc_info.argtypes = [P, P]
        _lib.orc_tables.argtypes = [P, P, P, P, P]
        _lib.orc_setup.restype = I32
        _lib.orc_setup.argtypes = [P, P, P, D, I32]
        _lib.orc_coefs.argtypes = [P, P]
        _lib.orc_setup_gmg.restype = I32
        _lib.orc_setup_gmg.argtypes = [P, P, P]
        _lib.orc_coefs_cycle.argtypes = [P, P]
        _lib.orc_ghost_coef.restype = I32
        _lib.orc_ghost_coef.argtypes = [P, I32, I64, I64, I64, P]
        _lib.orc_apply.argtypes = [P, P, P]
        _lib.orc_apply_level.argtypes = [P, I32, P, P]
        _lib.orc_rbgs_pass.argtypes = [P, I32, I32, P, P]
        _lib.orc_vcycle.argtypes = [P, P, P, P, I32]
        _lib.orc_pcg.restype = I32
        _lib.orc_pcg.argtypes = [P, P, I32, P, P, D, I32, I32, P, P, P, P, I32]
        _lib.orc_divergence.argtypes = [P, P, P, P]
        _lib.orc_subtract_gradient.argtypes = [P, P, P, P]
        _lib.orc_face_fluxes.argtypes = [P, I32, I32, P, P]
        _lib.orc_face_fraction.restype = D
        _lib.orc_face_fraction.argtypes = [P, D]
        _lib.orc_tank_fields.argtypes = [P, I64, I32, P, P, D, P, P, P]
        _lib.orc_leaf_diag.argtypes = [P, P]
        _lib.orc_direct_coarsest.argtypes = [P, P, P]
        _lib.orc_set_check_eq14.argtypes = [P, I32]
        _lib.orc_eq14.argtypes = [P, P]
        _lib.orc_mg_solve.restype = I32
        _lib.orc_mg_solve.argtypes = [P, P, I32, P, P, D, I32, I32, P, P, P, P, I32]
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def face_fraction(phi4, phi_centre):
    """Fluid (phi >= 0) area fraction of a unit face from corner samples (cyclic order)."""
    a = np.ascontiguousarray(phi4, dtype=np.float64)
    return lib().orc_face_fraction(_p(a), float(phi_centre))


def tank_fields(tiles_sorted, ext=(1, 1, 1), centre=(0.5, 0.5, 0.5), radius=0.3, B: int = 8):
    """Oracle cut-cell fields of the tank scene: kind u8[N], w f32[6][N], b f32[N]."""
    t = np.ascontiguousarray(np.asarray(tiles_sorted, dtype=np.int32).reshape(-1, 4))
    N = len(t) * B ** 3
    kind = np.zeros(N, dtype=np.uint8)
    w = np.zeros((6, N), dtype=np.float32)
    b = np.zeros(N, dtype=np.float32)
    e = np.asarray(ext, dtype=np.float64)
    c = np.asarray(centre, dtype=np.float64)
    lib().orc_tank_fields(_p(t), len(t), B, _p(e), _p(c), float(radius), _p(kind), _p(w), _p(b))
    return kind, w, b


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = STATUS.get(status, status)


def mg_params(alpha=2.0, beta=2.0, mu=1, nu_pre=2, nu_post=2, nu_coarsest=10, coarsest="smooth"):
    """coarsest: 'smooth' (nu_coarsest RBGS iterations) or 'direct' (Alg. 4 line 4)."""
    c = {"smooth": 0, "direct": 1}[coarsest]
    return np.array([alpha, beta, mu, nu_pre, nu_post, nu_coarsest, c], dtype=np.float64)


class Oracle:
    """One graded tile octree plus (after setup) its coefficient hierarchy, in fp64."""

    def __init__(self, tiles, ext=(1, 1, 1), wall_bc=(1, 1, 1, 1, 1, 1), B: int = 8):
        L = lib()
        t = np.ascontiguousarray(np.asarray(tiles, dtype=np.int32).reshape(-1, 4))
        e = np.asarray(ext, dtype=np.int32)
        w = np.asarray(wall_bc, dtype=np.int32)
        st = np.zeros(1, dtype=np.int32)
        self._h = L.orc_create(B, _p(e), _p(w), _p(t), len(t), _p(st))
        if not self._h:
            raise OracleError(int(st[0]), L.orc_last_error().decode())
        self.B = B
        self.B3 = B ** 3
        self.ext = tuple(ext)
        self.wall_bc = tuple(wall_bc)
        info = np.zeros(4, dtype=np.int64)
        L.orc_info(self._h, _p(np.zeros(4 + 4 * 32, dtype=np.int64)))
        buf = np.zeros(4 + 4 * 32, dtype=np.int64)
        L.orc_info(self._h, _p(buf))
        self.L, self.NL, self.NI, self.T = (int(v) for v in buf[:4])
        seg = buf[4:4 + 4 * (self.L + 1)].reshape(-1, 4)
        self.leaf_begin, self.leaf_count = seg[:, 0].copy(), seg[:, 1].copy()
        self.inner_begin, self.inner_count = seg[:, 2].copy(), seg[:, 3].copy()
        self.N = self.NL * self.B3
        del info

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().orc_destroy(self._h)
        except Exception:
            pass

    # ---- tree --------------------------------------------------------------------
    def tables(self):
        T, NI = self.T, self.NI
        tiles = np.zeros((T, 4), dtype=np.int32)
        nbr = np.zeros((T, 6), dtype=np.int32)
        parent = np.zeros(T, dtype=np.int32)
        child = np.zeros((max(NI, 1), 8), dtype=np.int32)
        lib().orc_tables(self._h, _p(tiles), _p(nbr), _p(parent), _p(child))
        return dict(tiles=tiles, nbr=nbr, parent=parent, child=child[:NI])

    # ---- setup ---------------------------------------------------------------------
    def setup(self, kind=None, w=None, alpha: float = 2.0, coarsen_literal: bool = False):
        N = self.N
        k = np.zeros(N, dtype=np.uint8) if kind is None else np.ascontiguousarray(kind, dtype=np.uint8)
        assert k.size == N
        if w is not None:
            wv = np.ascontiguousarray(np.asarray(w, dtype=np.float32).reshape(6, N))
            st = lib().orc_setup(self._h, _p(k), _p(wv), alpha, int(coarsen_literal))
        else:
            st = lib().orc_setup(self._h, _p(k), None, alpha, int(coarsen_literal))
        if st:
            raise OracleError(st, lib().orc_last_error().decode())
        self.alpha = alpha
        return self

    def setup_gmg(self, kind_inner=None, w_inner=None):
        """GMG comparison mode: the cycle's inner-cell records assembled
        by Eq. 3 from the inner cells' own kinds / face weights (inner-tile order; None = all fluid,
        w = 1) instead of Alg. 3; the composite operator is unchanged.  Call after setup()."""
        NI3 = self.NI * self.B3
        k = np.zeros(NI3, dtype=np.uint8) if kind_inner is None else np.ascontiguousarray(kind_inner, dtype=np.uint8)
        assert k.size == NI3
        if w_inner is not None:
            wv = np.ascontiguousarray(np.asarray(w_inner, dtype=np.float32).reshape(6, NI3))
            st = lib().orc_setup_gmg(self._h, _p(k), _p(wv))
        else:
            st = lib().orc_setup_gmg(self._h, _p(k), None)
        if st:
            raise OracleError(st, lib().orc_last_error().decode())
        return self

    def coefs(self):
        out = np.zeros((self.T * self.B3, 4), dtype=np.float64)
        lib().orc_coefs(self._h, _p(out))
        return out

    def coefs_cycle(self):
        """The records the cycle uses (= coefs() unless GMG mode)."""
        out = np.zeros((self.T * self.B3, 4), dtype=np.float64)
        lib().orc_coefs_cycle(self._h, _p(out))
        return out

    def coefs_diag_leaf(self):
        """The diagonal c of the leaf cells (c == 0: inactive), without the full export."""
        out = np.zeros(self.N)
        lib().orc_leaf_diag(self._h, _p(out))
        return out

    def ghost_coef(self, level, X, Y, Z):
        out = np.zeros(3)
        ok = lib().orc_ghost_coef(self._h, level, X, Y, Z, _p(out))
        return out if ok else None

    # ---- operators -------------------------------------------------------------------
    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.N)
        lib().orc_apply(self._h, _p(x), _p(y))
        return y

    def apply_level(self, level, u_all):
        u = np.ascontiguousarray(u_all, dtype=np.float64)
        y = np.zeros(self.T * self.B3)
        lib().orc_apply_level(self._h, level, _p(u), _p(y))
        return y

    def direct_coarsest(self, b_all, u_all):
        """Alg. 4 line 4 'or direct solve': u^0 = M0 b^0 on the level-0 cells (all-tile arrays)."""
        u = np.array(u_all, dtype=np.float64, copy=True)
        b = np.ascontiguousarray(b_all, dtype=np.float64)
        lib().orc_direct_coarsest(self._h, _p(b), _p(u))
        return u

    def rbgs_pass(self, level, colour, u_all, b_all):
        u = np.array(u_all, dtype=np.float64, copy=True)
        b = np.ascontiguousarray(b_all, dtype=np.float64)
        lib().orc_rbgs_pass(self._h, level, colour, _p(u), _p(b))
        return u

    def vcycle(self, r, form: str = "fas", **mg):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros(self.N)
        prm = mg_params(**mg)
        lib().orc_vcycle(self._h, _p(prm), _p(r), _p(z), 1 if form == "fas" else 0)
        return z

    def pcg(self, b, rtol=1e-6, max_iters=200, nullspace=-1, precond="fas", hcap=512, **mg):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.N)
        prm = mg_params(**mg)
        it = np.zeros(1, dtype=np.int32)
        rr = np.zeros(1)
        bn = np.zeros(1)
        hist = np.zeros(hcap)
        pk = {"identity": 0, "fas": 1, "alg2": 2}[precond]
        st = lib().orc_pcg(self._h, _p(prm), pk, _p(b), _p(x), rtol, max_iters, nullspace,
                           _p(it), _p(rr), _p(bn), _p(hist), hcap)
        n = int(it[0])
        return dict(x=x, iters=n, rel_residual=float(rr[0]), bnorm=float(bn[0]),
                    status=STATUS.get(st, st), history=hist[:min(n, hcap)].copy())

    def mg_solve(self, b, rtol=1e-6, max_iters=200, nullspace=-1, form="fas", hcap=512, **mg):
        """Standalone multigrid x += M(b - A x) (use beta = 1)."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.N)
        prm = mg_params(**mg)
        it = np.zeros(1, dtype=np.int32)
        rr = np.zeros(1)
        bn = np.zeros(1)
        hist = np.zeros(hcap)
        st = lib().orc_mg_solve(self._h, _p(prm), 1 if form == "fas" else 0, _p(b), _p(x), rtol, max_iters,
                                nullspace, _p(it), _p(rr), _p(bn), _p(hist), hcap)
        n = int(it[0])
        return dict(x=x, iters=n, rel_residual=float(rr[0]), bnorm=float(bn[0]),
                    status=STATUS.get(st, st), history=hist[:min(n, hcap)].copy())

    def eq14_check(self, on: bool = True):
        """Enable (and reset) the Eq. 14 check inside the FAS cycle."""
        lib().orc_set_check_eq14(self._h, int(on))

    def eq14_result(self):
        """(max |mean of active children - coarse value| after a prolongation, max |coarse value|)."""
        out = np.zeros(2)
        lib().orc_eq14(self._h, _p(out))
        return float(out[0]), float(out[1])

    # ---- projection ---------------------------------------------------
    def divergence(self, frac, u6):
        """b = -(net outflow) of the face velocities u6 (6, N) with fluid fractions frac (6, N)."""
        fr = np.ascontiguousarray(np.asarray(frac, dtype=np.float32).reshape(6, self.N))
        uu = np.ascontiguousarray(np.asarray(u6, dtype=np.float64).reshape(6, self.N))
        b = np.zeros(self.N)
        lib().orc_divergence(self._h, _p(fr), _p(uu), _p(b))
        return b

    def subtract_gradient(self, frac, p, u6):
        """u6 - G p (fp64 copy of u6), the projection step consistent with the operator."""
        fr = np.ascontiguousarray(np.asarray(frac, dtype=np.float32).reshape(6, self.N))
        pp = np.ascontiguousarray(p, dtype=np.float64)
        uu = np.array(u6, dtype=np.float64, copy=True).reshape(6, self.N)
        lib().orc_subtract_gradient(self._h, _p(fr), _p(pp), _p(uu))
        return uu

    def face_fluxes(self, t, off, p):
        pp = np.ascontiguousarray(p, dtype=np.float64)
        F = np.zeros(6)
        lib().orc_face_fluxes(self._h, int(t), int(off), _p(pp), _p(F))
        return F

    # ---- geometry helpers (plain index arithmetic on the exported tile list) -----------
    def cell_coords(self):
        """Global level coords (X,Y,Z) and level for every cell of every tile (all-tile
        order)."""
        t = self.tables()["tiles"].astype(np.int64)
        B = self.B
        off = np.arange(self.B3)
        lx, ly, lz = off % B, (off // B) % B, off // (B * B)
        X = (t[:, 1:2] * B + lx[None, :]).ravel()
        Y = (t[:, 2:3] * B + ly[None, :]).ravel()
        Z = (t[:, 3:4] * B + lz[None, :]).ravel()
        lev = np.repeat(t[:, 0], self.B3)
        return X, Y, Z, lev

    def leaf_centres(self):
        X, Y, Z, lev = self.cell_coords()
        n = self.N
        h = np.ldexp(1.0, -lev[:n]) / self.B
        cen = np.stack([(X[:n] + 0.5) * h, (Y[:n] + 0.5) * h, (Z[:n] + 0.5) * h], axis=1)
        return cen, h
