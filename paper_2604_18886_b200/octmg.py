"""Thin ctypes binding of the C ABI in include/octmg.h (argument marshalling only).

Every step of the solver runs in liboctmg.so (hand-written CUDA for sm_100a).  There is
no CPU fallback: if the shared object is missing, loading fails loudly.  PyTorch supplies
device memory (tensor.data_ptr()) and the current CUDA stream.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._build import LIB

STATUS = {0: "OK", 1: "INVALID", 2: "OVERLAP", 3: "GAP", 4: "NOT_GRADED", 5: "OOM", 6: "CUDA",
          7: "NCCL", 8: "NONFINITE", 9: "BREAKDOWN", 10: "MAXITER"}
MAX_LEVELS = 16


class OctmgError(RuntimeError):
    def __init__(self, status, msg):
        self.status = STATUS.get(status, status)
        super().__init__(f"octmg {self.status}: {msg}")


class TreeDesc(C.Structure):
    _fields_ = [("ext", C.c_int32 * 3), ("wall_bc", C.c_uint8 * 6), ("grade_repair", C.c_int32),
                ("rank", C.c_int32), ("nranks", C.c_int32), ("nccl_comm", C.c_void_p)]


class TreeInfo(C.Structure):
    _fields_ = [("levels", C.c_int32), ("n_leaf_tiles", C.c_int32), ("n_inner_tiles", C.c_int32),
                ("n_leaf_cells", C.c_int64),
                ("leaf_begin", C.c_int32 * MAX_LEVELS), ("leaf_count", C.c_int32 * MAX_LEVELS),
                ("inner_begin", C.c_int32 * MAX_LEVELS), ("inner_count", C.c_int32 * MAX_LEVELS),
                ("n_ghost_layers", C.c_int32)]


class MGParams(C.Structure):
    _fields_ = [("alpha", C.c_float), ("beta_overshoot", C.c_float), ("mu", C.c_int32), ("nu_pre", C.c_int32),
                ("nu_post", C.c_int32), ("nu_coarsest", C.c_int32), ("form", C.c_int32),
                ("coarsen_literal", C.c_int32), ("coarsest", C.c_int32), ("reserved0", C.c_int32),
                ("gather_below_cells", C.c_int64)]


class SolveParams(C.Structure):
    _fields_ = [("rtol", C.c_double), ("max_iters", C.c_int32), ("nullspace", C.c_int32)]


class SolveReport(C.Structure):
    _fields_ = [("iters", C.c_int32), ("converged", C.c_int32), ("rel_residual", C.c_double),
                ("bnorm", C.c_double), ("status", C.c_int32), ("history", C.POINTER(C.c_double)),
                ("history_cap", C.c_int32), ("kernel_launches", C.c_int64), ("history_len", C.c_int32),
                ("device_loop", C.c_int32)]


EXPORT_TILES, EXPORT_NBR, EXPORT_PARENT, EXPORT_CHILD = 0, 1, 2, 3

# every symbol include/octmg.h declares (checked by tests/test_abi.py)
ABI_SYMBOLS = ["octmg_last_error", "octmg_version", "octmg_build_tree", "octmg_tree_info_get",
               "octmg_tree_export", "octmg_setup_hierarchy", "octmg_hier_export_coefs", "octmg_apply",
               "octmg_vcycle", "octmg_pcg_solve", "octmg_profile_enable", "octmg_profile_read",
               "octmg_setup_hierarchy_loopback", "octmg_partition_info", "octmg_nccl_unique_id",
               "octmg_nccl_comm_init", "octmg_nccl_comm_destroy", "octmg_partition_plan_host",
               "octmg_hier_destroy", "octmg_tree_destroy", "octmg_mg_solve", "octmg_tank_fields",
               "octmg_divergence", "octmg_subtract_gradient",
               "octmg_grade_repair_host", "octmg_set_allocator", "octmg_profile_read_level",
               "octmg_band_tiles", "octmg_setup_hierarchy_gmg", "octmg_tank_fields_inner",
               "octmg_hier_export_cycle_coefs"]

_lib = None


def lib():
    """Load liboctmg.so (built by __graft_entry__.build()); raise if it is absent."""
    global _lib
    if _lib is None:
        path = os.environ.get("OCTMG_LIB_AB") or LIB  # (tools/: A/B of two builds of the library)
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
        L = C.CDLL(path)
        P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
        L.octmg_last_error.restype = C.c_char_p
        L.octmg_version.restype = C.c_char_p
        L.octmg_build_tree.argtypes = [C.POINTER(TreeDesc), P, I64, P, C.POINTER(P)]
        L.octmg_tree_info_get.argtypes = [P, C.POINTER(TreeInfo)]
        L.octmg_tree_export.argtypes = [P, I32, P, C.c_size_t]
        L.octmg_setup_hierarchy.argtypes = [P, P, P, P, C.POINTER(MGParams), P, C.POINTER(P)]
        L.octmg_hier_export_coefs.argtypes = [P, P, C.c_size_t]
        L.octmg_apply.argtypes = [P, P, P, P]
        L.octmg_vcycle.argtypes = [P, P, P, P]
        L.octmg_pcg_solve.argtypes = [P, P, P, C.POINTER(SolveParams), C.POINTER(SolveReport), P]
        L.octmg_mg_solve.argtypes = [P, P, P, C.POINTER(SolveParams), C.POINTER(SolveReport), P]
        L.octmg_mg_solve.restype = C.c_int
        L.octmg_tank_fields.argtypes = [P, P, C.c_double, P, P, P, P]
        L.octmg_tank_fields.restype = C.c_int
        L.octmg_set_allocator.argtypes = [P, P, P]
        L.octmg_set_allocator.restype = C.c_int
        L.octmg_grade_repair_host.argtypes = [P, I64, P, P, I64, P]
        L.octmg_grade_repair_host.restype = C.c_int
        L.octmg_divergence.argtypes = [P, P, P, P, P]
        L.octmg_divergence.restype = C.c_int
        L.octmg_subtract_gradient.argtypes = [P, P, P, P, P, P, P]
        L.octmg_subtract_gradient.restype = C.c_int
        L.octmg_profile_enable.argtypes = [P, I32]
        L.octmg_profile_read.argtypes = [P, P, P, P, P, I32, C.POINTER(I32)]
        L.octmg_profile_read_level.argtypes = [P, I32, P, P, P, I32, C.POINTER(I32)]
        L.octmg_profile_read_level.restype = C.c_int
        L.octmg_band_tiles.argtypes = [P, I32, I32, P, C.c_double, I32, P, I64, P, P]
        L.octmg_band_tiles.restype = C.c_int
        L.octmg_setup_hierarchy_loopback.argtypes = [P, I32, P, P, P, C.POINTER(MGParams), P, C.POINTER(P)]
        L.octmg_partition_info.argtypes = [P, I32, P, P, P, P, P]
        L.octmg_nccl_unique_id.argtypes = [P]
        L.octmg_nccl_comm_init.argtypes = [I32, I32, P, C.POINTER(P)]
        L.octmg_nccl_comm_destroy.argtypes = [P]
        L.octmg_nccl_comm_destroy.restype = None
        L.octmg_hier_destroy.argtypes = [P]
        L.octmg_tree_destroy.argtypes = [P]
        L.octmg_partition_plan_host.argtypes = [P, P, P, P, I32, I32, I32, P, I32, P, P, P, P, I64, I64]
        L.octmg_setup_hierarchy_gmg.argtypes = [P, P, P, P, P, P, P, C.POINTER(MGParams), P, C.POINTER(P)]
        L.octmg_setup_hierarchy_gmg.restype = C.c_int
        L.octmg_tank_fields_inner.argtypes = [P, P, C.c_double, P, P, P]
        L.octmg_tank_fields_inner.restype = C.c_int
        L.octmg_hier_export_cycle_coefs.argtypes = [P, P, C.c_size_t]
        L.octmg_hier_export_cycle_coefs.restype = C.c_int
        for name in ABI_SYMBOLS[2:16] + ["octmg_partition_plan_host"]:
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(st):
    if st != 0:
        raise OctmgError(st, lib().octmg_last_error().decode())


def _stream(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(stream)


def _ptr(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


def version() -> str:
    return lib().octmg_version().decode()


class NcclComm:
    """NCCL communicator for an nranks-GPU job, bootstrapped through torch.distributed
    (rank 0's unique id is broadcast over the default process group)."""

    def __init__(self, rank: int, nranks: int):
        import torch.distributed as dist
        buf = (C.c_char * 128)()
        if rank == 0:
            _check(lib().octmg_nccl_unique_id(C.cast(buf, C.c_void_p)))
        obj = [bytes(buf)] if rank == 0 else [None]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_char * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        _check(lib().octmg_nccl_comm_init(rank, nranks, C.cast(uid, C.c_void_p), C.byref(h)))
        self.handle = h
        self.rank, self.nranks = rank, nranks

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                lib().octmg_nccl_comm_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


class Tree:
    """octmg_build_tree: graded leaf tiles (host int array (n,4): level,i,j,k)."""

    def __init__(self, tiles, ext=(1, 1, 1), wall_bc=(1, 1, 1, 1, 1, 1), stream=None, comm: "NcclComm" = None,
                 grade_repair: bool = False):
        t = np.ascontiguousarray(np.asarray(tiles, dtype=np.int32).reshape(-1, 4))
        d = TreeDesc()
        for a in range(3):
            d.ext[a] = int(ext[a])
        for f in range(6):
            d.wall_bc[f] = int(wall_bc[f])
        d.grade_repair = 1 if grade_repair else 0
        if comm is None:
            d.rank, d.nranks, d.nccl_comm = 0, 1, None
        else:
            d.rank, d.nranks, d.nccl_comm = comm.rank, comm.nranks, comm.handle
        self.comm = comm
        h = C.c_void_p()
        _check(lib().octmg_build_tree(C.byref(d), t.ctypes.data_as(C.c_void_p), len(t), _stream(stream),
                                      C.byref(h)))
        self._h = h
        info = TreeInfo()
        _check(lib().octmg_tree_info_get(self._h, C.byref(info)))
        self.levels = info.levels
        self.L = info.levels - 1
        self.NL = info.n_leaf_tiles
        self.NI = info.n_inner_tiles
        self.T = self.NL + self.NI
        self.N = int(info.n_leaf_cells)
        self.leaf_begin = np.array(info.leaf_begin[:self.levels])
        self.leaf_count = np.array(info.leaf_count[:self.levels])
        self.inner_begin = np.array(info.inner_begin[:self.levels])
        self.inner_count = np.array(info.inner_count[:self.levels])
        self.n_ghost_layers = info.n_ghost_layers

    def export(self, what):
        shape = {EXPORT_TILES: (self.T, 4), EXPORT_NBR: (self.T, 6), EXPORT_PARENT: (self.T,),
                 EXPORT_CHILD: (self.NI, 8)}[what]
        out = np.zeros(shape, dtype=np.int32)
        _check(lib().octmg_tree_export(self._h, what, out.ctypes.data_as(C.c_void_p), out.nbytes))
        return out

    def tables(self):
        return dict(tiles=self.export(EXPORT_TILES), nbr=self.export(EXPORT_NBR),
                    parent=self.export(EXPORT_PARENT), child=self.export(EXPORT_CHILD))

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().octmg_tree_destroy(self._h)
                self._h = None
        except Exception:
            pass


def tank_fields(tree, centre=(0.5, 0.5, 0.5), radius=0.3, stream=None):
    """octmg_tank_fields on the device: (kind u8[N], face_frac f32[6][N], b f32[N]) torch tensors."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    N = tree.N
    kind = torch.empty(N, dtype=torch.uint8, device=dev)
    frac = torch.empty((6, N), dtype=torch.float32, device=dev)
    b = torch.empty(N, dtype=torch.float32, device=dev)
    c = (C.c_double * 3)(*centre)
    _check(lib().octmg_tank_fields(tree._h, C.cast(c, C.c_void_p), float(radius), _ptr(kind), _ptr(frac), _ptr(b),
                                   _stream(stream)))
    return kind, frac, b


def tank_fields_inner(tree, centre=(0.5, 0.5, 0.5), radius=0.3, stream=None):
    """octmg_tank_fields_inner: the inner cells' (kind u8[NI*512], face_frac f32[6][NI*512])."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    n = tree.NI * 512
    kind = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    frac = torch.empty((6, max(n, 1)), dtype=torch.float32, device=dev)
    c = (C.c_double * 3)(*centre)
    _check(lib().octmg_tank_fields_inner(tree._h, C.cast(c, C.c_void_p), float(radius), _ptr(kind), _ptr(frac),
                                         _stream(stream)))
    return kind[:n], frac[:, :n]


class Hierarchy:
    """octmg_setup_hierarchy + the solver calls.  Device tensors (torch, cuda) in and out.
    gmg=(kind_inner, face_beta_inner, face_frac_inner): the GMG comparison mode
    (octmg_setup_hierarchy_gmg; the beta / frac entries may be None)."""

    def __init__(self, tree: Tree, kind, face_beta=None, face_frac=None, alpha=2.0, beta=2.0, mu=1,
                 nu_pre=2, nu_post=2, nu_coarsest=10, stream=None, loopback_parts: int = 0, form="fas",
                 coarsen_literal=False, coarsest="smooth", gather_below_cells=0, gmg=None):
        self.tree = tree
        p = MGParams(alpha, beta, mu, nu_pre, nu_post, nu_coarsest, {"fas": 0, "alg2": 1}[form],
                     int(coarsen_literal), {"smooth": 0, "direct": 1}[coarsest], 0, int(gather_below_cells))
        h = C.c_void_p()
        if gmg is not None:
            ki, bi, fi = gmg
            _check(lib().octmg_setup_hierarchy_gmg(tree._h, _ptr(kind), _ptr(face_beta), _ptr(face_frac), _ptr(ki),
                                                   _ptr(bi), _ptr(fi), C.byref(p), _stream(stream), C.byref(h)))
        elif loopback_parts:
            _check(lib().octmg_setup_hierarchy_loopback(tree._h, loopback_parts, _ptr(kind), _ptr(face_beta),
                                                        _ptr(face_frac), C.byref(p), _stream(stream), C.byref(h)))
        else:
            _check(lib().octmg_setup_hierarchy(tree._h, _ptr(kind), _ptr(face_beta), _ptr(face_frac), C.byref(p),
                                               _stream(stream), C.byref(h)))
        self._h = h
        self.N = tree.N
        self.parts = max(1, loopback_parts)

    def partition(self, part: int = 0):
        """(lg, rank, nranks, owned leaf tiles per level as (begin, count) arrays)"""
        lg, rk, nr = C.c_int32(), C.c_int32(), C.c_int32()
        b = (C.c_int32 * MAX_LEVELS)()
        c = (C.c_int32 * MAX_LEVELS)()
        _check(lib().octmg_partition_info(self._h, part, C.byref(lg), C.byref(rk), C.byref(nr),
                                          C.cast(b, C.c_void_p), C.cast(c, C.c_void_p)))
        L = self.tree.levels
        return lg.value, rk.value, nr.value, np.array(b[:L]), np.array(c[:L])

    def apply(self, x, y, stream=None):
        _check(lib().octmg_apply(self._h, _ptr(x), _ptr(y), _stream(stream)))

    def vcycle(self, b, u, stream=None):
        _check(lib().octmg_vcycle(self._h, _ptr(b), _ptr(u), _stream(stream)))

    def pcg_solve(self, b, x, rtol=1e-6, max_iters=200, nullspace=-1, history_cap=256, stream=None,
                  raise_on_error=True):
        return self._solve(lib().octmg_pcg_solve, b, x, rtol, max_iters, nullspace, history_cap, stream,
                           raise_on_error)

    def mg_solve(self, b, x, rtol=1e-6, max_iters=200, nullspace=-1, history_cap=256, stream=None,
                 raise_on_error=True):
        """octmg_mg_solve: multigrid as a standalone solver (set up the hierarchy with beta=1)."""
        return self._solve(lib().octmg_mg_solve, b, x, rtol, max_iters, nullspace, history_cap, stream,
                           raise_on_error)

    def _solve(self, fn, b, x, rtol, max_iters, nullspace, history_cap, stream, raise_on_error):
        prm = SolveParams(rtol, max_iters, nullspace)
        hist = (C.c_double * max(history_cap, 1))()
        rep = SolveReport()
        rep.history = C.cast(hist, C.POINTER(C.c_double))
        rep.history_cap = history_cap
        st = fn(self._h, _ptr(b), _ptr(x), C.byref(prm), C.byref(rep), _stream(stream))
        out = dict(iters=rep.iters, converged=bool(rep.converged), rel_residual=rep.rel_residual,
                   bnorm=rep.bnorm, status=STATUS.get(st, st), kernel_launches=int(rep.kernel_launches),
                   history=np.array(hist[:rep.history_len]), device_loop=bool(rep.device_loop))
        if raise_on_error and st not in (0, 10):
            _check(st)
        return out

    def divergence(self, u6, b, face_frac=None, stream=None):
        """octmg_divergence: b = -(net outflow of the face velocities u6 (6, N))."""
        _check(lib().octmg_divergence(self._h, _ptr(face_frac), _ptr(u6), _ptr(b), _stream(stream)))

    def subtract_gradient(self, p, u6, kind, face_beta=None, face_frac=None, stream=None):
        """octmg_subtract_gradient: u6 -= G p in place (consistent with the operator)."""
        _check(lib().octmg_subtract_gradient(self._h, _ptr(kind), _ptr(face_beta), _ptr(face_frac), _ptr(p),
                                             _ptr(u6), _stream(stream)))

    def export_coefs(self):
        out = np.zeros((self.tree.T * 512, 4), dtype=np.float32)
        _check(lib().octmg_hier_export_coefs(self._h, out.ctypes.data_as(C.c_void_p), out.nbytes))
        return out

    def export_cycle_coefs(self):
        out = np.zeros((self.tree.T * 512, 4), dtype=np.float32)
        _check(lib().octmg_hier_export_cycle_coefs(self._h, out.ctypes.data_as(C.c_void_p), out.nbytes))
        return out

    def profile(self, on: bool):
        _check(lib().octmg_profile_enable(self._h, 1 if on else 0))

    def profile_read(self):
        cap = 32
        names = (C.c_char_p * cap)()
        ms = (C.c_double * cap)()
        cnt = (C.c_int64 * cap)()
        byt = (C.c_double * cap)()
        n = C.c_int32()
        _check(lib().octmg_profile_read(self._h, C.cast(names, C.c_void_p), C.cast(ms, C.c_void_p),
                                        C.cast(cnt, C.c_void_p), C.cast(byt, C.c_void_p), cap, C.byref(n)))
        return {names[k].decode(): dict(ms=ms[k], launches=int(cnt[k]), bytes=byt[k]) for k in range(n.value)}

    def profile_read_levels(self, levels):
        """{level: {class: dict(ms, launches, bytes)}} of the multigrid work per level."""
        cap = 32
        names = (C.c_char_p * cap)()
        n = C.c_int32()
        _check(lib().octmg_profile_read(self._h, C.cast(names, C.c_void_p), None, None, None, cap, C.byref(n)))
        out = {}
        for lv in levels:
            ms = (C.c_double * cap)()
            cnt = (C.c_int64 * cap)()
            byt = (C.c_double * cap)()
            _check(lib().octmg_profile_read_level(self._h, lv, C.cast(ms, C.c_void_p), C.cast(cnt, C.c_void_p),
                                                  C.cast(byt, C.c_void_p), cap, C.byref(n)))
            out[lv] = {names[k].decode(): dict(ms=ms[k], launches=int(cnt[k]), bytes=byt[k])
                       for k in range(n.value) if cnt[k]}
        return out

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().octmg_hier_destroy(self._h)
                self._h = None
        except Exception:
            pass


_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)
_allocator_refs = []  # keep the ctypes callbacks alive


def set_allocator(alloc=None, release=None):
    """octmg_set_allocator with Python callables alloc(nbytes) -> int and release(ptr);
    None, None restores cudaMalloc."""
    if alloc is None:
        _check(lib().octmg_set_allocator(None, None, None))
        return
    fa = _ALLOC_FN(lambda n, stream, ctx: alloc(int(n)) or None)
    ff = _FREE_FN(lambda p, stream, ctx: release(int(p)))
    _allocator_refs.append((fa, ff))
    _check(lib().octmg_set_allocator(C.cast(fa, C.c_void_p), C.cast(ff, C.c_void_p), None))


def use_torch_allocator():
    """Draw the library's device buffers from PyTorch's caching allocator."""
    import torch

    def alloc(n):
        try:
            return torch.cuda.caching_allocator_alloc(n)
        except RuntimeError:
            return 0

    set_allocator(alloc, torch.cuda.caching_allocator_delete)


def grade_repair_host(tiles, ext=(1, 1, 1)):
    """octmg_grade_repair_host: the least 2:1-graded refinement of a leaf-tile list (host, no GPU)."""
    t = np.ascontiguousarray(np.asarray(tiles, dtype=np.int32).reshape(-1, 4))
    e = np.asarray(ext, dtype=np.int32)
    n_out = C.c_int64()
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    cap = 8 * len(t) + 64
    while True:
        out = np.zeros((cap, 4), dtype=np.int32)
        st = lib().octmg_grade_repair_host(vp(t), len(t), vp(e), vp(out), cap, C.byref(n_out))
        if st == 0:
            return out[:n_out.value].copy()
        if n_out.value > cap:
            cap = n_out.value
            continue
        _check(st)


def band_tiles(l0, extra, centre=(0.5, 0.5, 0.5), radius=0.25, ext=(1, 1, 1), grade_repair=True, stream=None):
    """octmg_band_tiles: the narrow-band leaf tiles (n, 4) int32 (level, i, j, k), computed on
    the device (unspecified order); centre / radius in level-0 tile units."""
    e = (C.c_int32 * 3)(*ext)
    c = (C.c_double * 3)(*centre)
    n = C.c_int64()
    _check(lib().octmg_band_tiles(C.cast(e, C.c_void_p), int(l0), int(extra), C.cast(c, C.c_void_p), float(radius),
                                  1 if grade_repair else 0, None, 0, C.byref(n), _stream(stream)))
    out = np.zeros((n.value, 4), dtype=np.int32)
    _check(lib().octmg_band_tiles(C.cast(e, C.c_void_p), int(l0), int(extra), C.cast(c, C.c_void_p), float(radius),
                                  1 if grade_repair else 0, out.ctypes.data_as(C.c_void_p), n.value, C.byref(n),
                                  _stream(stream)))
    return out


def partition_plan_host(tables, L, NL, NI, level_counts, nranks, gather_below_cells=0):
    """octmg_partition_plan_host on host tables (no GPU): (lg, owner[T], items) where items is
    a dict (level, from, to) -> int32 array (n, 2) of (tile, kind)."""
    T = NL + NI
    t4 = np.ascontiguousarray(tables["tiles"], dtype=np.int32)
    nb = np.ascontiguousarray(tables["nbr"], dtype=np.int32)
    par = np.ascontiguousarray(tables["parent"], dtype=np.int32)
    ch = np.ascontiguousarray(tables["child"], dtype=np.int32).reshape(-1)
    if ch.size == 0:
        ch = np.zeros(8, dtype=np.int32)
    lcnt = np.ascontiguousarray(level_counts, dtype=np.int32)
    lg = C.c_int32()
    owner = np.zeros(T, dtype=np.int32)
    nitems = np.zeros((L + 1) * nranks * nranks, dtype=np.int32)
    cap = 64 * T + 1024
    items = np.zeros(2 * cap, dtype=np.int32)
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    _check(lib().octmg_partition_plan_host(vp(t4), vp(nb), vp(par), vp(ch), NL, NI, L, vp(lcnt), nranks,
                                           C.byref(lg), vp(owner), vp(nitems), vp(items), cap,
                                           int(gather_below_cells)))
    out, k = {}, 0
    for l in range(L + 1):
        for a in range(nranks):
            for b in range(nranks):
                n = int(nitems[(l * nranks + a) * nranks + b])
                out[(l, a, b)] = items[2 * k:2 * (k + n)].reshape(n, 2).copy()
                k += n
    return lg.value, owner, out


# C-ABI names as module-level functions (same names as include/octmg.h)
def octmg_build_tree(tiles, ext=(1, 1, 1), wall_bc=(1, 1, 1, 1, 1, 1), stream=None) -> Tree:
    return Tree(tiles, ext, wall_bc, stream)


def octmg_setup_hierarchy(tree, kind, face_beta=None, face_frac=None, stream=None, **mg) -> Hierarchy:
    return Hierarchy(tree, kind, face_beta, face_frac, stream=stream, **mg)


def octmg_apply(h: Hierarchy, x, y, stream=None):
    h.apply(x, y, stream)


def octmg_vcycle(h: Hierarchy, b, u, stream=None):
    h.vcycle(b, u, stream)


def octmg_pcg_solve(h: Hierarchy, b, x, **kw):
    return h.pcg_solve(b, x, **kw)


def octmg_tank_fields(tree, centre=(0.5, 0.5, 0.5), radius=0.3, stream=None):
    return tank_fields(tree, centre, radius, stream)


def octmg_mg_solve(h: Hierarchy, b, x, **kw):
    return h.mg_solve(b, x, **kw)
