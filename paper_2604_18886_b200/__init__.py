"""B200-native (sm_100a) matrix-free multigrid-preconditioned CG on adaptive octrees
(arXiv 2604.18886).  The compute path is liboctmg.so (hand-written CUDA); this package is
its build script and a thin ctypes binding."""
from .octmg import (  # noqa: F401
    Tree, Hierarchy, OctmgError, octmg_build_tree, octmg_setup_hierarchy, octmg_apply, octmg_vcycle,
    octmg_pcg_solve, octmg_mg_solve, octmg_tank_fields, tank_fields, version, lib, ABI_SYMBOLS, NcclComm,
    partition_plan_host, grade_repair_host, set_allocator, use_torch_allocator, band_tiles, tank_fields_inner,
)
