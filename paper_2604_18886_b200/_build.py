"""Build of the CUDA library (sm_100a).

``build_library()`` compiles paper_2604_18886_b200/csrc/*.cu with nvcc for sm_100a into
an in-tree shared object (liboctmg.so) that the ctypes binding loads.
"""
from __future__ import annotations

import concurrent.futures
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "liboctmg.so")
SOURCES = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")) + glob.glob(os.path.join(HERE, "csrc", "*.cpp")))
HEADERS = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + glob.glob(os.path.join(HERE, "csrc", "*.h"))) + [os.path.join(ROOT, "include", "octmg.h")]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "550,128"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in SOURCES + HEADERS)


def build_library(force: bool = False, verbose: bool = False) -> str:
    if force or _stale():
        nvcc = os.environ.get("NVCC", "nvcc")
        tmp = LIB + ".tmp%d" % os.getpid()
        objdir = os.path.join(HERE, "build")
        os.makedirs(objdir, exist_ok=True)
        cflags = [f for f in NVCC_FLAGS if f != "-shared"]
        objs, cmds = [], []
        for src in SOURCES:
            obj = os.path.join(objdir, os.path.basename(src) + ".o")
            objs.append(obj)
            # fp64 SDF / box tests = the host's IEEE operations (no FMA contraction)
            extra = ["-fmad=false"] if os.path.basename(src) in ("geometry.cu", "band.cu") else []
            cmds.append([nvcc] + cflags + extra + ["-c", "-o", obj, src])
        if verbose:
            for c in cmds:
                print(" ".join(c))
        # one nvcc per translation unit, in parallel, then one link
        with concurrent.futures.ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 4)) as ex:
            for f in [ex.submit(subprocess.check_call, c) for c in cmds]:
                f.result()
        link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] + objs + ["-ldl"]
        if verbose:
            print(" ".join(link))
        subprocess.check_call(link)
        os.replace(tmp, LIB)
    return LIB
