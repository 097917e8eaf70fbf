"""Where the end-to-end time of config 2 goes: the solve alone, the 67 MB host->device and
device->host copies alone and overlapped with a solve, and the pipelined e2e loop of
bench.py with each copy direction switched off in turn."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2604_18886_b200 as om
from octgen import make_config

cfg = make_config("cfg2_uniform256")
tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
h = om.Hierarchy(tree, torch.from_numpy(cfg["kind"]).cuda(), mu=cfg["mu"])
b_host = torch.from_numpy(cfg["b"]).pin_memory()
x_host = torch.empty_like(b_host).pin_memory()
b = b_host.cuda()
x = torch.zeros_like(b)
st = torch.cuda.current_stream()
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, n=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, (time.perf_counter() - t0) * 1e3 / n


print("solve           %.3f ms (events) %.3f ms (wall)" % timed(lambda: h.pcg_solve(b, x)))
print("h2d 67 MB       %.3f ms" % timed(lambda: b.copy_(b_host, non_blocking=True))[0])
print("d2h 67 MB       %.3f ms" % timed(lambda: x_host.copy_(x, non_blocking=True))[0])


def both():
    b.copy_(b_host, non_blocking=True)
    x_host.copy_(x, non_blocking=True)


print("h2d+d2h same st %.3f ms" % timed(both)[0])


def overlapped_copies():
    with torch.cuda.stream(s_in):
        b2.copy_(b_host, non_blocking=True)
    with torch.cuda.stream(s_out):
        x_host.copy_(x2, non_blocking=True)
    h.pcg_solve(b, x)
    st.wait_stream(s_in)
    st.wait_stream(s_out)


b2 = torch.empty_like(b)
x2 = torch.empty_like(x)
print("solve || h2d || d2h %.3f ms" % timed(overlapped_copies)[0])


def solve_h2d_only():
    with torch.cuda.stream(s_in):
        b2.copy_(b_host, non_blocking=True)
    h.pcg_solve(b, x)
    st.wait_stream(s_in)


def solve_d2h_only():
    with torch.cuda.stream(s_out):
        x_host.copy_(x2, non_blocking=True)
    h.pcg_solve(b, x)
    st.wait_stream(s_out)


print("solve || h2d    %.3f ms" % timed(solve_h2d_only)[0])
print("solve || d2h    %.3f ms" % timed(solve_d2h_only)[0])
