#!/usr/bin/env python
"""Benchmark: full PCG-MG solve throughput (leaf cells / s to relative residual 1e-6).

One "step" = one complete octmg_pcg_solve (Alg. 1 with the FAS mu-cycle preconditioner,
every PCG iteration until ||r|| <= 1e-6 ||r0||) on the workload BASELINE.json's metric is
quoted on: config 2, uniform 256^3 (16.78M leaf cells) with the paper's Sec. 5.3 setup
(Table 1 was measured on it).  Inputs are resident in HBM before
the timed region; setup (tree, coefficients, Galerkin hierarchy) is outside it, as in
Table 1 (reading #14).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl ours|reference]

N > 1: launched by torchrun (one process per GPU), or, when WORLD_SIZE is unset, bench.py
re-launches itself under torch.distributed.run with N processes.  The same workload is partitioned across the ranks by contiguous Morton
ranges: NCCL halo exchange after every kernel that
changes a partitioned level, fp64 allreduce for every PCG scalar.  value = total cells /
max-over-ranks time, "scaling": "strong".  --replicas instead solves one independent
instance per rank ("scaling": "weak", no data-path collective).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "full PCG-MG solve cells/sec to 1e-6 rel residual; HBM GB/s vs peak"
WORKLOADS = {
    "cfg2_uniform256": "BASELINE config 2: uniform 256^3 sinusoidal Poisson, paper Sec. 5.3 setup "
                       "(outermost cell layer Neumann, null-space projection), V-cycle mu=1, rtol 1e-6",
    "cfg1_octant": "BASELINE config 1: 16^3 base + one refined octant (7680 leaves), Dirichlet walls",
    "cfg3_sphere": "BASELINE config 3: sphere band l0=4..7 (60.1M leaves), paper Sec. 5.3 setup",
    "uniform128": "uniform 128^3 (paper Table 1 uniform (4-4)), Sec. 5.3 setup",
    "tank_mid": "cut-cell tank, sphere obstacle r=0.3, levels 3..5, W-cycle mu=2",
    "cfg4_tank": "BASELINE config 4: cut-cell tank, sphere obstacle r=0.30, l0=4..8 (155.2M leaves), W-cycle mu=2",
    "cfg5_tank": "BASELINE config 5: cut-cell tank, sphere obstacle r=0.35, l0=4..9 (838.8M leaves), W-cycle mu=2",
}
CPU_SAMPLE = "uniform64"  # same recipe as cfg2 at 64^3: the bounded oracle sample


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2_uniform256")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rtol", type=float, default=1e-6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--replicas", action="store_true", help="N>1: independent instance per rank")
    ap.add_argument("--no-wcycle", action="store_true",
                    help="skip the W-cycle configs 4/5 timed beside the headline (extra keys)")
    ap.add_argument("--wcycle-steps", type=int, default=5)
    return ap.parse_args()


def spawn_ranks(args):
    """--gpus N > 1 without a torchrun environment: re-launch this script under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1); rank 0 prints the
    line.  Returns the launcher's exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def check_solve(rep, what):
    """Every timed / warm-up solve must converge: a MAXITER or failed solve
    never becomes a throughput number."""
    if not rep["converged"] or rep["status"] != "OK":
        raise RuntimeError(f"{what}: solve did not converge (status {rep['status']}, iters {rep['iters']}, "
                           f"rel residual {rep['rel_residual']:.3e})")
    return rep


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for k, nm in enumerate(names):
                    if r[5 + k].strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model():
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _oracle_solves(name, seconds, threads, max_solves=None):
    """Full fp64 oracle solves of workload `name` for >= `seconds` (at least one), with
    `threads` OpenMP threads (set before the oracle library is first loaded)."""
    from octgen import make_config
    from oracle.oracle import Oracle
    cfg = make_config(name)
    o = Oracle(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    o.setup(cfg["kind"], cfg["w"])
    b = cfg["b"].astype(np.float64)
    n, t0, iters = 0, time.perf_counter(), 0
    while True:
        r = o.pcg(b, rtol=1e-6, mu=cfg["mu"])
        n += 1
        iters = r["iters"]
        el = time.perf_counter() - t0
        if el >= seconds or (max_solves and n >= max_solves):
            break
    return {"cells_per_s": n * o.N / el, "solves": n, "seconds": el, "iters": iters, "cells": o.N,
            "threads": threads}


def _oracle_leg(name, seconds, threads, max_solves=None):
    """One oracle timing leg in a child process (OMP_NUM_THREADS must be fixed before the
    OpenMP runtime starts)."""
    code = ("import json, sys; sys.path.insert(0, %r); import bench; "
            "print(json.dumps(bench._oracle_solves(%r, %r, %d, %r)))" % (ROOT, name, seconds, threads, max_solves))
    env = dict(os.environ, OMP_NUM_THREADS=str(threads))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=900)
    if out.returncode != 0:
        raise RuntimeError(out.stderr[-2000:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def cpu_baseline(seconds: float, config: str):
    """The fp64 oracle as it stands, timed on the host cores: one full solve of the headline
    workload itself at all cores (same_config), and a single-thread leg on a bounded 64^3
    sample of the same recipe."""
    ncores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    full = _oracle_leg(config, 0.0, ncores, max_solves=1)
    one = _oracle_leg(CPU_SAMPLE, seconds, 1)
    return {"value": full["cells_per_s"], "unit": "cells/s", "cores": ncores, "kind": "oracle",
            "same_config": True, "cpu_model": cpu_model(),
            "sample": f"{config} itself: {full['solves']} full fp64 solve to 1e-6 ({full['iters']} PCG iterations, "
                      f"{full['cells']} leaf cells) in {full['seconds']:.1f} s on {ncores} threads",
            "single_thread": {"value": one["cells_per_s"], "unit": "cells/s", "cores": 1,
                              "sample": f"{CPU_SAMPLE} (64^3, same recipe): {one['solves']} full fp64 solves "
                                        f"({one['iters']} PCG iterations each) in {one['seconds']:.1f} s"}}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from octgen import make_config
    from oracle.oracle import Oracle
    cfg = make_config(CPU_SAMPLE)
    o = Oracle(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    o.setup(cfg["kind"], cfg["w"])
    b = cfg["b"].astype(np.float64)
    for _ in range(args.warmup):
        o.pcg(b, rtol=args.rtol, mu=cfg["mu"])
    t0 = time.perf_counter()
    iters = 0
    for _ in range(args.steps):
        iters = o.pcg(b, rtol=args.rtol, mu=cfg["mu"])["iters"]
    el = time.perf_counter() - t0
    value = args.steps * o.N / el
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    line = {"metric": METRIC, "value": value, "unit": "cells/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": WORKLOADS.get(args.config, args.config),
                       "reference_sample": f"{CPU_SAMPLE}: 64^3 instance of the same recipe per step",
                       "leaf_cells": o.N, "iters": iters},
            "cpu_baseline": {"value": value, "unit": "cells/s", "cores": cores, "kind": "oracle",
                             "sample": f"{CPU_SAMPLE} per step, {args.steps} steps"},
            "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def time_config(om, torch, name, steps, warmup, rtol):
    """ms per solve of one more BASELINE config on this GPU (device-resident inputs, same
    timing rules as the headline), plus its per-class profile (separate pass)."""
    from octgen import make_config
    cfg = make_config(name, with_fields=False)
    tank = cfg["bc"] == "tank"
    if not tank:
        cfg = make_config(name)
    t0 = time.perf_counter()
    tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    if tank:
        kind, frac, b = om.tank_fields(tree, (0.5, 0.5, 0.5), cfg["radius"])
    else:
        kind = torch.from_numpy(cfg["kind"]).cuda()
        frac = None if cfg["w"] is None else torch.from_numpy(np.ascontiguousarray(cfg["w"])).cuda()
        b = torch.from_numpy(cfg["b"]).cuda()
    h = om.Hierarchy(tree, kind, face_frac=frac, mu=cfg["mu"])
    del frac, kind
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    x = torch.zeros_like(b)
    for _ in range(warmup):
        check_solve(h.pcg_solve(b, x, rtol=rtol), name + " warm-up")
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    reps = [h.pcg_solve(b, x, rtol=rtol) for _ in range(steps)]
    ev1.record(stream)
    torch.cuda.synchronize()
    for rep in reps:
        check_solve(rep, name)
    ms = ev0.elapsed_time(ev1) / steps
    h.profile(True)
    check_solve(h.pcg_solve(b, x, rtol=rtol), name + " profiling")
    prof = h.profile_read()
    h.profile(False)
    top = sorted(((k, v["ms"]) for k, v in prof.items() if v["launches"]), key=lambda kv: -kv[1])[:4]
    out = {"workload": WORKLOADS.get(name, name), "leaf_cells": tree.N, "mu": cfg["mu"], "steps": steps,
           "warmup": warmup, "ms_per_solve": ms, "cells_per_s": tree.N / (ms * 1e-3), "pcg_iters": reps[-1]["iters"],
           "setup_s": setup_s, "profile_top_ms": {k: v for k, v in top},
           "profile_note": "per-class ms of one solve with CUDA events around every launch (graph replay off)"}
    del h, tree, b, x
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def traffic_from_profiles(config):
    """ncu dram bytes per launch of the dominant kernel, from the committed summary."""
    p = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    try:
        d = json.load(open(p))
        return d.get(config)
    except Exception:
        return None


def main():
    args = parse()
    rank, world, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one process per GPU")
    if args.impl == "reference":
        return run_reference(args)
    import torch
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    import paper_2604_18886_b200 as om
    from octgen import make_config
    assert args.warmup >= 3 or os.environ.get("BENCH_ALLOW_SHORT"), "timing rules need >= 3 warm-up steps"

    # cut-cell tank configs: the fields come from the device geometry pipeline
    # (octmg_tank_fields, parity-tested against the oracle); the others from octgen
    cfg = make_config(args.config, with_fields=False)
    tank = cfg["bc"] == "tank"
    if not tank:
        cfg = make_config(args.config)
    partitioned = world > 1 and not args.replicas
    setup_note = None
    comm = None
    if partitioned:
        # every rank takes the same branch: a failed NCCL bootstrap / partitioned tree build on
        # any rank switches all ranks to independent replicas, and the line says so
        try:
            comm = om.NcclComm(rank, world)
            tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"], comm=comm)
            ok = 1.0
        except Exception as e:  # noqa: BLE001
            setup_note = f"partitioned setup failed on rank {rank}: {e}"
            ok = 0.0
        flag = torch.tensor([ok], device=dev)
        torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)
        if flag.item() < 1.0:
            partitioned = False
            comm = None
            setup_note = setup_note or "partitioned setup failed on another rank"
    if not partitioned:
        tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    if tank:
        kind, frac, b = om.tank_fields(tree, (0.5, 0.5, 0.5), cfg["radius"])
        b_host = b.cpu().pin_memory()
    else:
        kind = torch.from_numpy(cfg["kind"]).to(dev)
        frac = None if cfg["w"] is None else torch.from_numpy(np.ascontiguousarray(cfg["w"])).to(dev)
        b_host = torch.from_numpy(cfg["b"]).pin_memory()
    h = om.Hierarchy(tree, kind, face_frac=frac, mu=cfg["mu"])
    del frac
    b = b_host.to(dev)
    x = torch.zeros_like(b)
    x_host = torch.empty_like(b_host).pin_memory()
    N = tree.N
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timing --------------------------------------------------------
    for _ in range(args.warmup):
        rep = check_solve(h.pcg_solve(b, x, rtol=args.rtol), "warm-up")
    torch.cuda.synchronize()
    barrier()
    sampler = ClockSampler(dev.index)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    launches = 0
    iters = []
    reps = []
    for _ in range(args.steps):
        rep = h.pcg_solve(b, x, rtol=args.rtol)
        reps.append(rep)
        launches += rep["kernel_launches"]
        iters.append(rep["iters"])
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    for rep in reps:
        check_solve(rep, "timed")
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    units = N if partitioned else world * N  # cells solved by the whole job per step
    value = units / (ms * 1e-3)

    # ---- end to end through the public API with host buffers --------------------------
    # Every step copies its rhs from pinned host memory and its solution back (the bytes
    # counted below), pipelined the way a serving loop would: the next step's rhs is
    # uploaded on one copy stream while this step solves, and this step's solution is
    # downloaded on another while the next one solves (double-buffered device vectors).
    s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    b2 = [b, torch.empty_like(b)]
    x2 = [x, torch.empty_like(x)]
    xh2 = [x_host, torch.empty_like(x_host).pin_memory()]
    e_b = [torch.cuda.Event(), torch.cuda.Event()]
    e_x = [torch.cuda.Event(), torch.cuda.Event()]
    e_d = [torch.cuda.Event(), torch.cuda.Event()]

    e2e_reps = []

    def run_e2e(n):
        s_in.wait_stream(stream)
        s_out.wait_stream(stream)
        for i in (0, 1):
            e_d[i].record(s_out)
        with torch.cuda.stream(s_in):
            b2[0].copy_(b_host, non_blocking=True)
        e_b[0].record(s_in)
        for k in range(n):
            i = k & 1
            if k + 1 < n:  # the buffer of step k-1 is free (pcg_solve returned after it)
                with torch.cuda.stream(s_in):
                    b2[1 - i].copy_(b_host, non_blocking=True)
                e_b[1 - i].record(s_in)
            stream.wait_event(e_b[i])
            stream.wait_event(e_d[i])  # the download of x2[i] from step k-2 is done
            e2e_reps.append(h.pcg_solve(b2[i], x2[i], rtol=args.rtol, stream=stream))
            e_x[i].record(stream)
            s_out.wait_event(e_x[i])
            with torch.cuda.stream(s_out):
                xh2[i].copy_(x2[i], non_blocking=True)
            e_d[i].record(s_out)
        stream.wait_stream(s_out)
        stream.wait_stream(s_in)

    run_e2e(max(2, args.warmup))
    torch.cuda.synchronize()
    barrier()
    ev0.record(stream)
    run_e2e(args.steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_e2e = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    for rep in e2e_reps:
        check_solve(rep, "e2e")

    # ---- per-kernel device time (profiling pass: events around every launch) -----------
    h.profile(True)
    for _ in range(2):
        check_solve(h.pcg_solve(b, x, rtol=args.rtol), "profiling")
    prof = h.profile_read()
    h.profile(False)
    dom = max((k for k in prof if prof[k]["launches"]), key=lambda k: prof[k]["ms"])
    tot_ms = sum(v["ms"] for v in prof.values())
    d = prof[dom]
    achieved = d["bytes"] / (d["ms"] * 1e-3) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    solve_bytes = sum(v["bytes"] for v in prof.values()) / 2
    traffic = traffic_from_profiles(args.config)

    line = {}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if partitioned else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOADS.get(args.config, args.config), "name": args.config,
                       "leaf_cells": N, "levels": tree.levels, "mu": cfg["mu"], "rtol": args.rtol,
                       "pcg_iters": iters[-1], "parallelism": (f"Morton-range partition x{world} (NCCL halo + allreduce)" if partitioned
                                       else f"replicas x{world}" if world > 1 else "1 GPU"),
                       "l2": "working set > 126 MB L2 (coefficient store alone %.0f MB); no flush"
                             % (tree.T * 512 * 16 / 1e6)},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": "committed ncu --set full capture (profiles/roofline_traffic.json), "
                                           "not measured in this run",
                         "share_of_step": d["ms"] / tot_ms if tot_ms else None,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"},
            "model_gbs_solve": solve_bytes / (ms * 1e-3) / 1e9,
            "kernels": {k: {"ms_per_solve": v["ms"] / 2, "launches_per_solve": v["launches"] // 2,
                            "gbs": (v["bytes"] / (v["ms"] * 1e-3) / 1e9) if v["ms"] else None}
                        for k, v in prof.items() if v["launches"]},
            "e2e": {"value": units / (ms_e2e * 1e-3), "unit": "cells/s", "h2d_bytes_per_step": 4 * N * world,
                    "d2h_bytes_per_step": 4 * N * world, "ms_per_step": ms_e2e,
                    "pipeline": "next rhs upload and previous solution download overlap the solve (2 copy streams)"},
            "gpu_launches": launches,
            "clocks": clocks,
            "paper_context": "RTX 4090: uniform (5-5) 256^3 = 2.41e8 cells/s (Table 1, P:L1797, M = 2^20)",
            "setup_note": setup_note,
        }
    if world == 1 and not args.no_wcycle and args.config == "cfg2_uniform256":
        # the W-cycle configs (BASELINE configs 4, 5) timed in the same run, as extra keys
        del h, tree, b, x, b2, x2, kind
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        extra = {}
        for name in ("cfg4_tank", "cfg5_tank"):
            extra[name] = time_config(om, torch, name, args.wcycle_steps, 3, args.rtol)
        line["wcycle_configs"] = extra
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(args.cpu_seconds, args.config)
        print(json.dumps(line), flush=True)
    if world > 1:
        del h, tree
        comm = None
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
