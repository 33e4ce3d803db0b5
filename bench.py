#!/usr/bin/env python3
"""Benchmark of the B200 AMG-DD hot path (BASELINE.json metric).

One step = one full pass of the hot path on BASELINE config 2 (1024×1024
rotated anisotropy, n = 1,048,576): ``setup(G)`` (aggregation, batched local
GEVPs, Schwarz factorisation, Galerkin recursion) followed by a PCG solve to
rtol 1e-8 with the V(1,1) cycle. Metric: unknowns/s = n / (T_setup + T_solve).

* ``value``: inputs (G as CSR, the RHS) resident in HBM before the timed
  region; setup and solve through the C ABI on device pointers.
* ``e2e``: the same step through the C ABI with host buffers (G and b copied
  in, x copied out inside the timed region).
* ``--impl reference``: the reference's own CPU implementation (the
  unmodified headers compiled into oracle/_ref, else the C oracle) on the
  host cores, on the same 1024×1024 problem: its level-0 stages and the
  level-0 work of the PCG iterations (the coarse levels, which the reference
  cannot finish at this size, are left out — an upper bound for the CPU).
  The GPU line carries the same stages as ``same_stages`` for a like-for-like
  ratio.

Multi-GPU: ``python -m torch.distributed.run --nproc-per-node N bench.py
--gpus N`` runs the row/aggregate partition of paper_2601_04112_b200/dist.py
(DESIGN.md §6): the same 1024² problem split into N strips, one process per
GPU, halo exchange / reverse-halo add / dot all-reduce / gathered coarse
vector over NCCL; value = n / max-over-ranks step time (``"scaling":
"strong"``). The N = 1 line is the single-GPU library path.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AMG-DD setup+PCG solve unknowns/s"
UNIT = "unknowns/s"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def load_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi style clock/throttle sampling during the timed region."""

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        self.device = device

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                getattr(pynvml, "nvmlClocksThrottleReasonHwSlowdown", 0x8): "hw_slowdown",
                getattr(pynvml, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
                getattr(pynvml, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
                getattr(pynvml, "nvmlClocksThrottleReasonSwPowerCap", 0x4): "sw_power_cap",
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        for bit, nm in names.items():
                            if r & bit:
                                self.reasons.add(nm)
                    except Exception:
                        pass
                    time.sleep(0.2)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self) -> dict:
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup(n_gpus: int):
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    pg = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        import torch

        # NCCL between the GPUs of the box; gloo for the CPU tests of this plumbing and for the
        # one-GPU plumbing check of the partitioned path (LSB_DIST_BACKEND=gloo: the ranks share a GPU)
        backend = os.environ.get("LSB_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        dist.init_process_group(backend)
        pg = dist
    return world, rank, local, pg


def barrier_max(pg, value: float, device) -> float:
    if pg is None:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device=device)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


# PCG iterations of the bench workload (what the GPU arm reports for it); the
# reference arm multiplies its level-0 per-iteration time by this count
WORKLOAD_ITERS = {("c2", 1024): 70}

LEVEL0_STAGES = ("level-0 setup stages (A0 = G^T G, topology, build_smoother, all local GEVPs, P0, Galerkin G1/A1) "
                 "+ per PCG iteration the level-0 operator and smoother applications (G p, G^T(G p), RAS, RAS-T)")


def reference_checker():
    from oracle import refbind

    try:
        return refbind.reference(), "reference"
    except (FileNotFoundError, OSError):
        return refbind.oracle(), "port"


def reference_level0_step(chk, cfg, threads: int, iters: int) -> dict:
    """The reference's own functions on the level-0 share of the workload at its
    full grid (probe_levels = 1). The coarse levels are left out: the reference's
    sequential Jacobi eigensolves on them take days at this size,
    so the resulting unknowns/s is an upper bound for the CPU."""
    from oracle import refbind
    from paper_2601_04112_b200 import abi

    os.environ["LSAMGDD_REF_THREADS"] = str(threads)
    p = refbind.params_for(cfg, probe_levels=1)
    t0 = time.perf_counter()
    h = chk.setup(cfg, p)
    t_setup = time.perf_counter() - t0
    x = cfg.rhs
    t0 = time.perf_counter()
    y = h.spmv(x, 0, abi.EXPORT_G, False, nout=cfg.m)
    h.spmv(y, 0, abi.EXPORT_G, True, nout=cfg.n)
    e = h.schwarz_apply(x, 0, abi.RAS)
    h.schwarz_apply(e, 0, abi.RAST)
    t_iter = time.perf_counter() - t0
    stages = {}
    for nm, sec in h.timings():
        stages[nm] = stages.get(nm, 0.0) + sec * 1e3
    del h
    return {"seconds": t_setup + iters * t_iter, "setup_ms": t_setup * 1e3, "iter_ms": t_iter * 1e3,
            "stages_ms": {k: round(v, 1) for k, v in stages.items()}}


def run_reference(args) -> dict:
    """The reference CPU path on the bench workload's own grid: its level-0 share, all host threads."""
    from paper_2601_04112_b200 import configs

    chk, kind = reference_checker()
    cfg = configs.config(args.config, args.grid)
    grid = cfg.meta["grid"]
    iters = WORKLOAD_ITERS.get((cfg.name, grid), 50)
    threads = max(1, min(os.cpu_count() or 1, 64))
    for _ in range(args.warmup):
        last = reference_level0_step(chk, cfg, threads, iters)
    times = []
    for _ in range(args.steps):
        last = reference_level0_step(chk, cfg, threads, iters)
        times.append(last["seconds"])
    ms = 1e3 * statistics.mean(times)
    value = cfg.n / (ms / 1e3)
    sample = (f"{LEVEL0_STAGES} of the same {grid}x{grid} problem, {iters} iterations; the coarse levels are left out "
              f"(the reference cannot finish them at this size), so this is an upper bound for the CPU; "
              f"per-aggregate stages on {threads} host threads")
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "grid": grid, "n": cfg.n, "m": cfg.m, "nnz_G": cfg.nnz,
                   "parallelism": f"{threads} host threads over the independent aggregates",
                   "setup_ms": last["setup_ms"], "iter_ms": last["iter_ms"], "stages_ms": last["stages_ms"],
                   "pcg_iterations": iters},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def cpu_baseline_sample(cfg, iters: int) -> dict:
    chk, kind = reference_checker()
    threads = max(1, min(os.cpu_count() or 1, 64))
    r = reference_level0_step(chk, cfg, threads, iters)
    return {"value": cfg.n / r["seconds"], "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{LEVEL0_STAGES} of the same {cfg.meta['grid']}x{cfg.meta['grid']} problem, {iters} iterations, "
                      f"{threads} host threads: setup stages {r['setup_ms'] / 1e3:.2f} s + {iters} x {r['iter_ms']:.1f} ms; "
                      f"coarse levels left out (upper bound for the CPU)",
            "level0_ms": r["seconds"] * 1e3, "setup_ms": r["setup_ms"], "iter_ms": r["iter_ms"],
            "stages_ms": r["stages_ms"]}


def run_partitioned(args, cfg, world, rank, local, pg, dev) -> None:
    """N > 1: the strip partition (strong scaling). One step = partitioned setup (level-0 stages
    per strip, all-gathered P0, replicated coarse hierarchy) + distributed PCG to 1e-8."""
    import torch

    from paper_2601_04112_b200 import dist as pdist, lsamgdd

    comm = pdist.TorchComm(pg, dev if pg.get_backend() == "nccl" else "cpu")
    over = {"device": local}
    if "thresh_override" not in dict(cfg.params) or not dict(cfg.params).get("thresh_override"):
        # the reference's threshold rule needs the global colour count and multiplicity bound
        # (splitting.hpp:170-180): take them from a level-0 probe of the whole problem on rank 0
        thr = torch.zeros(1, dtype=torch.float64, device=dev)
        if rank == 0:
            hp = lsamgdd.setup(cfg, lsamgdd.params_for(cfg, probe_levels=1, device=local))
            thr[0] = hp.summary[0].thresh
            del hp
        if pg.get_backend() != "nccl":
            thr = thr.cpu()
        pg.broadcast(thr, 0)
        over["level0_thresh"] = float(thr.item())
    lvl0_thr = over.pop("level0_thresh", None)

    def step():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        solver = pdist.build_gpu_solver(cfg, comm, over, level0_thresh=lvl0_thr)
        t1 = time.perf_counter()
        x, its, conv, hist = solver.pcg(cfg.rhs[solver.plan.own], 1e-8, 1000)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        levels = solver.ops.h_coarse.num_levels + 1
        solver.ops.close()
        return (t2 - t0) * 1e3, (t1 - t0) * 1e3, (t2 - t1) * 1e3, its, conv, levels

    for _ in range(args.warmup):
        step()
    c0 = lib_launches()
    with ClockSampler(local) as clk:
        recs = []
        for _ in range(args.steps):
            pg.barrier()
            recs.append(step())
    launches = (lib_launches() - c0) // max(args.steps, 1)
    rdev = dev if pg.get_backend() == "nccl" else torch.device("cpu")
    ms_step = barrier_max(pg, statistics.mean(r[0] for r in recs), rdev)
    setup_ms = barrier_max(pg, statistics.mean(r[1] for r in recs), rdev)
    solve_ms = barrier_max(pg, statistics.mean(r[2] for r in recs), rdev)
    value = cfg.n / (ms_step / 1e3)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": cfg.name, "grid": cfg.meta["grid"], "n": cfg.n, "m": cfg.m, "nnz_G": cfg.nnz,
                   "levels": recs[-1][5], "pcg_iterations": recs[-1][3], "converged": bool(recs[-1][4]),
                   "setup_ms": setup_ms, "solve_ms": solve_ms,
                   "l2": "inputs larger than L2 (G0 CSR %.0f MB > 126 MB)" % ((cfg.g_rowptr.nbytes + cfg.g_cols.nbytes + cfg.g_vals.nbytes) / 1e6),
                   "parallelism": f"{world} strips of level-0 aggregates (halo exchange, reverse-halo add, dot all-reduce, "
                                  "gathered coarse vector; coarse hierarchy replicated; vectors staged through the host)"},
        "roofline": None,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": int(cfg.g_rowptr.nbytes + cfg.g_cols.nbytes + cfg.g_vals.nbytes + cfg.rhs.nbytes),
                "d2h_bytes_per_step": int(8 * cfg.n), "ms_per_step": ms_step,
                "note": "the partitioned path takes host buffers: every operator call copies its strip vectors in and out"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    pg.destroy_process_group()


def lib_launches() -> int:
    from paper_2601_04112_b200 import lsamgdd

    return int(lsamgdd.library().lsamgdd_launch_count())


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--grid", type=int, default=None, help="override the grid (debug only; not a bench number)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world, rank, local, pg = dist_setup(args.gpus)
    if args.impl == "reference":
        # the reference is a CPU library: rank 0 alone runs it, the other ranks exit 0
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return

    import torch

    from paper_2601_04112_b200 import abi, configs, lsamgdd

    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = lsamgdd.library()
    cfg = configs.config(args.config, args.grid)
    if world > 1:
        run_partitioned(args, cfg, world, rank, local, pg, dev)
        return
    params = lsamgdd.params_for(cfg, device=local)
    pabi, keep = params.to_abi()
    n, m, nnz = cfg.n, cfg.m, cfg.nnz

    # device-resident inputs (value) and pinned host inputs (e2e)
    d_rp = torch.from_numpy(cfg.g_rowptr).to(dev)
    d_col = torch.from_numpy(cfg.g_cols).to(dev)
    d_val = torch.from_numpy(cfg.g_vals).to(dev)
    d_b = torch.from_numpy(cfg.rhs).to(dev)
    d_x = torch.empty(n, dtype=torch.float64, device=dev)
    h_rp = torch.from_numpy(cfg.g_rowptr).pin_memory()
    h_col = torch.from_numpy(cfg.g_cols).pin_memory()
    h_val = torch.from_numpy(cfg.g_vals).pin_memory()
    h_b = torch.from_numpy(cfg.rhs).pin_memory()
    h_x = torch.empty(n, dtype=torch.float64).pin_memory()

    def csr(memory: int, rp, col, val) -> abi.Csr:
        g = abi.Csr()
        g.n_rows, g.n_cols, g.nnz = m, n, nnz
        g.row_offsets, g.col_indices, g.values = rp.data_ptr(), col.data_ptr(), val.data_ptr()
        g.memory = memory
        return g

    g_dev = csr(abi.DEVICE, d_rp, d_col, d_val)
    g_host = csr(abi.HOST, h_rp, h_col, h_val)
    err = C.create_string_buffer(1024)

    def step(device_inputs: bool, stats=None):
        h = C.c_void_p()
        g = g_dev if device_inputs else g_host
        st = lib.lsamgdd_setup(C.byref(g), C.byref(pabi), C.byref(h), err, C.c_size_t(1024))
        lsamgdd._check(st, err)
        rep = abi.Report()
        b = d_b if device_inputs else h_b
        x = d_x if device_inputs else h_x
        mem = abi.DEVICE if device_inputs else abi.HOST
        if stats is not None:
            st = lib.lsamgdd_profile_pcg(h, C.c_void_p(b.data_ptr()), C.c_double(1e-8), C.c_uint64(1000),
                                         C.c_void_p(x.data_ptr()), C.c_int32(mem), C.byref(rep), C.byref(stats), err,
                                         C.c_size_t(1024))
        else:
            st = lib.lsamgdd_pcg(h, None, C.c_void_p(b.data_ptr()), C.c_double(1e-8), C.c_uint64(1000),
                                 C.c_void_p(x.data_ptr()), C.c_int32(mem), C.byref(rep), err, C.c_size_t(1024))
        lsamgdd._check(st, err)
        names = (C.c_char_p * 64)()
        ms = (C.c_double * 64)()
        cnt = C.c_int64()
        lib.lsamgdd_setup_timings(h, names, ms, C.c_int64(64), C.byref(cnt))
        setup_ms = sum(ms[i] for i in range(min(cnt.value, 64)))
        stages = {}
        stages_list = []
        for i in range(min(cnt.value, 64)):
            stages[names[i].decode()] = stages.get(names[i].decode(), 0.0) + ms[i]
            stages_list.append((names[i].decode(), ms[i]))
        summ = []
        nl = C.c_int64()
        lib.lsamgdd_num_levels(h, C.byref(nl))
        oc = C.c_double()
        lib.lsamgdd_operator_complexity(h, C.byref(oc))
        lib.lsamgdd_destroy(h)
        return {"iterations": rep.iterations, "converged": bool(rep.converged), "setup_ms": setup_ms,
                "solve_ms": rep.solve_seconds * 1e3, "levels": nl.value, "opcx": oc.value, "stages": stages,
                "stages_list": stages_list}

    def timed(device_inputs: bool, k: int, stats=None):
        times, infos = [], []
        for _ in range(k):
            if pg:
                pg.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.cuda.synchronize()
            info = step(device_inputs, stats)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            infos.append(info)
        return times, infos

    for _ in range(args.warmup):
        step(True)
    c0 = lib.lsamgdd_launch_count()
    with ClockSampler(local) as clk:
        times, infos = timed(True, args.steps)
    launches = (lib.lsamgdd_launch_count() - c0) // max(args.steps, 1)
    ms_step = barrier_max(pg, statistics.mean(times), dev)
    value = world * n / (ms_step / 1e3)

    # end to end through host buffers (H2D of G and b, D2H of x inside the step)
    e2e_times, _ = timed(False, max(1, min(args.steps, 2)))
    e2e_ms = barrier_max(pg, statistics.mean(e2e_times), dev)
    h2d = int(cfg.g_rowptr.nbytes + cfg.g_cols.nbytes + cfg.g_vals.nbytes + cfg.rhs.nbytes)
    d2h = int(8 * n)

    # the same step with the factor written on the device (lsamgdd_generate_stencil_rows inside the
    # timed region): only b goes up and x comes down
    generated = None
    stencil = configs.config_stencil(cfg.name, cfg.meta["grid"])
    if stencil is not None:
        def step_generated():
            gd = lsamgdd.generate_stencil_rows(*stencil, device=local)
            try:
                h = C.c_void_p()
                gcsr = gd.to_abi()
                lsamgdd._check(lib.lsamgdd_setup(C.byref(gcsr), C.byref(pabi), C.byref(h), err, C.c_size_t(1024)), err)
                rep = abi.Report()
                st = lib.lsamgdd_pcg(h, None, C.c_void_p(h_b.data_ptr()), C.c_double(1e-8), C.c_uint64(1000),
                                     C.c_void_p(h_x.data_ptr()), C.c_int32(abi.HOST), C.byref(rep), err, C.c_size_t(1024))
                lib.lsamgdd_destroy(h)
                lsamgdd._check(st, err)
                return rep.iterations
            finally:
                gd.close()

        gt = []
        for _ in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.cuda.synchronize()
            its = step_generated()
            e1.record()
            torch.cuda.synchronize()
            gt.append(e0.elapsed_time(e1))
        gms = statistics.mean(gt)
        generated = {"value": world * n / (gms / 1e3), "unit": UNIT, "ms_per_step": gms, "pcg_iterations": int(its),
                     "h2d_bytes_per_step": int(cfg.rhs.nbytes), "d2h_bytes_per_step": int(8 * n),
                     "note": "factor generated in HBM by lsamgdd_generate_stencil_rows inside the timed step "
                             "(bit-identical to the host generator); host b in, host x out"}

    # dominant HBM kernel: level-0 Schwarz sweeps, CUDA events on their stream
    ks = abi.KernelStats()
    step(True, ks)
    peaks = load_peaks()
    roofline = None
    if ks.schwarz_ms > 0:
        achieved = ks.schwarz_bytes / (ks.schwarz_ms / 1e3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "schwarz_traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                    "kernel": "level-0 Schwarz RAS + RAS-T sweep pair (k_schwarz_tma: persistent TMA-pipelined sweeps, RAS-T followed by k_rast_slots)",
                    "bytes_per_launch": ks.schwarz_bytes / max(ks.schwarz_launches, 1),
                    "peak_source": peaks["source"]}
    # second HBM-bound kernel pair: the PCG operator Gᵀ(G p) (k_sell_spmv + k_ap_dot),
    # algorithmic bytes B(spmv_G) + B(spmvT_G) of SURVEY.md §8(d)
    roofline_spmv = None
    if ks.spmv_ms > 0:
        a2 = ks.spmv_bytes / (ks.spmv_ms / 1e3) / 1e9
        roofline_spmv = {"bound": "hbm", "achieved": a2, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": a2 / peaks["hbm_gbs"],
                         "kernel": "PCG operator y = Gᵀ(G p): k_sell_spmv<0> then k_ap_dot (fused <p, y>)",
                         "bytes_per_launch": ks.spmv_bytes / max(ks.spmv_launches, 1),
                         "peak_source": peaks["source"]}

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": cfg.name, "grid": cfg.meta["grid"], "n": n, "m": m, "nnz_G": nnz,
                   "levels": infos[-1]["levels"], "operator_complexity": infos[-1]["opcx"],
                   "pcg_iterations": infos[-1]["iterations"], "converged": infos[-1]["converged"],
                   "setup_ms": statistics.mean(i["setup_ms"] for i in infos),
                   "solve_ms": statistics.mean(i["solve_ms"] for i in infos),
                   "stages_ms": {k: round(v, 2) for k, v in infos[-1]["stages"].items()},
                   "l2": "inputs larger than L2 (G0 CSR %.0f MB > 126 MB)" % (h2d / 1e6),
                   "parallelism": "replicas" if world > 1 else "single"},
        "roofline": roofline,
        "roofline_spmv": roofline_spmv,
        "e2e": {"value": world * n / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if generated is not None:
        out["e2e_device_generated"] = generated
    # the same stages on the GPU: level-0 setup stage timers + per-iteration event times of the
    # operator pair and the Schwarz pair (measured inside the captured PCG graph)
    st0 = infos[-1]["stages_list"]
    lvl0 = {}
    seen = set()
    for nm, v in st0:
        if nm in seen:
            break  # the stage names repeat from level 1 on
        seen.add(nm)
        lvl0[nm] = v
    it = max(int(ks.spmv_launches) // 2, 1)  # graph-launched iterations the event times were summed over
    gpu_iter_ms = (ks.schwarz_ms + ks.spmv_ms) / it
    gpu_level0_ms = sum(lvl0.values()) + infos[-1]["iterations"] * gpu_iter_ms
    out["same_stages"] = {"stages": LEVEL0_STAGES, "gpu_ms": gpu_level0_ms, "gpu_setup_ms": sum(lvl0.values()),
                          "gpu_iter_ms": gpu_iter_ms, "gpu_stages_ms": {k: round(v, 2) for k, v in lvl0.items()}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline_sample(cfg, int(infos[-1]["iterations"]))
            out["same_stages"]["cpu_ms"] = out["cpu_baseline"]["level0_ms"]
            out["same_stages"]["cpu_cores"] = out["cpu_baseline"]["cores"]
            out["same_stages"]["ratio"] = out["cpu_baseline"]["level0_ms"] / gpu_level0_ms
        except Exception as e:  # the checker is test infrastructure; report its absence
            out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                                   "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
