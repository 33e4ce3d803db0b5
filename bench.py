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
  host cores, one bounded sample of the same workload per host thread.

Multi-GPU: ``python -m torch.distributed.run --nproc-per-node N bench.py
--gpus N`` runs N independent replicas (round 1 is
"replicas only"); value = N·n / max-over-ranks step time.
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
SAMPLE_GRID = 384  # bounded CPU sample of config 2 (same generator and parameters, ~30 s single-threaded)


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

        # NCCL between the GPUs of the box; gloo only for the CPU tests of this plumbing
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
        pg = dist
    return world, rank, local, pg


def barrier_max(pg, value: float, device) -> float:
    if pg is None:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device=device)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def run_reference(args) -> dict:
    """The reference CPU path: bounded samples of config 2, all host threads."""
    from oracle import refbind
    from paper_2601_04112_b200 import configs

    try:
        chk, kind = refbind.reference(), "reference"
    except FileNotFoundError:
        chk, kind = refbind.oracle(), "port"
    grid = args.sample_grid
    cfg = configs.config("c2", grid)
    p = refbind.params_for(cfg)
    threads = max(1, min(os.cpu_count() or 1, 64))

    def one_step():
        def work():
            h = chk.setup(cfg, p)
            h.pcg(cfg.rhs, 1e-8, 1000)

        ts = [threading.Thread(target=work) for _ in range(threads)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        one_step()
    times = [one_step() for _ in range(args.steps)]
    ms = 1e3 * statistics.mean(times)
    value = threads * cfg.n / (ms / 1e3)
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c2", "grid": grid, "n": cfg.n, "sample_of": "c2 1024x1024",
                   "parallelism": f"{threads} independent single-threaded solves"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"config-2 generator at {grid}x{grid} (n={cfg.n}), setup+PCG end to end, "
                                   f"one per thread on {threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def cpu_baseline_sample() -> dict:
    from oracle import refbind
    from paper_2601_04112_b200 import configs

    try:
        chk, kind = refbind.reference(), "reference"
    except FileNotFoundError:
        chk, kind = refbind.oracle(), "port"
    cfg = configs.config("c2", SAMPLE_GRID)
    p = refbind.params_for(cfg)
    t0 = time.perf_counter()
    h = chk.setup(cfg, p)
    t1 = time.perf_counter()
    _, rep = h.pcg(cfg.rhs, 1e-8, 1000)
    t2 = time.perf_counter()
    return {"value": cfg.n / (t2 - t0), "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"config-2 generator at {SAMPLE_GRID}x{SAMPLE_GRID} (n={cfg.n}), setup {t1 - t0:.2f}s + "
                      f"PCG {t2 - t1:.2f}s ({rep['iterations']} it), single-threaded reference"}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--grid", type=int, default=None, help="override the grid (debug only; not a bench number)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sample-grid", type=int, default=SAMPLE_GRID,
                    help="grid of the CPU reference sample (the default is the documented bench sample)")
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

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = lsamgdd.library()
    cfg = configs.config(args.config, args.grid)
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
        for i in range(min(cnt.value, 64)):
            stages[names[i].decode()] = stages.get(names[i].decode(), 0.0) + ms[i]
        summ = []
        nl = C.c_int64()
        lib.lsamgdd_num_levels(h, C.byref(nl))
        oc = C.c_double()
        lib.lsamgdd_operator_complexity(h, C.byref(oc))
        lib.lsamgdd_destroy(h)
        return {"iterations": rep.iterations, "converged": bool(rep.converged), "setup_ms": setup_ms,
                "solve_ms": rep.solve_seconds * 1e3, "levels": nl.value, "opcx": oc.value, "stages": stages}

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
                    "kernel": "level-0 Schwarz RAS + RAS-T sweep pair (k_schwarz_lrow: 1 RAS + 4 colour launches)",
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
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline_sample()
        except Exception as e:  # the checker is test infrastructure; report its absence
            out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                                   "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
