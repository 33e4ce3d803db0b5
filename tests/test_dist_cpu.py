"""Multi-process plumbing of bench.py on CPU (gloo, world size 2): the
max-over-ranks timing reduction and the reference arm's rank-0-only run."""
import json
import os
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import bench

    v = bench.barrier_max(dist, float(10 * (rank + 1)), torch.device("cpu"))
    out[rank] = v
    dist.destroy_process_group()


def test_barrier_max_gloo():
    port = 29731
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == 20.0 and out[1] == 20.0


def test_reference_arm_rank0_only():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29733", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3", "--grid", "32"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["value"] > 0
    assert rec["e2e"]["h2d_bytes_per_step"] == 0 and rec["cpu_baseline"]["cores"] >= 1


# ---- the row/aggregate partition (paper_2601_04112_b200/dist.py) on CPU ----------------------
#
# The distributed driver (strip plan, halo exchange, reverse-halo add, all-gathered coarse
# vector, fused dot all-reduce) runs with numpy/oracle operators in place of the GPU ones and
# must reproduce the single-process oracle solve. Two-level hierarchies (large coarse_size), so
# the replicated coarse level is a dense solve.

def _cpu_ops_and_solver(cfg, comm, over):
    import numpy as np
    import scipy.sparse as sp

    from oracle import refbind
    from paper_2601_04112_b200 import abi, dist as pdist

    class CpuOps(pdist.LocalOps):
        def __init__(self, plan):
            self.plan = plan
            gs = plan.g_sub
            arr = (gs.indptr.astype(np.int64), gs.indices.astype(np.int64), gs.data.astype(np.float64), gs.shape[1])
            sub_over = dict(over, max_levels=2, coarse_size=1)  # the strip builds exactly its level-0 stages
            p = abi.default_params(level0_partition=plan.sub_part.astype(np.int64).ctypes.data,
                                   level0_n_aggregates=int(plan.sub_aggs.shape[0]), **sub_over)
            self._part = plan.sub_part.astype(np.int64)
            p.level0_partition = self._part.ctypes.data
            self.h = refbind.oracle().setup(arr, p)
            rp, ci, va, shape = self.h.export(0, abi.EXPORT_P)
            self.p_loc = pdist.slice_own_p(plan, sp.csr_matrix((va, ci, rp), shape=shape))
            rp, ci, va, shape = self.h.export(0, abi.EXPORT_A)
            self.a_own = sp.csr_matrix((va, ci, rp), shape=shape)[plan.own_in_ext].tocsr()
            self.g_own = gs[plan.g_own_rows].tocsr()
            self.a1 = None

        def g_apply(self, p_ext): return self.g_own @ p_ext
        def gt_apply(self, q): return self.g_own.T @ q
        def a_apply(self, e_ext): return self.a_own @ e_ext
        def ras(self, r_ext): return self.h.schwarz_apply(r_ext, 0, abi.RAS)
        def rast(self, r_ext): return self.h.schwarz_apply(r_ext, 0, abi.RAST)
        def restrict(self, res): return self.p_loc.T @ res
        def prolong(self, ec): return self.p_loc @ ec
        def coarse(self, rc): return np.linalg.solve(self.a1, rc)

    g = sp.csr_matrix((cfg.g_vals, cfg.g_cols, cfg.g_rowptr), shape=(cfg.m, cfg.n))
    plan = pdist.build_plan(g, cfg.level0_partition, int(cfg.level0_n_aggregates), int(over.get("level0_overlap", 1)), comm)
    ops = CpuOps(plan)
    p0, coff = pdist.gather_p0(plan, ops.p_loc, cfg.n, comm)
    g1 = (g @ p0).toarray()
    ops.a1 = g1.T @ g1
    return plan, pdist.DistSolver(plan, ops, comm, coff)


def _global_oracle(cfg, over):
    from oracle import refbind

    return refbind.oracle().setup(cfg, refbind.params_for(cfg, **over))


DIST_CASES = [("c3", 32, {"thresh_override": 10.0, "max_levels": 2}),
              ("c2", 24, {"thresh_override": 10.0, "max_levels": 2})]


def _dist_rank_check(cfg, comm, over, out):
    import numpy as np

    kw = dict(cfg.params)
    kw.update(over)
    kw.pop("level0_partition", None)
    kw.pop("level0_n_aggregates", None)
    plan, solver = _cpu_ops_and_solver(cfg, comm, kw)
    ho = _global_oracle(cfg, over)
    assert ho.num_levels == 2
    r = cfg.rhs
    e = solver.vcycle(r[plan.own])
    eo = ho.vcycle(r)
    x, its, conv, hist = solver.pcg(r[plan.own], 1e-8, 1000)
    xo, repo = ho.pcg(r, 1e-8, 1000)
    out[comm.rank] = dict(
        vc=float(np.linalg.norm(e - eo[plan.own]) / np.linalg.norm(eo)),
        ap=float(np.linalg.norm(solver.apply_a(r[plan.own]) - (ho.spmv(ho.spmv(r, 0, 1, False, cfg.m), 0, 1, True, cfg.n))[plan.own])),
        its=its, its_ref=int(repo["iterations"]), conv=conv,
        x=float(np.linalg.norm(x - xo[plan.own]) / np.linalg.norm(xo)), n_own=int(plan.own.shape[0]),
        halo=int(sum(v.shape[0] for v in plan.recv.values())))


@pytest.mark.parametrize("name,grid,over", DIST_CASES)
@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_solve_equals_single_process(name, grid, over, world):
    """Ranks as threads (ThreadComm): strips with 1- and 2-cell halos reproduce the oracle's V-cycle
    (1e-10), operator application and PCG (iterations ±1, solution 1e-8)."""
    import threading

    from paper_2601_04112_b200 import configs, dist as pdist

    cfg = configs.config(name, grid)
    hub = pdist.ThreadComm.Hub(world)
    out, errs = {}, []

    def work(rank):
        try:
            _dist_rank_check(cfg, pdist.ThreadComm(hub, rank), over, out)
        except Exception as e:  # surface worker failures in the main thread
            errs.append(repr(e))
            hub.barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    assert sum(o["n_own"] for o in out.values()) == cfg.n
    for o in out.values():
        assert o["halo"] > 0
        assert o["vc"] <= 1e-10 and o["ap"] <= 1e-9
        assert o["conv"] and abs(o["its"] - o["its_ref"]) <= 1 and o["x"] <= 1e-8


def _gloo_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    from paper_2601_04112_b200 import configs, dist as pdist

    name, grid, over = DIST_CASES[0]
    cfg = configs.config(name, grid)
    res = {}
    _dist_rank_check(cfg, pdist.TorchComm(dist, "cpu"), over, res)
    out[rank] = res[rank]
    dist.destroy_process_group()


def test_partitioned_solve_gloo_world2():
    """The same check with one process per rank over torch.distributed (gloo)."""
    out = mp.Manager().dict()
    mp.spawn(_gloo_worker, args=(2, 29741, out), nprocs=2, join=True)
    for r in (0, 1):
        o = out[r]
        assert o["vc"] <= 1e-10 and o["conv"] and abs(o["its"] - o["its_ref"]) <= 1 and o["x"] <= 1e-8
