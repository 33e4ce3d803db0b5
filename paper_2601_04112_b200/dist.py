"""Row/aggregate partition of the hot path over the GPUs of one node
(SURVEY.md §8(e)): contiguous strips (2-D) or slabs (3-D) of level-0
aggregates, one process per GPU.

* Setup. Level-0 aggregates are independent units: every rank builds the
  local GEVPs, the Schwarz blocks and the P panels of its own aggregates from
  the rows of G that touch them (its strip plus one layer of halo
  aggregates, whose results are discarded). The panels are all-gathered; the
  Galerkin product G₁ = G₀P₀ and the coarse hierarchy (levels ≥ 1, built with
  ``level_offset = 1``) are replicated on every rank — the reference's coarse
  aggregation is sequential and must stay bit-exact (aggregation.hpp:71-117).
* Solve. PCG on the strips: halo exchange of the owner's values before every
  SpMV and Schwarz gather, reverse-halo add after Gᵀ and after the RAS-T
  scatter (smoother.hpp:79-80), one fused all-reduce per group of PCG dots
  (krylov.hpp:62-76), all-gather of the restricted residual and a replicated
  coarse cycle (hierarchy.hpp:209).

The numerical work of a rank goes through ``LocalOps`` — on a B200 the C ABI
(``GpuOps``: strip handle, matrix handles, coarse handle, device vectors); the
CPU tests plug numpy operators into the same driver to check the partition,
the halo maps and the collectives against the single-process result.
Collectives go through a ``Comm``: ``TorchComm`` (torch.distributed, NCCL on
GPUs / gloo on CPU) or ``ThreadComm`` (ranks as threads of one process, used to
run the partitioned path on a single GPU without kernels waiting on each
other).
"""
from __future__ import annotations

import threading
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np
import scipy.sparse as sp


# ---- communicators ---------------------------------------------------------------------------


class Comm:
    rank: int
    world: int

    def allgather(self, arr: np.ndarray) -> list:
        """Arrays of every rank (variable lengths), in rank order."""
        raise NotImplementedError

    def allreduce_sum(self, vals: np.ndarray) -> np.ndarray:
        """Sum over ranks in rank order (deterministic)."""
        parts = self.allgather(np.ascontiguousarray(vals, dtype=np.float64))
        out = parts[0].copy()
        for p in parts[1:]:
            out = out + p
        return out

    def exchange(self, send: dict) -> dict:
        """Point-to-point exchange: send[dst] -> returns recv[src] (float64 arrays)."""
        raise NotImplementedError


class TorchComm(Comm):
    """torch.distributed process group (NCCL between GPUs, gloo on CPU)."""

    def __init__(self, dist_module, device="cpu"):
        self.d = dist_module
        self.rank = dist_module.get_rank()
        self.world = dist_module.get_world_size()
        self.device = device

    def _t(self, a):
        import torch

        return torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def allgather(self, arr):
        import torch

        arr = np.ascontiguousarray(arr)
        n = torch.tensor([arr.shape[0]], dtype=torch.int64, device=self.device)
        ns = [torch.zeros_like(n) for _ in range(self.world)]
        self.d.all_gather(ns, n)
        sizes = [int(x.item()) for x in ns]
        mx = max(sizes + [1])
        buf = torch.zeros(mx, dtype=self._t(arr[:0]).dtype if arr.shape[0] == 0 else self._t(arr[:1]).dtype, device=self.device)
        if arr.shape[0]:
            buf[: arr.shape[0]] = self._t(arr)
        outs = [torch.zeros_like(buf) for _ in range(self.world)]
        self.d.all_gather(outs, buf)
        return [o[:k].cpu().numpy() for o, k in zip(outs, sizes)]

    def exchange(self, send):
        import torch

        # sizes first, then one all_to_all of the padded payloads (neighbours only carry data)
        counts = np.zeros(self.world, dtype=np.int64)
        for dst, a in send.items():
            counts[dst] = a.shape[0]
        all_counts = self.allgather(counts)
        recv_counts = [int(all_counts[src][self.rank]) for src in range(self.world)]
        ins = [self._t(send[dst]) if dst in send else torch.zeros(0, dtype=torch.float64, device=self.device)
               for dst in range(self.world)]
        outs = [torch.zeros(k, dtype=torch.float64, device=self.device) for k in recv_counts]
        self.d.all_to_all(outs, ins) if self.d.get_backend() != "gloo" else self._gloo_all_to_all(outs, ins)
        return {src: outs[src].cpu().numpy() for src in range(self.world) if recv_counts[src]}

    def _gloo_all_to_all(self, outs, ins):
        # gloo has no all_to_all: ordered pairwise send/recv
        reqs = []
        for peer in range(self.world):
            if peer == self.rank:
                outs[peer].copy_(ins[peer])
                continue
            if ins[peer].numel():
                reqs.append(self.d.isend(ins[peer], peer))
            if outs[peer].numel():
                reqs.append(self.d.irecv(outs[peer], peer))
        for r in reqs:
            r.wait()


class ThreadComm(Comm):
    """Ranks as threads of one process (shared mailbox + barrier)."""

    class Hub:
        def __init__(self, world: int):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world
            self.mail = [dict() for _ in range(world)]

    def __init__(self, hub: "ThreadComm.Hub", rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world

    def allgather(self, arr):
        self.hub.slots[self.rank] = np.array(arr, copy=True)
        self.hub.barrier.wait()
        out = [self.hub.slots[r].copy() for r in range(self.world)]
        self.hub.barrier.wait()
        return out

    def exchange(self, send):
        for dst, a in send.items():
            self.hub.mail[dst][self.rank] = np.array(a, copy=True)
        self.hub.barrier.wait()
        got = dict(self.hub.mail[self.rank])
        self.hub.barrier.wait()
        self.hub.mail[self.rank].clear()
        self.hub.barrier.wait()
        return got


# ---- the partition ---------------------------------------------------------------------------


def aggregate_ranges(n_agg: int, world: int) -> list:
    """Contiguous aggregate-id ranges: strips of block rows in 2-D, z-slabs in 3-D
    (the configs number their level-0 blocks lexicographically)."""
    base, rem = divmod(n_agg, world)
    out, a = [], 0
    for r in range(world):
        b = a + base + (1 if r < rem else 0)
        out.append((a, b))
        a = b
    return out


@dataclass
class StripPlan:
    rank: int
    world: int
    agg_range: tuple          # owned aggregates [a0, a1)
    own: np.ndarray           # owned nodes (global ids, ascending)
    ext: np.ndarray           # nodes of the strip sub-problem: owned aggregates + halo aggregates (global, ascending)
    own_in_ext: np.ndarray    # positions of the owned nodes inside ext
    sub_aggs: np.ndarray      # global ids of the sub-problem's aggregates (ascending)
    sub_part: np.ndarray      # node -> local aggregate id over ext
    g_sub: sp.csr_matrix      # rows of G touching ext, columns restricted to ext (row order kept)
    g_own_rows: np.ndarray    # rows of G owned by this rank (min column node owned), as indices into g_sub's rows
    recv: dict                # src rank -> positions in ext filled from that owner
    send: dict                # dst rank -> positions in own sent to that rank's halo


def build_plan(g: sp.csr_matrix, part: np.ndarray, n_agg: int, overlap: int, comm: Comm) -> StripPlan:
    """Strip plan of this rank (collective: the halo lists are exchanged)."""
    rank, world = comm.rank, comm.world
    a0, a1 = aggregate_ranges(n_agg, world)[rank]
    n = g.shape[1]
    own = np.flatnonzero((part >= a0) & (part < a1))
    pat = g.copy()
    pat.data[:] = 1.0
    # Ω of the owned aggregates: `overlap` graph layers of A = GᵀG around the owned nodes
    mask = np.zeros(n, dtype=bool)
    mask[own] = True
    gt = pat.T.tocsr()
    for _ in range(max(1, overlap)):
        rows = np.flatnonzero(pat @ mask.astype(np.float64))
        sel = np.zeros(g.shape[0])
        sel[rows] = 1.0
        mask |= (gt @ sel) > 0
    sub_aggs = np.unique(part[mask])
    in_sub = np.zeros(n_agg, dtype=bool)
    in_sub[sub_aggs] = True
    ext = np.flatnonzero(in_sub[part])
    loc_of = -np.ones(n, dtype=np.int64)
    loc_of[ext] = np.arange(ext.shape[0])
    agg_loc = -np.ones(n_agg, dtype=np.int64)
    agg_loc[sub_aggs] = np.arange(sub_aggs.shape[0])
    sub_part = agg_loc[part[ext]]
    # rows of G touching ext, restricted to ext columns
    ext_mask = np.zeros(n)
    ext_mask[ext] = 1.0
    rows = np.flatnonzero(pat @ ext_mask)
    g_rows = g[rows]
    keep = sp.csr_matrix((np.ones(ext.shape[0]), (ext, np.arange(ext.shape[0]))), shape=(n, ext.shape[0]))
    g_sub = (g_rows @ keep).tocsr()
    g_sub.sort_indices()
    # a row belongs to the owner of its first (lowest-index) node
    first_col = g.indices[g.indptr[rows]]
    own_rows = np.flatnonzero((part[first_col] >= a0) & (part[first_col] < a1))
    # halo lists: which of my ext nodes are owned elsewhere, and who needs mine
    ranges = aggregate_ranges(n_agg, world)
    owner = np.empty(n_agg, dtype=np.int64)
    for r, (b0, b1) in enumerate(ranges):
        owner[b0:b1] = r
    ext_owner = owner[part[ext]]
    recv = {int(src): np.flatnonzero(ext_owner == src) for src in np.unique(ext_owner) if src != rank}
    wanted = comm.allgather(ext)  # every rank's ext nodes (global ids)
    own_pos = -np.ones(n, dtype=np.int64)
    own_pos[own] = np.arange(own.shape[0])
    send = {}
    for dst in range(world):
        if dst == rank:
            continue
        mine = wanted[dst][(part[wanted[dst]] >= a0) & (part[wanted[dst]] < a1)]
        if mine.shape[0]:
            send[dst] = own_pos[mine]
    return StripPlan(rank, world, (a0, a1), own, ext, loc_of[own], sub_aggs, sub_part, g_sub, own_rows, recv, send)


# ---- local operators -------------------------------------------------------------------------


class LocalOps:
    """What one rank computes on its strip. Vectors are numpy float64 (the GPU
    operators keep the data on the device between calls where it matters)."""

    n_own: int
    n_ext: int
    n_coarse_own: int

    def g_apply(self, p_ext): raise NotImplementedError          # rows owned: G_own p_ext
    def gt_apply(self, q_own): raise NotImplementedError         # G_ownᵀ q -> ext vector
    def a_apply(self, e_ext): raise NotImplementedError          # A₀ rows of the owned nodes
    def ras(self, r_ext): raise NotImplementedError              # -> ext vector (owned entries valid)
    def rast(self, r_ext): raise NotImplementedError             # -> ext vector of contributions
    def restrict(self, res_own): raise NotImplementedError       # P_locᵀ res
    def prolong(self, ec_own): raise NotImplementedError         # P_loc ec
    def coarse(self, rc_global): raise NotImplementedError       # replicated cycle on levels >= 1


class DistSolver:
    """Distributed V(1,1)-preconditioned CG over the strips."""

    def __init__(self, plan: StripPlan, ops: LocalOps, comm: Comm, coarse_offsets: Sequence[int]):
        self.plan, self.ops, self.comm = plan, ops, comm
        self.coff = list(coarse_offsets)  # global coarse column offsets per rank (world + 1)

    # -- halo plumbing
    def halo_fill(self, x_own: np.ndarray) -> np.ndarray:
        p = self.plan
        x_ext = np.zeros(p.ext.shape[0])
        x_ext[p.own_in_ext] = x_own
        got = self.comm.exchange({dst: x_own[idx] for dst, idx in p.send.items()})
        for src in sorted(got):
            x_ext[p.recv[src]] = got[src]
        return x_ext

    def reverse_add(self, y_ext: np.ndarray) -> np.ndarray:
        """Owned part of y_ext plus what the other ranks computed for my nodes (ascending rank order)."""
        p = self.plan
        y_own = y_ext[p.own_in_ext].copy()
        got = self.comm.exchange({src: y_ext[idx] for src, idx in p.recv.items()})
        for dst in sorted(got):
            y_own[p.send[dst]] += got[dst]
        return y_own

    # -- operators
    def apply_a(self, p_own: np.ndarray) -> np.ndarray:
        """Gᵀ(G p) (lsamgdd_cli.cpp:137-142) on the strip."""
        q = self.ops.g_apply(self.halo_fill(p_own))
        return self.reverse_add(self.ops.gt_apply(q))

    def vcycle(self, r_own: np.ndarray) -> np.ndarray:
        """hierarchy.hpp:205-227 with level 0 on the strips and levels >= 1 replicated."""
        ops = self.ops
        e_own = ops.ras(self.halo_fill(r_own))[self.plan.own_in_ext]
        res = r_own - ops.a_apply(self.halo_fill(e_own))
        rc = np.concatenate(self.comm.allgather(ops.restrict(res)))
        ec = ops.coarse(rc)
        e_own = e_own + ops.prolong(ec[self.coff[self.comm.rank]: self.coff[self.comm.rank + 1]])
        res = r_own - ops.a_apply(self.halo_fill(e_own))
        r_ext = np.zeros(self.plan.ext.shape[0])
        r_ext[self.plan.own_in_ext] = res  # halo aggregates see a zero residual: they contribute nothing
        return e_own + self.reverse_add(ops.rast(r_ext))

    def dots(self, *pairs) -> np.ndarray:
        return self.comm.allreduce_sum(np.array([float(a @ b) for a, b in pairs]))

    def pcg(self, b_own: np.ndarray, tol: float = 1e-8, maxit: int = 1000):
        """krylov.hpp:42-92; returns (x_own, iterations, converged, residual history)."""
        x = np.zeros_like(b_own)
        r = b_own.copy()
        r0 = float(np.sqrt(self.dots((r, r))[0]))
        hist = [r0]
        if r0 == 0.0:
            return x, 0, True, hist
        z = self.vcycle(r)
        rz = float(self.dots((r, z))[0])
        if not rz > 0.0:
            raise ArithmeticError("pcg: preconditioned product <r, Br> is not positive")
        p = z.copy()
        k, converged = 0, False
        while k < maxit:
            ap = self.apply_a(p)
            pap = float(self.dots((p, ap))[0])
            if not pap > 0.0:
                raise ArithmeticError("pcg: curvature <p, Ap> is not positive")
            alpha = rz / pap
            x += alpha * p
            r -= alpha * ap
            k += 1
            rn = float(np.sqrt(self.dots((r, r))[0]))
            hist.append(rn)
            if rn <= tol * r0:
                converged = True
                break
            z = self.vcycle(r)
            rz_next = float(self.dots((r, z))[0])
            if not rz_next > 0.0:
                raise ArithmeticError("pcg: preconditioned product <r, Br> is not positive")
            p = z + (rz_next / rz) * p
            rz = rz_next
        return x, k, converged, hist


# ---- B200 operators through the C ABI ----------------------------------------------------------


class GpuOps(LocalOps):
    """Strip operators on the rank's GPU: the level-0 stages of the strip sub-problem
    (lsamgdd_setup with probe_levels = 1), matrix handles for G_own, A_own and P_loc,
    and the replicated coarse hierarchy (level_offset = 1)."""

    def __init__(self, plan: StripPlan, cfg, comm: Comm, params_over: Optional[dict] = None):
        from . import abi, lsamgdd

        self.plan = plan
        self._lsamgdd = lsamgdd
        self._abi = abi
        self._lib = lsamgdd.library()
        self._keep = []
        over = dict(cfg.params)
        over.update(params_over or {})
        over.pop("level0_partition", None)
        over.pop("level0_n_aggregates", None)
        over["coarse_size"] = 1  # the strip always builds its level-0 stages (probe_levels stops it there)
        gs = plan.g_sub
        sub = (gs.indptr.astype(np.int64), gs.indices.astype(np.int64), gs.data.astype(np.float64), gs.shape[1])
        self.h_strip = lsamgdd.setup(sub, lsamgdd.LevelParams(level0_partition=plan.sub_part.astype(np.int64),
                                                              level0_n_aggregates=int(plan.sub_aggs.shape[0]),
                                                              probe_levels=1, **over))
        self.n_own, self.n_ext = plan.own.shape[0], plan.ext.shape[0]
        # P of the owned aggregates: rows of the owned nodes, columns of the owned aggregates
        pm = self.h_strip.levels[0].P
        p_sub = sp.csr_matrix((pm.values, pm.col_indices, pm.row_offsets), shape=(pm.n_rows, pm.n_cols))
        self.p_loc = slice_own_p(plan, p_sub)
        self.n_coarse_own = self.p_loc.shape[1]
        am = self.h_strip.levels[0].A
        a_sub = sp.csr_matrix((am.values, am.col_indices, am.row_offsets), shape=(am.n_rows, am.n_cols))
        self.m_g = self._matrix(gs[plan.g_own_rows].tocsr())
        self.m_a = self._matrix(a_sub[plan.own_in_ext].tocsr())
        self.m_p = self._matrix(self.p_loc)
        self.h_coarse = None

    def _matrix(self, m: sp.csr_matrix):
        import ctypes as C

        m.sort_indices()
        rp, ci, va = m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data.astype(np.float64)
        csr = self._abi.csr_struct(rp, ci, va, m.shape[1])
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        self._lsamgdd._check(self._lib.lsamgdd_matrix_create(C.byref(csr), C.byref(h), err, C.c_size_t(1024)), err)
        self._keep.append((rp, ci, va))
        return (h, m.shape)

    def _spmv(self, mat, x, transpose: bool):
        import ctypes as C

        h, shape = mat
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(shape[1] if transpose else shape[0])
        err = C.create_string_buffer(1024)
        self._lsamgdd._check(self._lib.lsamgdd_matrix_spmv(h, C.c_int32(1 if transpose else 0), self._abi.ptr(x), self._abi.ptr(y),
                                                            C.c_int32(self._abi.HOST), err, C.c_size_t(1024)), err)
        return y

    def set_coarse(self, g1: sp.csr_matrix, cfg, params_over: Optional[dict] = None):
        """Replicated hierarchy of the levels >= 1 from the gathered G₁ = G₀P₀."""
        over = {k: v for k, v in dict(cfg.params).items() if not k.startswith("level0_")}
        over.update(params_over or {})
        g1.sort_indices()
        arr = (g1.indptr.astype(np.int64), g1.indices.astype(np.int64), g1.data.astype(np.float64), g1.shape[1])
        self.h_coarse = self._lsamgdd.setup(arr, self._lsamgdd.LevelParams(level_offset=1, **over))

    def g_apply(self, p_ext): return self._spmv(self.m_g, p_ext, False)
    def gt_apply(self, q_own): return self._spmv(self.m_g, q_own, True)
    def a_apply(self, e_ext): return self._spmv(self.m_a, e_ext, False)
    def ras(self, r_ext): return self._lsamgdd.apply(self.h_strip, 0, r_ext, self._lsamgdd.RAS)
    def rast(self, r_ext): return self._lsamgdd.apply(self.h_strip, 0, r_ext, self._lsamgdd.RAST)
    def restrict(self, res_own): return self._spmv(self.m_p, res_own, True)
    def prolong(self, ec_own): return self._spmv(self.m_p, ec_own, False)
    def coarse(self, rc_global): return self._lsamgdd.vcycle(self.h_coarse, rc_global, 0)

    def close(self):
        for h, _ in (self.m_g, self.m_a, self.m_p):
            self._lib.lsamgdd_matrix_destroy(h)


def slice_own_p(plan: StripPlan, p_sub: sp.csr_matrix) -> sp.csr_matrix:
    """Rows of the owned nodes and columns of the owned aggregates of the strip's P."""
    csc = p_sub.tocsc()
    col_agg = plan.sub_part[csc.indices[csc.indptr[:-1]]]  # aggregate of a column: that of any of its rows
    own_local = np.flatnonzero((plan.sub_aggs >= plan.agg_range[0]) & (plan.sub_aggs < plan.agg_range[1]))
    own_cols = np.flatnonzero(np.isin(col_agg, own_local))
    return p_sub[plan.own_in_ext][:, own_cols].tocsr()


def gather_p0(plan: StripPlan, p_loc: sp.csr_matrix, n: int, comm: Comm):
    """All-gather of the owned P panels: (global P₀ as CSR, coarse offsets per rank)."""
    counts = comm.allgather(np.array([p_loc.shape[1]], dtype=np.int64))
    coff = np.concatenate([[0], np.cumsum([int(c[0]) for c in counts])])
    coo = p_loc.tocoo()
    rows = comm.allgather(plan.own[coo.row].astype(np.int64))
    cols = comm.allgather((coo.col + coff[comm.rank]).astype(np.int64))
    vals = comm.allgather(coo.data.astype(np.float64))
    p0 = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, int(coff[-1])))
    p0.sort_indices()
    return p0, coff


def build_gpu_solver(cfg, comm: Comm, params_over: Optional[dict] = None,
                     spgemm: Optional[Callable] = None, level0_thresh: Optional[float] = None) -> DistSolver:
    """The partitioned solver of a BASELINE config on this rank's GPU (collective).

    level0_thresh: the global level-0 threshold when the config leaves it to the reference's
    rule (eigen_threshold needs the global colour count and multiplicity bound, splitting.hpp:
    170-180); the strips then use it directly, the coarse hierarchy keeps the rule."""
    g = sp.csr_matrix((cfg.g_vals, cfg.g_cols, cfg.g_rowptr), shape=(cfg.m, cfg.n))
    overlap = int(dict(cfg.params).get("level0_overlap", 1))
    plan = build_plan(g, cfg.level0_partition, int(cfg.level0_n_aggregates), overlap, comm)
    strip_over = dict(params_over or {})
    if level0_thresh is not None:
        strip_over["thresh_override"] = float(level0_thresh)
    ops = GpuOps(plan, cfg, comm, strip_over)
    p0, coff = gather_p0(plan, ops.p_loc, cfg.n, comm)
    g1 = (spgemm or gpu_spgemm)(g, p0)
    ops.set_coarse(g1, cfg, params_over)
    return DistSolver(plan, ops, comm, coff)


def gpu_spgemm(a: sp.csr_matrix, b: sp.csr_matrix) -> sp.csr_matrix:
    """a·b with the library's Symbolic-mode product (bit-identical to sparse.hpp:167-204)."""
    import ctypes as C

    from . import abi, lsamgdd

    lib = lsamgdd.library()
    a.sort_indices()
    b.sort_indices()
    keep = []

    def view(m):
        rp, ci, va = m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data.astype(np.float64)
        keep.append((rp, ci, va))
        return abi.csr_struct(rp, ci, va, m.shape[1])

    ca, cb = view(a), view(b)
    h = C.c_void_p()
    err = C.create_string_buffer(1024)
    lsamgdd._check(lib.lsamgdd_spgemm(C.byref(ca), C.byref(cb), C.byref(h), err, C.c_size_t(1024)), err)
    sizes = (C.c_int64 * 3)()
    lsamgdd._check(lib.lsamgdd_matrix_export(h, sizes, None, None, None))
    off = np.empty(sizes[0] + 1, np.int64)
    col = np.empty(sizes[2], np.int64)
    val = np.empty(sizes[2])
    lsamgdd._check(lib.lsamgdd_matrix_export(h, sizes, abi.ptr(off), abi.ptr(col), abi.ptr(val)))
    lib.lsamgdd_matrix_destroy(h)
    return sp.csr_matrix((val, col, off), shape=(sizes[0], sizes[1]))
