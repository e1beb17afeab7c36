"""QAOA MaxCut energy expectation driver on B200.

No reference counterpart exists; the driver is built on the
reference-named primitives mirrored in this package:

    E(gamma, beta) = sum_{(i,j) in E} (1 - <Z_i Z_j>) / 2

with each <Z_i Z_j> the contraction of the edge's light-cone network
(lightcone.py).  `EnergyPlan` is the plan cache: per edge the network
template, the reference rgreedy order and the compiled bucket program are
computed once; every evaluation then runs, for any number of angle sets:

    tensorgen (angles -> gate tensors, on device)
      -> SMEM executor: one launch, one warp per (edge network, angle set)
      -> HBM executor: fused per-bucket kernels for the wide networks
      -> energy reduction

Multi-GPU: `shard_edges` splits the edges by longest-processing-time on
CostReport.flops_sum (ordering.py:60-61); each rank evaluates its shard and a
single all-reduce of the per-set partial energies (float64) finishes the job.
"""

from __future__ import annotations

import ctypes as C
import heapq
import time

import numpy as np

from . import _native as N
from .circuit import ProblemGraph, QaoaParams
from .contraction import (DEFAULT_MIXED_RANK, DEFAULT_RANK_CAP, DEFAULT_SMEM_BUDGET,
                          ContractionPlan)
from .lightcone import EnergyTemplate, energy_template
from .ordering import ContractionOrder, CostReport, rgreedy_order

__all__ = ["EdgeJob", "EnergyPlan", "plan_edges", "shard_edges", "rank_shard", "reduce_partials",
           "energy_expectation"]


class EdgeJob:
    """Template + order + compiled plan of one edge network."""

    def __init__(self, index: int, template: EnergyTemplate, order: ContractionOrder,
                 report: CostReport, plan: ContractionPlan):
        self.index = index
        self.template = template
        self.order = order
        self.report = report
        self.plan = plan


def plan_edges(graph: ProblemGraph, p: int, mode: str, edge_ids, rank_cap=DEFAULT_RANK_CAP,
               dtype="complex64", mixed_rank=DEFAULT_MIXED_RANK, smem_budget=DEFAULT_SMEM_BUDGET,
               n_repeats=10, temp=0.02, seed=0, compile_plans=True):
    """Host planning for a set of edges: template, rgreedy order, plan."""
    jobs = []
    for e in edge_ids:
        tpl = energy_template(graph, graph.edges[e], p, mode)
        order, report = rgreedy_order(tpl.line_graph(), n_repeats=n_repeats, temp=temp, seed=seed)
        plan = None
        if compile_plans:
            plan = ContractionPlan(tpl.structure, tpl.variable_count, tpl.fixed, order.sequence,
                                   rank_cap=rank_cap, dtype=dtype, mixed_rank=mixed_rank,
                                   smem_budget=smem_budget)
        jobs.append(EdgeJob(e, tpl, order, report, plan))
    return jobs


def shard_edges(costs, world_size: int):
    """LPT partition: heaviest first onto the least-loaded rank; ties by rank
    id; each shard returned in ascending edge order (deterministic)."""
    heap = [(0.0, r) for r in range(world_size)]
    heapq.heapify(heap)
    shards = [[] for _ in range(world_size)]
    for e in sorted(range(len(costs)), key=lambda k: (-costs[k], k)):
        load, r = heapq.heappop(heap)
        shards[r].append(e)
        heapq.heappush(heap, (load + float(costs[e]), r))
    return [sorted(s) for s in shards]


class EnergyPlan:
    """Cached plans for the energy of `graph` at depth p over `edge_ids`."""

    def __init__(self, graph: ProblemGraph, p: int, mode: str = "zz+diagonal",
                 dtype="complex64", edge_ids=None, rank_cap=DEFAULT_RANK_CAP,
                 mixed_rank=DEFAULT_MIXED_RANK, smem_budget=DEFAULT_SMEM_BUDGET,
                 n_repeats=10, temp=0.02, seed=0, jobs=None):
        self.graph = graph
        self.p = p
        self.mode = mode
        self.edge_ids = list(range(graph.edge_count)) if edge_ids is None else list(edge_ids)
        t0 = time.perf_counter()
        if jobs is None:
            jobs = plan_edges(graph, p, mode, self.edge_ids, rank_cap, dtype, mixed_rank,
                              smem_budget, n_repeats, temp, seed)
        self.jobs = jobs
        self.plan_seconds = time.perf_counter() - t0
        self.smem_jobs = [j for j in jobs if j.plan.executor == N.EXEC_SMEM]
        self.hbm_jobs = [j for j in jobs if j.plan.executor == N.EXEC_HBM]
        self._device = None
        self._bufs = {}

    # ---------------------------------------------------------- statistics
    @property
    def widths(self):
        return [j.report.width for j in self.jobs]

    @property
    def alg_bytes(self) -> float:
        """Algorithmic bytes of one evaluation (one angle set)."""
        return float(sum(j.plan.alg_bytes for j in self.jobs))

    @property
    def flops_sum(self) -> float:
        return float(sum(j.report.flops_sum for j in self.jobs))

    # ---------------------------------------------------------- device side
    def _prepare(self):
        if self._device is not None:
            return
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("a CUDA device is required: the B200 backend has no CPU fallback")
        dev = torch.device("cuda", torch.cuda.current_device())
        self._torch = torch
        self._device = dev
        # input-set layout: [SMEM batch inputs | HBM network 0 | HBM network 1 | ...]
        self._batch = None
        base = 0
        recs = []
        if self.smem_jobs:
            arr = (C.c_void_p * len(self.smem_jobs))(*[j.plan.handle for j in self.smem_jobs])
            b = C.c_void_p()
            N.check(N.lib.qtn_batch_create(arr, len(self.smem_jobs), C.byref(b)), "batch create")
            self._batch = b
            nel = C.c_int64()
            N.check(N.lib.qtn_batch_input_elems(b, C.byref(nel)))
            offs = np.zeros(len(self.smem_jobs), dtype=np.int64)
            N.check(N.lib.qtn_batch_input_offsets(b, N.i64(offs)))
            for j, o in zip(self.smem_jobs, offs):
                r = j.template.recipes.copy()
                r["out_offset"] = j.plan.input_offsets + o
                recs.append(r)
            base = int(nel.value)
        self._hbm_offsets = []
        for j in self.hbm_jobs:
            base = (base + 1) & ~1
            r = j.template.recipes.copy()
            r["out_offset"] = j.plan.input_offsets + base
            recs.append(r)
            self._hbm_offsets.append(base)
            base += j.plan.input_elems
        self.set_elems = max(base, 2)
        allrec = np.concatenate(recs) if recs else np.zeros(0, dtype=N.RECIPE_DTYPE)
        self._n_recipes = len(allrec)
        self._recipes = torch.from_numpy(allrec.view(np.uint8).copy()).to(dev)
        ws = max([j.plan.workspace_bytes for j in self.hbm_jobs] or [16])
        self._ws = torch.empty(ws, dtype=torch.uint8, device=dev)

    def _buffers(self, n_sets):
        if n_sets not in self._bufs:
            t = self._torch
            dev = self._device
            self._bufs[n_sets] = dict(
                inputs=t.zeros(n_sets * self.set_elems, dtype=t.complex128, device=dev),
                res_smem=t.zeros((n_sets, max(len(self.smem_jobs), 1)), dtype=t.complex128, device=dev),
                res_hbm=t.zeros((n_sets, max(len(self.hbm_jobs), 1)), dtype=t.complex128, device=dev),
                e_smem=t.zeros(n_sets, dtype=t.float64, device=dev),
                e_hbm=t.zeros(n_sets, dtype=t.float64, device=dev),
            )
        return self._bufs[n_sets]

    def launch(self, angles_dev, stream=None):
        """Enqueue one evaluation for every angle set in `angles_dev`
        ([n_sets, 2p] float64 on the device).  Returns the buffer dict; the
        energies are bufs['e_smem'] + bufs['e_hbm'] once the stream is done.
        Kernel launches: 1 tensorgen + 1 SMEM batch + per-bucket HBM + reductions."""
        self._prepare()
        t = self._torch
        n_sets = int(angles_dev.shape[0])
        b = self._buffers(n_sets)
        st = stream if stream is not None else t.cuda.current_stream(self._device)
        sp = st.cuda_stream
        N.check(N.lib.qtn_tensorgen(self._recipes.data_ptr(), self._n_recipes,
                                    angles_dev.data_ptr(), 2 * self.p, n_sets, self.set_elems,
                                    b["inputs"].data_ptr(), sp), "tensorgen")
        self.launches = 1
        if self._batch is not None:
            N.check(N.lib.qtn_batch_execute(self._batch, b["inputs"].data_ptr(), self.set_elems,
                                            n_sets, b["res_smem"].data_ptr(), sp), "batch")
            N.check(N.lib.qtn_energy_reduce(b["res_smem"].data_ptr(), len(self.smem_jobs), n_sets,
                                            b["e_smem"].data_ptr(), None, sp), "energy")
            self.launches += 2
        if self.hbm_jobs:
            esz = 16
            ip = b["inputs"].data_ptr()
            rp = b["res_hbm"].data_ptr()
            nh = len(self.hbm_jobs)
            for s in range(n_sets):
                for k, (j, off) in enumerate(zip(self.hbm_jobs, self._hbm_offsets)):
                    j.plan.execute(ip + esz * (s * self.set_elems + off), self._ws.data_ptr(),
                                   rp + esz * (s * nh + k), sp)
                    self.launches += j.plan.n_buckets + 1
            N.check(N.lib.qtn_energy_reduce(rp, nh, n_sets, b["e_hbm"].data_ptr(), None, sp),
                    "energy")
            self.launches += 1
        return b

    def energies(self, angle_sets) -> np.ndarray:
        """Energy per angle set; angle_sets: QaoaParams, a [2p] vector or an
        [n_sets, 2p] array of [gammas..., betas...]."""
        self._prepare()
        t = self._torch
        if isinstance(angle_sets, QaoaParams):
            angle_sets = angle_sets.as_vector()
        a = np.atleast_2d(np.asarray(angle_sets, dtype=np.float64))
        if a.shape[1] != 2 * self.p:
            raise ValueError(f"expected {2 * self.p} angles per set, got {a.shape[1]}")
        dev_a = t.from_numpy(a).pin_memory().to(self._device, non_blocking=True)
        b = self.launch(dev_a)
        out = (b["e_smem"] if self.smem_jobs else 0) + (b["e_hbm"] if self.hbm_jobs else 0)
        return out.cpu().numpy().copy()

    def zz_values(self, params: QaoaParams) -> dict:
        """Per-edge <Z_iZ_j> (complex) for one angle set, keyed by edge index."""
        self._prepare()
        t = self._torch
        a = t.from_numpy(np.atleast_2d(params.as_vector())).to(self._device)
        b = self.launch(a)
        out = {}
        rs = b["res_smem"][0].cpu().numpy()
        rh = b["res_hbm"][0].cpu().numpy()
        for k, j in enumerate(self.smem_jobs):
            out[j.index] = complex(rs[k])
        for k, j in enumerate(self.hbm_jobs):
            out[j.index] = complex(rh[k])
        return out

    def __del__(self):
        b = getattr(self, "_batch", None)
        if b is not None and N is not None and N.lib is not None:
            N.lib.qtn_batch_destroy(b)
            self._batch = None


def rank_shard(graph: ProblemGraph, p: int, mode: str, rank: int, world: int,
               n_repeats=10, temp=0.02, seed=0):
    """This rank's edges: LPT over the reference cost model.  Every rank
    computes the same (deterministic) orders, so no exchange is needed."""
    allj = plan_edges(graph, p, mode, range(graph.edge_count), compile_plans=False,
                      n_repeats=n_repeats, temp=temp, seed=seed)
    return shard_edges([j.report.flops_sum for j in allj], world)[rank]


def reduce_partials(partial: np.ndarray, group=None, device=None) -> np.ndarray:
    """Sum per-angle-set partial energies over the ranks (one all_reduce;
    NCCL on GPUs, gloo on CPU)."""
    import torch

    dist = torch.distributed
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return partial
    buf = torch.tensor(np.asarray(partial, dtype=np.float64),
                       device=device if device is not None else "cpu")
    dist.all_reduce(buf, group=group)
    return buf.cpu().numpy()


def energy_expectation(graph: ProblemGraph, params: QaoaParams, mode: str = "zz+diagonal",
                       dtype="complex64", plan: EnergyPlan | None = None, group=None,
                       **kw) -> float:
    """E(gamma, beta) on the GPU(s).  With an initialised torch.distributed
    process group the edges are LPT-sharded over the ranks and the partial
    energies are all-reduced (one collective)."""
    import torch

    dist = torch.distributed
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if plan is None:
        edge_ids = None
        if world > 1:
            edge_ids = rank_shard(graph, params.p, mode, dist.get_rank(group), world,
                                  **{k: v for k, v in kw.items()
                                     if k in ("n_repeats", "temp", "seed")})
        plan = EnergyPlan(graph, params.p, mode, dtype, edge_ids=edge_ids, **kw)
    e = plan.energies(params)
    dev = torch.device("cuda", torch.cuda.current_device()) if world > 1 else None
    return float(reduce_partials(e, group, dev)[0])
