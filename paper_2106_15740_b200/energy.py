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
      -> HBM executor: one streaming launch per elimination-tree level for
         all wide networks and angle sets, then one scalar-fold launch
      -> energy reduction

Multi-GPU: `shard_edges` splits the edges by longest-processing-time on
CostReport.flops_sum (ordering.py:60-61); each rank evaluates its shard and a
single all-reduce of the per-set partial energies (float64) finishes the job.
"""

from __future__ import annotations

import heapq
import os
from concurrent.futures import ThreadPoolExecutor
import time

import numpy as np

from . import _native as N
from .circuit import ProblemGraph, QaoaParams
from .contraction import (DEFAULT_MIXED_RANK, DEFAULT_RANK_CAP, DEFAULT_SMEM_BUDGET,
                          ContractionPlan, PlanBatch)
from .lightcone import EnergyTemplate, energy_template
from .slicing import choose_slice_vars, slice_assignments
from .ordering import ContractionOrder, CostReport, rgreedy_order

__all__ = ["EdgeJob", "EnergyPlan", "plan_edges", "compile_jobs", "shard_edges", "rank_shard",
           "reduce_partials", "energy_expectation"]


class EdgeJob:
    """Template + order + compiled plan of one edge network (or of one slice
    of it: `weight` = 1/2^k, `assignment` = the sliced variables' bits)."""

    def __init__(self, index: int, template: EnergyTemplate, order: ContractionOrder,
                 report: CostReport, plan: ContractionPlan, weight: float = 1.0,
                 assignment: dict | None = None):
        self.index = index
        self.template = template
        self.order = order
        self.report = report
        self.plan = plan
        self.weight = weight
        self.assignment = assignment or {}

    @property
    def cost(self) -> float:
        return self.report.flops_sum


def plan_edges(graph: ProblemGraph, p: int, mode: str, edge_ids, rank_cap=DEFAULT_RANK_CAP,
               dtype="complex64", mixed_rank=DEFAULT_MIXED_RANK, smem_budget=DEFAULT_SMEM_BUDGET,
               n_repeats=10, temp=0.02, seed=0, compile_plans=True, slice_k: int = 0,
               workers: int | None = None):
    """Host planning for a set of edges: template, reference rgreedy order,
    compiled plan.  slice_k > 0 splits every edge network into 2^slice_k
    slices (slicing.py) that share one plan and differ only in their data.

    Edges are planned on a thread pool: the ordering
    passes and the plan compiler are native calls that release the GIL, and
    every edge is independent, so the result is identical to a serial loop
    (jobs in `edge_ids` order).  workers=1 plans serially."""
    def plan_one(e):
        out = []
        tpl = energy_template(graph, graph.edges[e], p, mode)
        order, report = rgreedy_order(tpl.line_graph(), n_repeats=n_repeats, temp=temp, seed=seed)
        assigns = [{}]
        if slice_k > 0:
            svars, _, order, report = choose_slice_vars(tpl.line_graph(), order, slice_k)
            assigns = slice_assignments(svars)
        tpls = [tpl.resliced(a) if a else tpl for a in assigns]
        for a, t in zip(assigns, tpls):
            out.append(EdgeJob(e, t, order, report, None, 1.0 / len(assigns), a))
        if compile_plans:
            compile_jobs(out, rank_cap=rank_cap, dtype=dtype, mixed_rank=mixed_rank,
                         smem_budget=smem_budget, workers=1)
        return out

    edge_ids = list(edge_ids)
    if workers is None:
        workers = min(32, os.cpu_count() or 1)
    if workers <= 1 or len(edge_ids) <= 1:
        per_edge = [plan_one(e) for e in edge_ids]
    else:
        with ThreadPoolExecutor(max_workers=min(workers, len(edge_ids))) as ex:
            per_edge = list(ex.map(plan_one, edge_ids))
    return [j for js in per_edge for j in js]


def compile_jobs(jobs, rank_cap=DEFAULT_RANK_CAP, dtype="complex64",
                 mixed_rank=DEFAULT_MIXED_RANK, smem_budget=DEFAULT_SMEM_BUDGET,
                 workers: int | None = None):
    """Compile the bucket program of every job that has none yet; the slices
    of one edge share one plan (they differ only in their data).  Lets a rank
    order every edge (the LPT partition needs all costs) but compile only the
    shard it keeps."""
    groups = {}
    for j in jobs:
        if j.plan is None:
            groups.setdefault((j.index, tuple(j.order.sequence)), []).append(j)

    def one(js):
        t0 = js[0].template
        plan = ContractionPlan(t0.structure, t0.variable_count, t0.fixed, js[0].order.sequence,
                               rank_cap=rank_cap, dtype=dtype, mixed_rank=mixed_rank,
                               smem_budget=smem_budget)
        for j in js:
            j.plan = plan

    todo = list(groups.values())
    if workers is None:
        workers = min(32, os.cpu_count() or 1)
    if workers <= 1 or len(todo) <= 1:
        for js in todo:
            one(js)
    else:
        with ThreadPoolExecutor(max_workers=min(workers, len(todo))) as ex:
            list(ex.map(one, todo))
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
                 n_repeats=10, temp=0.02, seed=0, jobs=None, slice_k: int = 0):
        self.graph = graph
        self.p = p
        self.mode = mode
        t0 = time.perf_counter()
        if jobs is None:
            ids = list(range(graph.edge_count)) if edge_ids is None else list(edge_ids)
            jobs = plan_edges(graph, p, mode, ids, rank_cap, dtype, mixed_rank,
                              smem_budget, n_repeats, temp, seed, slice_k=slice_k)
        self.jobs = list(jobs)
        self.edge_ids = sorted({j.index for j in self.jobs})
        self.plan_seconds = time.perf_counter() - t0
        if any(j.plan is None for j in self.jobs):
            compile_jobs(self.jobs, rank_cap=rank_cap, dtype=dtype, mixed_rank=mixed_rank,
                         smem_budget=smem_budget)
        self.smem_jobs = [j for j in jobs if j.plan.executor == N.EXEC_SMEM]
        self.hbm_jobs = [j for j in jobs if j.plan.executor == N.EXEC_HBM]
        self._device = None
        self._bufs = {}
        self.fused = True  # generate gate tensors inside the executors

    # ---------------------------------------------------------- statistics
    @property
    def widths(self):
        return [j.report.width for j in self.jobs]

    @property
    def alg_bytes(self) -> float:
        """Algorithmic bytes of one evaluation (one angle set)."""
        return float(sum(j.plan.alg_bytes for j in self.jobs))

    def alg_bytes_eval(self, n_sets: int) -> float:
        """Algorithmic bytes of one evaluation of n_sets angle sets, each tensor
        counted at the element size it is stored in: the
        set-major executor's complex64 rows count 8 bytes per entry."""
        self._prepare()
        if self._batch is None:
            return 0.0
        eb = self._batch.setmajor_elem_bytes(n_sets)
        small = float(sum(j.plan.alg_bytes for j in self.smem_jobs))
        big = float(sum(j.plan.alg_bytes for j in self.hbm_jobs))
        return n_sets * (big + small * (eb / 16.0 if eb else 1.0))

    def exec_bytes_eval(self, n_sets: int) -> float:
        """Bytes the HBM executor's kernels actually move for one evaluation
        (fused chains read their head operands and write their tail output
        only; everything else as alg_bytes_eval)."""
        self._prepare()
        if self._batch is None:
            return 0.0
        eb = self._batch.setmajor_elem_bytes(n_sets)
        small = float(sum(j.plan.alg_bytes for j in self.smem_jobs))
        big = float(sum(j.plan.exec_bytes for j in self.hbm_jobs))
        return n_sets * (big + small * (eb / 16.0 if eb else 1.0))

    @property
    def flops_sum(self) -> float:
        return float(sum(j.report.flops_sum for j in self.jobs))

    # ---------------------------------------------------------- device side
    def _prepare(self):
        if self._device is not None:
            return
        import torch

        self._torch = torch
        if not self.jobs:
            # an empty shard (more ranks than jobs): no device program; the
            # rank contributes zero partial energies to the all-reduce
            self._batch = None
            self.set_elems = 0
            self._device = (torch.device("cuda", torch.cuda.current_device())
                            if torch.cuda.is_available() else torch.device("cpu"))
            return
        if not torch.cuda.is_available():
            raise RuntimeError("a CUDA device is required: the B200 backend has no CPU fallback")
        dev = torch.device("cuda", torch.cuda.current_device())
        self._device = dev
        # one device program for every edge network; input set layout from it
        self._batch = PlanBatch([j.plan for j in self.jobs])
        self.set_elems = self._batch.set_elems
        recs = [j.template.recipes.copy() for j in self.jobs]
        for r, j in zip(recs, self.jobs):
            r["out_offset"] = j.plan.input_offsets
        # fused path: SMEM networks build their tensors inside the executor
        self._batch.set_recipes(recs)
        # unfused path (tensorgen into an input buffer, then the executors)
        allrec = np.concatenate([r.copy() for r in recs]) if recs else np.zeros(
            0, dtype=N.RECIPE_DTYPE)
        pos = 0
        for r, off in zip(recs, self._batch.input_offsets):
            allrec["out_offset"][pos: pos + len(r)] += off
            pos += len(r)
        self._n_recipes = len(allrec)
        self._recipes = torch.from_numpy(allrec.view(np.uint8).copy()).to(dev)
        w = np.asarray([j.weight for j in self.jobs], dtype=np.float64)
        self._weights = torch.from_numpy(w).to(dev)

    def _buffers(self, n_sets):
        if n_sets not in self._bufs:
            t = self._torch
            dev = self._device
            need_inputs = self._batch is not None and ((not self.fused) or self._batch.has_hbm)
            ws_bytes = self._batch.workspace_bytes(n_sets) if self._batch is not None else 0
            # device-memory fit check: the evaluation's buffers
            # against what the device has free, before any allocation
            need = (16 * n_sets * self.set_elems if need_inputs else 0) + ws_bytes
            if dev.type == "cuda" and need > 0:
                free, total = t.cuda.mem_get_info(dev)
                if need > free:
                    raise MemoryError(
                        f"an evaluation of {n_sets} angle set(s) needs {need / 2**30:.2f} GiB of "
                        f"device memory (inputs + intermediate arena); {free / 2**30:.2f} GiB of "
                        f"{total / 2**30:.2f} GiB are free: use fewer angle sets per call or slice "
                        f"the networks (slice_k)")
            self._bufs[n_sets] = dict(
                inputs=t.zeros(n_sets * self.set_elems if need_inputs else 2, dtype=t.complex128,
                               device=dev),
                ws=t.empty(max(ws_bytes, 16), dtype=t.uint8, device=dev),
                res=t.zeros((n_sets, max(len(self.jobs), 1)), dtype=t.complex128, device=dev),
                energy=t.zeros(n_sets, dtype=t.float64, device=dev),
                # host <-> device staging of the public energies() call
                angles=t.empty((n_sets, 2 * self.p), dtype=t.float64, device=dev),
                angles_host=t.empty((n_sets, 2 * self.p), dtype=t.float64).pin_memory(),
                energy_host=t.empty(n_sets, dtype=t.float64).pin_memory(),
                launches=self.launches_per_eval(n_sets),
            )
        return self._bufs[n_sets]

    def launches_per_eval(self, n_sets: int = 1) -> int:
        """Kernel launches of one evaluation (executors + energy reduction)."""
        self._prepare()
        if self._batch is None:
            return 0
        return self._batch.launches_for(n_sets) + 1 + (0 if self.fused else 1)

    def launch(self, angles_dev, stream=None):
        """Enqueue one evaluation for every angle set in `angles_dev`
        ([n_sets, 2p] float64 on the device); returns the buffer dict
        (bufs['energy'][s], bufs['res'][s, job]) valid once the stream is done."""
        self._prepare()
        t = self._torch
        n_sets = int(angles_dev.shape[0])
        b = self._buffers(n_sets)
        st = stream if stream is not None else t.cuda.current_stream(self._device)
        sp = st.cuda_stream
        if self._batch is None:
            with t.cuda.stream(st):
                b["energy"].zero_()
            self.launches = 0
            return b
        if self.fused:
            self._batch.execute_angles(angles_dev.data_ptr(), 2 * self.p, n_sets,
                                       b["inputs"].data_ptr(), b["ws"].data_ptr(),
                                       b["res"].data_ptr(), sp)
        else:
            N.check(N.lib.qtn_tensorgen(self._recipes.data_ptr(), self._n_recipes,
                                        angles_dev.data_ptr(), 2 * self.p, n_sets, self.set_elems,
                                        b["inputs"].data_ptr(), sp), "tensorgen")
            self._batch.execute(b["inputs"].data_ptr(), n_sets, b["ws"].data_ptr(),
                                b["res"].data_ptr(), sp, set_stride=self.set_elems)
        N.check(N.lib.qtn_energy_reduce(b["res"].data_ptr(), self._weights.data_ptr(),
                                        len(self.jobs), n_sets, b["energy"].data_ptr(), None, sp),
                "energy")
        self.launches = b["launches"]
        return b

    def execute_only(self, angles_dev, stream=None):
        """The contraction executors alone for every angle set in
        `angles_dev` (no energy reduction): the launches the bench's roofline
        times."""
        self._prepare()
        if self._batch is None:
            return
        t = self._torch
        n_sets = int(angles_dev.shape[0])
        b = self._buffers(n_sets)
        st = stream if stream is not None else t.cuda.current_stream(self._device)
        self._batch.execute_angles(angles_dev.data_ptr(), 2 * self.p, n_sets,
                                   b["inputs"].data_ptr(), b["ws"].data_ptr(),
                                   b["res"].data_ptr(), st.cuda_stream)

    def describe(self, n_sets: int) -> dict:
        """Executor and arithmetic of one evaluation of n_sets angle sets."""
        self._prepare()
        if self._batch is None:
            return {"kernel": "none (empty shard)", "dtype": "none"}
        if self.hbm_jobs:
            kernel = "hbm_executor"
            dtype = ("c128 inputs, c64 storage + f32 math for rank>=12"
                     if any(j.plan.dtype == "complex64" for j in self.hbm_jobs) else "c128")
        elif self._batch.uses_setmajor(n_sets):
            c64 = self._batch.setmajor_elem_bytes(n_sets) == 8
            kernel = "sm_level_kernel_c64" if c64 else "sm_level_kernel"
            dtype = ("c64 (set-major rows complex64, f32 products; gate entries formed in f64)"
                     if c64 else "c128")
        else:
            kernel = "smem_net_kernel"
            dtype = "c128"
        return {"kernel": kernel, "dtype": dtype}

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
        if self._batch is None:
            self.launches = 0
            return np.zeros(a.shape[0], dtype=np.float64)
        b = self._buffers(a.shape[0])
        st = t.cuda.current_stream(self._device)
        if self.fused:
            # one native call: H2D of the angles, the captured evaluation,
            # the energy reduction, D2H and the stream wait
            a = np.ascontiguousarray(a)
            out = np.empty(a.shape[0], dtype=np.float64)
            N.check(N.lib.qtn_batch_energies_host(
                self._batch.handle, a.ctypes.data, 2 * self.p, a.shape[0], b["angles"].data_ptr(),
                b["inputs"].data_ptr(), b["ws"].data_ptr(), b["res"].data_ptr(),
                self._weights.data_ptr(), b["energy"].data_ptr(), out.ctypes.data,
                st.cuda_stream), "energies")
            self.launches = b["launches"]
            return out
        b["angles_host"].numpy()[...] = a
        b["angles"].copy_(b["angles_host"], non_blocking=True)
        self.launch(b["angles"], st)
        b["energy_host"].copy_(b["energy"], non_blocking=True)
        st.synchronize()
        return b["energy_host"].numpy().copy()

    def zz_values(self, params: QaoaParams) -> dict:
        """Per-edge <Z_iZ_j> (complex) for one angle set, keyed by edge index."""
        self._prepare()
        t = self._torch
        a = t.from_numpy(np.atleast_2d(params.as_vector())).to(self._device)
        b = self.launch(a)
        r = b["res"][0].cpu().numpy()
        out = {}
        for k, j in enumerate(self.jobs):  # slices of one edge add up
            out[j.index] = out.get(j.index, 0j) + complex(r[k])
        return out


def rank_shard(graph: ProblemGraph, p: int, mode: str, rank: int, world: int,
               n_repeats=10, temp=0.02, seed=0, slice_k: int = 0, edge_ids=None,
               compile_plans=True, **plan_kw):
    """This rank's jobs (edges, or edge slices): LPT over the reference cost
    model.  Every rank computes the same deterministic orders (the partition
    needs every job's cost, and no exchange), then compiles plans only for
    the jobs it keeps.  May be empty when there are fewer jobs than ranks."""
    ids = range(graph.edge_count) if edge_ids is None else edge_ids
    allj = plan_edges(graph, p, mode, ids, n_repeats=n_repeats, temp=temp, seed=seed,
                      slice_k=slice_k, compile_plans=False,
                      **{k: v for k, v in plan_kw.items() if k == "workers"})
    keep = shard_edges([j.cost for j in allj], world)[rank]
    mine = [allj[k] for k in keep]
    if compile_plans:
        compile_jobs(mine, **plan_kw)
    return mine


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
        jobs = None
        if world > 1:
            jobs = rank_shard(graph, params.p, mode, dist.get_rank(group), world, dtype=dtype,
                              **kw)
        plan = EnergyPlan(graph, params.p, mode, dtype, jobs=jobs, **kw)
    e = plan.energies(params)
    dev = torch.device("cuda", torch.cuda.current_device()) if world > 1 else None
    return float(reduce_partials(e, group, dev)[0])
