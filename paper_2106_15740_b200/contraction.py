"""Bucket-elimination contraction on B200 — the drop-in boundary.

`contract(network, order, rank_cap=DEFAULT_RANK_CAP)` keeps the signature,
return type (Python complex) and error behaviour of the reference entry
point /root/reference/pkg/src/qtnsim/contraction.py:114-123:

  * ValueError if `order` is not a permutation of the unfixed variables
    (contraction.py:60-62);
  * RankCapExceeded(rank, cap) — a RuntimeError — raised while compiling the
    plan, i.e. before any device allocation (contraction.py:32-39, 85-87);
  * `_contract_with_ranks` returns (value, step_ranks) whose peak equals the
    CostReport width of the same order.

Evaluation differs from the reference only in *how* each bucket runs: the
plan compiler (csrc/qtn_plan.cpp) turns the order into a bucket program and
one of two sm_100a executors runs it — a warp-per-network shared-memory
interpreter for networks whose whole live set fits on chip, or fused
per-bucket kernels over an HBM arena.  There is no CPU fallback: without a
CUDA device these functions raise.
"""

from __future__ import annotations

import collections
import ctypes as C
import threading

import numpy as np

from . import _native as N
from .network import TensorNetwork, sliced_tensors
from .ordering import ContractionOrder

__all__ = [
    "DEFAULT_RANK_CAP",
    "DEFAULT_MIXED_RANK",
    "DEFAULT_SMEM_BUDGET",
    "RankCapExceeded",
    "ContractionPlan",
    "PlanBatch",
    "contract",
    "contract_many",
]

DEFAULT_RANK_CAP = 30
# complex64 storage applies to intermediates of rank >= this (SURVEY §7:
# all-complex64 fails 1e-5 on config 4; rank >= 10..14 keeps ~1e-8)
DEFAULT_MIXED_RANK = 12
# shared memory one network may use in the warp-resident executor
DEFAULT_SMEM_BUDGET = 100 * 1024


class RankCapExceeded(RuntimeError):
    """An intermediate tensor would exceed the rank cap; contraction aborted
    before allocation."""

    def __init__(self, rank: int, cap: int):
        super().__init__(f"intermediate of rank {rank} exceeds rank cap {cap}")
        self.rank = rank
        self.cap = cap


def _dtype_code(dtype) -> int:
    name = str(dtype).replace("torch.", "").replace("numpy.", "")
    if name in ("complex64", "c64", "cfloat", "<class 'numpy.complex64'>"):
        return N.DTYPE_C64
    if name in ("complex128", "c128", "cdouble", "complex", "<class 'numpy.complex128'>",
                "<class 'complex'>"):
        return N.DTYPE_C128
    raise ValueError(f"unsupported dtype {dtype!r}; use complex64 or complex128")


class ContractionPlan:
    """A compiled (sliced-network structure, elimination order) pair.

    The structure is the list of variable tuples of `sliced_tensors` in
    network order; data is supplied at execution time as one packed
    complex128 buffer (tensor k at `input_offsets[k]`).
    """

    def __init__(self, structure, variable_count, fixed, sequence, rank_cap=DEFAULT_RANK_CAP,
                 dtype="complex128", mixed_rank=DEFAULT_MIXED_RANK,
                 smem_budget=DEFAULT_SMEM_BUDGET):
        self._h = None
        self.dtype = "complex64" if _dtype_code(dtype) == N.DTYPE_C64 else "complex128"
        ranks = np.asarray([len(s) for s in structure] or [0], dtype=np.int32)
        offs = np.zeros(len(structure) + 1, dtype=np.int32)
        offs[1:] = np.cumsum([len(s) for s in structure])
        flat = np.asarray([v for s in structure for v in s] or [0], dtype=np.int32)
        is_fixed = np.zeros(max(variable_count, 1), dtype=np.uint8)
        for v in fixed:
            is_fixed[v] = 1
        seq = np.asarray(list(sequence) or [0], dtype=np.int32)
        desc = N.NetworkDesc(len(structure), N.i32(ranks), N.i32(offs), N.i32(flat),
                             variable_count, N.u8(is_fixed))
        h = C.c_void_p()
        bad = C.c_int32(0)
        rc = N.lib.qtn_plan_create(C.byref(desc), N.i32(seq), len(sequence), int(rank_cap),
                                   _dtype_code(dtype), int(mixed_rank), int(smem_budget),
                                   C.byref(h), C.byref(bad))
        if rc == N.QTN_ERANKCAP:
            raise RankCapExceeded(int(bad.value), int(rank_cap))
        N.check(rc, "plan compile")
        self._h = h
        info = N.PlanInfo()
        N.check(N.lib.qtn_plan_info(h, C.byref(info)))
        self.executor = int(info.executor)
        self.n_buckets = int(info.n_buckets)
        self.n_empty_buckets = int(info.n_empty_buckets)
        self.width = int(info.width)
        self.input_elems = int(info.input_elems)
        self.workspace_bytes = int(info.workspace_bytes)
        self.smem_bytes = int(info.smem_bytes)
        self.program_bytes = int(info.program_bytes)
        self.alg_bytes = float(info.alg_bytes)
        self.flops_sum = float(info.flops_sum)
        self.n_levels = int(info.n_levels)
        self.n_fused_chains = int(info.n_fused_chains)
        self.exec_bytes = float(info.exec_bytes)
        self.n_pairs = int(info.n_pairs)
        self.n_tails = int(info.n_tails)
        sr = np.zeros(max(len(sequence), 1), dtype=np.int32)
        N.check(N.lib.qtn_plan_step_ranks(h, N.i32(sr)))
        self.step_ranks = tuple(int(x) for x in sr[: len(sequence)])
        io = np.zeros(max(len(structure), 1), dtype=np.int64)
        N.check(N.lib.qtn_plan_input_offsets(h, N.i64(io)))
        self.input_offsets = io[: len(structure)].copy()
        sizes = np.array([1 << len(v) for v in structure], dtype=np.int64)
        ends = self.input_offsets + sizes
        self._dense = bool(len(structure) and self.input_offsets[0] == 0
                           and np.array_equal(self.input_offsets[1:], ends[:-1]))
        self._dense_end = int(ends[-1]) if len(structure) else 0
        self.n_inputs = len(structure)

    @classmethod
    def from_network(cls, network: TensorNetwork, order: ContractionOrder, **kw):
        sl = sliced_tensors(network)
        plan = cls([t.variables for t in sl], network.variable_count, network.fixed,
                   order.sequence, **kw)
        return plan, sl

    @property
    def handle(self):
        return self._h

    def pack(self, datas, out: np.ndarray | None = None) -> np.ndarray:
        """Pack sliced tensor data (network order) into the input layout."""
        buf = out if out is not None else np.empty(self.input_elems, dtype=np.complex128)
        if self._dense and len(datas) == len(self.input_offsets):
            # tensors lie back to back in network order: one concatenate call
            try:
                # (Tensor.data is always an ndarray; concatenate casts other dtypes into buf)
                np.concatenate([d.ravel() for d in datas], out=buf[: self._dense_end])
                return buf
            except (ValueError, AttributeError, TypeError):
                pass  # not arrays, or sizes differ from the structure: per-tensor placement below
        for off, d in zip(self.input_offsets, datas):
            flat = np.asarray(d, dtype=np.complex128).reshape(-1)
            buf[off: off + flat.size] = flat
        return buf

    def execute(self, inputs_ptr: int, workspace_ptr: int, result_ptr: int, stream: int) -> None:
        """Run on device buffers: packed inputs, >= workspace_bytes of
        workspace (HBM executor), one complex128 result."""
        N.check(N.lib.qtn_plan_execute(self._h, inputs_ptr, workspace_ptr or None, result_ptr,
                                       stream), "plan execute")

    def __del__(self):
        if self._h is not None and N is not None and N.lib is not None:
            N.lib.qtn_plan_destroy(self._h)
            self._h = None


def _torch_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("a CUDA device is required: the B200 backend has no CPU fallback")
    return torch


class PlanBatch:
    """Device program for many plans (qtn_batch): SMEM-executor networks in
    one warp-per-network launch, HBM-executor networks level-synchronously
    (one streaming launch per elimination-tree level for all of them)."""

    def __init__(self, plans):
        _torch_cuda()
        self.plans = list(plans)
        self._recipes_set = False
        arr = (C.c_void_p * len(self.plans))(*[p.handle for p in self.plans])
        h = C.c_void_p()
        N.check(N.lib.qtn_batch_create(arr, len(self.plans), C.byref(h)), "batch create")
        self._h = h
        nel = C.c_int64()
        N.check(N.lib.qtn_batch_input_elems(h, C.byref(nel)))
        self.set_elems = int(nel.value)
        offs = np.zeros(len(self.plans), dtype=np.int64)
        N.check(N.lib.qtn_batch_input_offsets(h, N.i64(offs)))
        self.input_offsets = offs
        self.launches = self.launches_for(1)

    def launches_for(self, n_sets: int) -> int:
        nl = C.c_int32()
        N.check(N.lib.qtn_batch_launches(self._h, int(n_sets), C.byref(nl)))
        return int(nl.value) + (1 if (self.has_hbm and self._recipes_set) else 0)

    @property
    def handle(self):
        return self._h

    def uses_setmajor(self, n_sets: int) -> bool:
        """Whether n_sets input sets run the small networks set-major."""
        f = C.c_int32()
        N.check(N.lib.qtn_batch_uses_setmajor(self._h, int(n_sets), C.byref(f)))
        return bool(f.value)

    def setmajor_elem_bytes(self, n_sets: int) -> int:
        """Bytes per set-major element at n_sets sets: 8 (complex64 rows), 16, or 0."""
        f = C.c_int32()
        N.check(N.lib.qtn_batch_setmajor_elem_bytes(self._h, int(n_sets), C.byref(f)))
        return int(f.value)

    def workspace_bytes(self, n_sets: int) -> int:
        w = C.c_int64()
        N.check(N.lib.qtn_batch_workspace_bytes(self._h, int(n_sets), C.byref(w)))
        return int(w.value)

    def pack(self, datas_list, out: np.ndarray | None = None) -> np.ndarray:
        host = out if out is not None else np.zeros(max(self.set_elems, 1), dtype=np.complex128)
        for p, off, datas in zip(self.plans, self.input_offsets, datas_list):
            p.pack(datas, host[off: off + p.input_elems])
        return host

    def execute(self, inputs_ptr, n_sets, workspace_ptr, results_ptr, stream, set_stride=0):
        N.check(N.lib.qtn_batch_execute(self._h, inputs_ptr, int(set_stride), int(n_sets),
                                        workspace_ptr or None, results_ptr, stream),
                "batch execute")

    @property
    def has_hbm(self) -> bool:
        return any(p.executor == N.EXEC_HBM for p in self.plans)

    def set_recipes(self, recipes_per_plan):
        """Tensor recipes (RECIPE_DTYPE arrays, offsets relative to each
        network's packed input); enables execute_angles."""
        allrec = np.concatenate(recipes_per_plan) if recipes_per_plan else np.zeros(
            0, dtype=N.RECIPE_DTYPE)
        allrec = np.ascontiguousarray(allrec)
        offs = np.zeros(len(recipes_per_plan) + 1, dtype=np.int64)
        offs[1:] = np.cumsum([len(r) for r in recipes_per_plan])
        N.check(N.lib.qtn_batch_set_recipes(self._h, allrec.ctypes.data, N.i64(offs)),
                "set recipes")
        self._recipes_set = True  # execute_angles adds a tensorgen launch for HBM networks

    def execute_angles(self, angles_ptr, n_angles, n_sets, scratch_ptr, workspace_ptr,
                       results_ptr, stream):
        N.check(N.lib.qtn_batch_execute_angles(self._h, angles_ptr, int(n_angles), int(n_sets),
                                               scratch_ptr or None, workspace_ptr or None,
                                               results_ptr, stream), "batch execute (angles)")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and N is not None and N.lib is not None:
            N.lib.qtn_batch_destroy(h)
            self._h = None


def _run_plans(plans, datas_list):
    """Execute plans as one batch on the current device; returns complex list."""
    torch = _torch_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    batch = PlanBatch(plans)
    inp = torch.from_numpy(batch.pack(datas_list)).pin_memory().to(dev, non_blocking=True)
    ws = torch.empty(max(batch.workspace_bytes(1), 16), dtype=torch.uint8, device=dev)
    res = torch.empty(len(plans), dtype=torch.complex128, device=dev)
    batch.execute(inp.data_ptr(), 1, ws.data_ptr(), res.data_ptr(), stream.cuda_stream)
    out = res.cpu().numpy()
    del batch
    return [complex(x) for x in out]


class _CachedRun:
    """A compiled plan with its device program and buffers, reused by every
    contract() call on the same (sliced structure, order, options): the QAOA
    loop re-contracts the same networks with new tensor data."""

    def __init__(self, plan):
        torch = _torch_cuda()
        dev = torch.device("cuda", torch.cuda.current_device())
        self.plan = plan
        self.batch = PlanBatch([plan])
        self.host = torch.zeros(max(self.batch.set_elems, 1), dtype=torch.complex128).pin_memory()
        self.inp = torch.empty_like(self.host, device=dev)
        self.ws = torch.empty(max(self.batch.workspace_bytes(1), 16), dtype=torch.uint8, device=dev)
        self.res = torch.empty(1, dtype=torch.complex128, device=dev)
        self.res_host = torch.empty(1, dtype=torch.complex128).pin_memory()
        self._res_np = self.res_host.numpy()
        self.dev = dev
        self.device_bytes = int(self.ws.numel()) + 16 * int(self.inp.numel())
        # the staging buffers, workspace and the batch's graph cache are
        # shared by every caller of this structure: one contraction at a time
        # (distinct structures still run concurrently)
        self.lock = threading.Lock()

    def run(self, datas) -> complex:
        with self.lock:
            return self._run(datas)

    def _run(self, datas) -> complex:
        torch = _torch_cuda()
        stream = torch.cuda.current_stream(self.dev)
        h = self.host.numpy()
        self.batch.pack([datas], out=h)
        # one native call: H2D of the packed inputs, the evaluation, D2H, stream wait
        N.check(N.lib.qtn_batch_execute_host(
            self.batch.handle, self.host.data_ptr(), 16 * int(self.host.numel()),
            self.inp.data_ptr(), self.ws.data_ptr(), self.res.data_ptr(),
            self.res_host.data_ptr(), stream.cuda_stream), "contract")
        return complex(self._res_np[0])


_RUNS: "collections.OrderedDict" = collections.OrderedDict()
_RUNS_LOCK = threading.Lock()
_RUNS_MAX = 64
# device bytes (workspace + inputs) the cache may keep alive: networks of
# width 23-26 hold GBs of workspace each
_RUNS_MAX_BYTES = 8 << 30


def _contract_with_ranks(network: TensorNetwork, order: ContractionOrder, rank_cap: int,
                         dtype="complex128", **kw):
    unfixed = network.unfixed_variables()
    if sorted(order.sequence) != list(unfixed):
        raise ValueError("order is not a permutation of the network's unfixed variables")
    import torch

    # the unsliced structure and the set of fixed variables determine the
    # sliced structure (the fixed values only pick the data, network.py:153-165)
    fx = network.fixed
    key = (tuple(t.variables for t in network.tensors), network.variable_count, frozenset(fx),
           tuple(order.sequence), int(rank_cap), _dtype_code(dtype), tuple(sorted(kw.items())),
           torch.cuda.current_device() if torch.cuda.is_available() else -1)
    with _RUNS_LOCK:
        run = _RUNS.get(key)
        if run is not None:
            _RUNS.move_to_end(key)
    if run is not None:
        # known structure: pin the fixed variables on the data only (no Tensor objects)
        datas = [t.data for t in network.tensors]
        for k in run.touched:
            t = network.tensors[k]
            datas[k] = t.data[tuple(fx[v] if v in fx else slice(None) for v in t.variables)]
        return run.run(datas), list(run.plan.step_ranks)
    sl = sliced_tensors(network)
    # RankCapExceeded / ValueError surface here, before any device work
    plan = ContractionPlan([t.variables for t in sl], network.variable_count, network.fixed,
                           order.sequence, rank_cap=rank_cap, dtype=dtype, **kw)
    run = _CachedRun(plan)  # raises without a CUDA device (no CPU fallback)
    run.touched = [k for k, t in enumerate(network.tensors) if any(v in fx for v in t.variables)]
    with _RUNS_LOCK:
        _RUNS[key] = run
        total = sum(r.device_bytes for r in _RUNS.values())
        while len(_RUNS) > 1 and (len(_RUNS) > _RUNS_MAX or total > _RUNS_MAX_BYTES):
            _, old = _RUNS.popitem(last=False)
            total -= old.device_bytes
    return run.run([t.data for t in sl]), list(run.plan.step_ranks)


def contract(network: TensorNetwork, order: ContractionOrder, rank_cap: int = DEFAULT_RANK_CAP,
             dtype="complex128", **kw) -> complex:
    """Contract all unfixed variables along `order` on the GPU; returns the
    amplitude.  Raises RankCapExceeded before allocating any intermediate
    whose rank would exceed `rank_cap`."""
    value, _ = _contract_with_ranks(network, order, rank_cap, dtype=dtype, **kw)
    return value


def contract_many(networks, orders, rank_cap: int = DEFAULT_RANK_CAP, dtype="complex128", **kw):
    """Contract independent networks; shared-memory-resident ones run as one
    batched launch (one warp per network)."""
    plans, datas = [], []
    for net, order in zip(networks, orders):
        plan, sl = ContractionPlan.from_network(net, order, rank_cap=rank_cap, dtype=dtype, **kw)
        plans.append(plan)
        datas.append([t.data for t in sl])
    return _run_plans(plans, datas)
