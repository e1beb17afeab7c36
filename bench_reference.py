"""CPU legs of bench.py: the reference's own implementation of the path,
timed on the host cores.

Used by `bench.py --impl reference` (all host cores, the driver's reference
arm) and by the `cpu_baseline` records of the B200 arm (one core).  Nothing
here imports the B200 package or loads its library:

* with `baseline/_ref/qtnsim` present (the unmodified reference, installed
  by `pip install --target baseline/_ref`), every contraction goes through
  the reference's public API: `Gate` / `Circuit` (circuit.py:93-176),
  `circuit_to_network` (network.py:93-150), `line_graph`
  (network.py:210-218), `rgreedy_order` (ordering.py:154-189) and
  `contract` (contraction.py:114-123), the way its own benchmark loop calls
  them (bench.py:225-251) — `kind: "reference"`;
* otherwise the oracle restatement (oracle/qtn_oracle.py) stands in —
  `kind: "port"`.

The per-edge light cone has no reference function; it is the
oracle's composer (`edge_cone_gates`) emitting reference gate objects, the
same construction tests/golden/make_golden.py pins the goldens with.
"""

from __future__ import annotations

import itertools
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
ORACLE_DIR = os.path.join(ROOT, "oracle")

MODES = {"default": (False, False), "diagonal": (False, True), "zz": (True, False),
         "zz+diagonal": (True, True)}  # pipeline.py:38-43: name -> (fused, diagonal)


def _oracle():
    if ORACLE_DIR not in sys.path:
        sys.path.insert(0, ORACLE_DIR)
    import qtn_oracle

    return qtn_oracle


def load_reference():
    """The installed reference package, or None (then the oracle port)."""
    if not os.path.isdir(os.path.join(REF_DIR, "qtnsim")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import qtnsim
    except Exception:
        return None
    return qtnsim


def host_cpu():
    """nproc and CPU model of the box (record them)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


# ------------------------------------------------------------ one edge network
class EdgeWork:
    """Network build + contraction of one (edge, angle set), through the
    reference when it is installed, else through the oracle port."""

    def __init__(self, n, p, mode, edge_ids):
        self.Q = load_reference()
        self.O = _oracle()
        self.kind = "reference" if self.Q is not None else "port"
        self.n, self.p, self.mode = n, p, mode
        self.fused, self.diagonal = MODES[mode]
        if self.Q is not None:
            self.graph = self.Q.random_regular_graph(n, 3, 0)  # bench.py:48-78
            self.edges = [tuple(e) for e in self.graph.edges]
        else:
            self.edges = [tuple(e) for e in self.O.random_regular_graph(n, 3, 0)]
        self.edge_ids = list(edge_ids) if edge_ids is not None else list(range(len(self.edges)))
        self.orders = {}
        self.slices = {e: [{}] for e in self.edge_ids}

    # network of edge e at angles (gammas, betas)
    def network(self, e, gammas, betas, assignment=None):
        m, gates, phase, _ = self.O.edge_cone_gates(self.n, self.edges, self.edges[e],
                                                     list(gammas), list(betas), self.fused)
        if self.Q is None:
            tensors, nv, fixed = self.O.circuit_tensors(m, gates, phase, self.diagonal, "0" * m)
            return tensors, nv, {**fixed, **(assignment or {})}
        Q = self.Q
        circ = Q.Circuit(m, tuple(Q.Gate(Q.GateKind(k), qs, t) for k, qs, t in gates), phase)
        net = Q.circuit_to_network(circ, Q.get_mode(self.mode).network_mode, "0" * m)
        if assignment:
            net = Q.TensorNetwork(net.tensors, net.variable_count, {**net.fixed, **assignment})
        return net

    def order(self, e, gammas, betas):
        """Reference rgreedy(10, 0.02, seed 0) order; angle-independent, so
        computed once per edge (the plan cache of the B200 arm)."""
        if e not in self.orders:
            if self.Q is None:
                tensors, nv, fixed = self.network(e, gammas, betas)
                verts = [v for v in range(nv) if v not in fixed]
                seq, _ = self.O.rgreedy(verts, self.O.hyperedges(tensors, fixed))
                self.orders[e] = list(seq)
            else:
                order, _ = self.Q.rgreedy_order(self.Q.line_graph(self.network(e, gammas, betas)),
                                                n_repeats=10, temp=0.02, seed=0)
                self.orders[e] = order
        return self.orders[e]

    def slice_edge(self, e, gammas, betas, k):
        """2^k slices of edge e over its k most-used variables of the widest
        steps (the fixed-variable mechanism, network.py:78, 153-165; the
        order loses the sliced variables, contraction.py:60-62)."""
        if k <= 0:
            return
        order = self.order(e, gammas, betas)
        seq = list(order.sequence) if self.Q is not None else list(order)
        if self.Q is not None:
            lg = self.Q.line_graph(self.network(e, gammas, betas))
            adj = {v: set(lg.adjacency[v]) for v in lg.vertices}
        else:
            tensors, nv, fixed = self.network(e, gammas, betas)
            adj = {v: set() for v in range(nv) if v not in fixed}
            for he in self.O.hyperedges(tensors, fixed):
                for a in he:
                    adj[a] |= set(he) - {a}
        steps = []
        for v in seq:
            nb = adj.pop(v)
            for a in nb:
                adj[a].discard(v)
                adj[a] |= nb - {a}
            steps.append((len(nb), nb | {v}))
        width = max(r for r, _ in steps)
        score = {}
        for r, members in steps:
            if r >= width - 3:
                for u in members:
                    score[u] = score.get(u, 0.0) + 2.0 ** r
        chosen = sorted(score, key=lambda u: (-score[u], u))[:k]
        rest = [v for v in seq if v not in chosen]
        self.orders[e] = self.Q.ContractionOrder(tuple(rest)) if self.Q is not None else rest
        self.slices[e] = [dict(zip(chosen, bits))
                          for bits in itertools.product((0, 1), repeat=len(chosen))]

    def zz(self, e, gammas, betas, assignment=None):
        """<Z_iZ_j> (or one slice's share of it) at these angles."""
        order = self.order(e, gammas, betas)
        if self.Q is None:
            tensors, nv, fixed = self.network(e, gammas, betas, assignment)
            val, _ = self.O.contract(tensors, nv, fixed, order)
            return complex(val)
        return complex(self.Q.contract(self.network(e, gammas, betas, assignment), order))


# ------------------------------------------------------------- process pools
_W = None


def _init(n, p, mode, edge_ids, orders, slices):
    global _W
    _W = EdgeWork(n, p, mode, edge_ids)
    _W.orders = orders
    _W.slices = slices


def _job(task):
    e, angles, assignment = task
    p = _W.p
    return _W.zz(e, angles[:p], angles[p:], assignment)


def prepare(n, p, mode, edge_ids, angles0, slice_k=0):
    """Orders (and slices) computed once, outside every timed region."""
    w = EdgeWork(n, p, mode, edge_ids)
    for e in w.edge_ids:
        w.order(e, angles0[:p], angles0[p:])
        w.slice_edge(e, angles0[:p], angles0[p:], slice_k)
    return w


def tasks_for(w, sets):
    return [(e, s, a) for s in sets for e in w.edge_ids for a in w.slices[e]]


def timed_steps(w, step_sets, warmup, steps, cores):
    """Run warmup + steps steps; step k evaluates every (edge, slice) at the
    angle sets step_sets(k).  Returns (per-step seconds of the timed steps,
    contractions per step, values of the last step)."""
    import multiprocessing as mp

    times, vals = [], None
    if cores <= 1:
        _init(w.n, w.p, w.mode, w.edge_ids, w.orders, w.slices)
        run = lambda ts: [_job(t) for t in ts]
        pool = None
    else:
        ctx = mp.get_context("fork")
        pool = ctx.Pool(cores, initializer=_init,
                        initargs=(w.n, w.p, w.mode, w.edge_ids, w.orders, w.slices))
        run = lambda ts: pool.map(_job, ts, chunksize=max(1, len(ts) // (4 * cores)))
    try:
        per = None
        for it in range(warmup + steps):
            sets = step_sets(it)
            ts = tasks_for(w, sets)
            t0 = time.perf_counter()
            vals = run(ts)
            dt = time.perf_counter() - t0
            per = len(w.edge_ids) * len(sets)  # edge contractions (slices add up)
            if it >= warmup:
                times.append(dt)
    finally:
        if pool is not None:
            pool.close()
            pool.join()
    return times, per, vals


def sample_rate(n, p, mode, edge_ids, sets, seconds=10.0, cores=1, slice_k=0):
    """cpu_baseline leg (one core): edge contractions/s over a bounded sample
    of about `seconds`: (edge, slice) contractions in workload order, angle
    sets cycled, each slice counted as 1/2^k of an edge contraction."""
    w = prepare(n, p, mode, edge_ids, sets[0], slice_k)
    _init(w.n, w.p, w.mode, w.edge_ids, w.orders, w.slices)
    tasks = tasks_for(w, sets)
    done, units = 0, 0.0
    t0 = time.perf_counter()
    while True:
        e, s, a = tasks[done % len(tasks)]
        _job((e, s, a))
        done += 1
        units += 1.0 / len(w.slices[e])
        dt = time.perf_counter() - t0
        if dt >= seconds:
            break
    return {"value": units / dt, "unit": "contractions/s", "cores": 1, "kind": w.kind,
            "host": host_cpu(),
            "sample": f"{done} (edge{', slice' if slice_k else ''}) contractions = {units:.2f} "
                      f"edge contractions in {dt:.1f}s over {len(w.edge_ids)} edge(s)"
                      f"{f' x 2^{slice_k} slices' if slice_k else ''}, angle sets cycled: " +
                      ("qtnsim circuit_to_network + contract" if w.kind == "reference" else
                       "oracle network build + bucket elimination") +
                      ", complex128, orders cached"}


# ------------------------------------------------------- config-5 bucket ops
def bucket_rate(w_bits=22, m=16, seed=0, reps=2):
    """The reference bucket operations on one synthetic config-5 bucket: the
    pairwise `_product` chain in ascending id and the `.sum` over v
    (contraction.py:42-54, 90-96), complex128 as the reference stores tensor
    data (network.py:50).  One core.  Returns GB/s of algorithmic bytes."""
    O = _oracle()
    Q = load_reference()
    ops = O.synthetic_bucket(w_bits, m, seed, dtype=np.complex128)
    if Q is not None:
        from qtnsim.contraction import _product
        kind = "reference"
    else:
        _product = O.pair_product
        kind = "port"
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        va, da = ops[0]
        for vb, db in ops[1:]:
            va, da = _product(tuple(va), da, tuple(vb), db)
        ax = list(va).index(0)
        out = da.sum(axis=ax)
        ts.append(time.perf_counter() - t0)
        del out, da
    t = min(ts)
    alg = 16.0 * (sum(1 << len(v) for v, _ in ops) + (1 << w_bits))
    return {"value": alg / t / 1e9, "unit": "GB/s", "cores": 1, "kind": kind,
            "host": host_cpu(), "seconds_per_bucket": t,
            "sample": f"one w={w_bits}, m={m} bucket (seed {seed}), complex128, best of {reps}: "
                      "pairwise _product chain + .sum over v"}
