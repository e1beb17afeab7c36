"""Elimination orderings and the cost model — reference API, native passes.

Public names follow /root/reference/pkg/src/qtnsim/ordering.py:
ContractionOrder (31-43), CostReport (46-68), contraction_width (93-100),
greedy_order (132-136), rgreedy_order (154-189).  The reference's passes
are reused unchanged in *algorithm*: the same min-degree / Boltzmann rule,
the same RNG streams (`default_rng(seed + pass)`, one variate per step),
the same (width, flops_sum, pass) selection.  The passes themselves run in
C++ (csrc/qtn_order.cpp, bitset adjacency); numpy draws the variates and the
weight table exp(-d/temp) so every float the selection sees is the one the
reference would compute — orders, and hence widths, are identical.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .network import LineGraph

__all__ = [
    "ContractionOrder",
    "CostReport",
    "contraction_width",
    "greedy_order",
    "rgreedy_order",
]


@dataclass(frozen=True)
class ContractionOrder:
    """Elimination sequence: a permutation of the line-graph vertex ids."""

    sequence: tuple

    def __post_init__(self):
        seq = tuple(int(v) for v in self.sequence)
        object.__setattr__(self, "sequence", seq)
        if len(set(seq)) != len(seq):
            raise ValueError("order contains repeated vertices")

    def __len__(self) -> int:
        return len(self.sequence)


@dataclass(frozen=True)
class CostReport:
    width: int
    step_ranks: tuple
    flops_2c: float
    flops_sum: float
    memory_bytes: float

    @classmethod
    def from_step_ranks(cls, step_ranks) -> "CostReport":
        r = tuple(int(x) for x in step_ranks)
        w = max(r, default=0)
        # 2^(rank+1) per step: one multiply-add per summed-over entry
        return cls(w, r, 2.0**w, float(sum(2.0 ** (x + 1) for x in r)), 16.0 * 2.0**w)


def _csr(lg: LineGraph):
    """Hyperedges over compact ids 0..V-1 (ascending vertex id), as CSR."""
    index = {v: k for k, v in enumerate(lg.vertices)}
    offs = [0]
    flat = []
    for he in lg.hyperedges:
        flat.extend(index[v] for v in he)
        offs.append(len(flat))
    return (np.asarray(offs, dtype=np.int32), np.asarray(flat if flat else [0], dtype=np.int32),
            len(lg.hyperedges))


def contraction_width(lg: LineGraph, order: ContractionOrder) -> CostReport:
    if sorted(order.sequence) != list(lg.vertices):
        raise ValueError("order is not a permutation of the line-graph vertices")
    nv = lg.vertex_count
    offs, flat, ne = _csr(lg)
    index = {v: k for k, v in enumerate(lg.vertices)}
    seq = np.asarray([index[v] for v in order.sequence] or [0], dtype=np.int32)
    ranks = np.zeros(max(nv, 1), dtype=np.int32)
    N.check(N.lib.qtn_order_ranks(nv, ne, N.i32(offs), N.i32(flat), N.i32(seq), N.i32(ranks)),
            "contraction_width")
    return CostReport.from_step_ranks(ranks[:nv])


def greedy_order(lg: LineGraph) -> ContractionOrder:
    """Deterministic min-degree order; ties to the smallest vertex id."""
    nv = lg.vertex_count
    offs, flat, ne = _csr(lg)
    order = np.zeros(max(nv, 1), dtype=np.int32)
    ranks = np.zeros(max(nv, 1), dtype=np.int32)
    N.check(N.lib.qtn_order_pass(nv, ne, N.i32(offs), N.i32(flat), None, None, 0,
                                 N.i32(order), N.i32(ranks)), "greedy_order")
    return ContractionOrder(tuple(lg.vertices[i] for i in order[:nv]))


def rgreedy_order(lg: LineGraph, n_repeats: int = 10, temp: float = 0.02, seed: int = 0):
    """Best of `n_repeats` passes (pass 0 = min degree, pass k Boltzmann
    sampling with default_rng(seed + k)); returns (ContractionOrder, CostReport)."""
    if n_repeats < 1:
        raise ValueError("n_repeats must be >= 1")
    if temp < 0.0:
        raise ValueError("temp must be >= 0")
    nv = lg.vertex_count
    offs, flat, ne = _csr(lg)
    # the variates the reference consumes: one rng.random() per step per pass
    draws = np.zeros(max((n_repeats - 1) * nv, 1), dtype=np.float64)
    for rep in range(1, n_repeats):
        draws[(rep - 1) * nv: rep * nv] = np.random.default_rng(seed + rep).random(nv)
    if temp == 0.0:
        table = np.zeros(1, dtype=np.float64)
    else:
        # same ufunc on the same int64 differences as ordering.py:146
        table = np.exp(-(np.arange(nv + 1, dtype=np.int64)) / temp)
    order = np.zeros(max(nv, 1), dtype=np.int32)
    ranks = np.zeros(max(nv, 1), dtype=np.int32)
    best = np.zeros(1, dtype=np.int32)
    N.check(N.lib.qtn_rgreedy(nv, ne, N.i32(offs), N.i32(flat), n_repeats, N.f64(draws),
                              N.f64(table), 1 if temp == 0.0 else 0, N.i32(order), N.i32(ranks),
                              N.i32(best)), "rgreedy_order")
    seq = ContractionOrder(tuple(lg.vertices[i] for i in order[:nv]))
    return seq, CostReport.from_step_ranks(ranks[:nv])
