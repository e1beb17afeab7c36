"""Slicing: split one network into 2^k independent sub-networks.

The reference's only slicing mechanism is fixing variables:
`TensorNetwork.fixed` + `sliced_tensors` (network.py:78, 153-165), which it
uses for output bits; "index slicing for distributed contraction" is a
non-goal there.  The north star asks for it (2^k slices
over the GPUs, config 4), built on the same mechanism: slice assignment a is
the network with {**fixed, **a}, contracted with the reference order minus
the sliced variables (still a permutation of the unfixed variables,
contraction.py:60-62), and the value is the sum over the 2^k assignments.

Variable choice (SURVEY §7 "Slice-variable choice"): degree in the initial
line graph is uninformative for these networks, membership in the largest
intermediates along the reference order is not.  Greedily, k times: replay
the elimination (ordering.py:79-90), give every variable of every step whose
rank is within `window` of the current width a score 2^rank, fix the best
(ties to the smallest id), drop it from the line graph and the order.  The
resulting width is evaluated with the reference cost model
(`contraction_width` on the sliced line graph), so it is oracle-checkable.
"""

from __future__ import annotations

import itertools

from .network import LineGraph
from .ordering import ContractionOrder, contraction_width

__all__ = ["choose_slice_vars", "slice_assignments", "remove_vertices"]


def _replay(lg: LineGraph, order: ContractionOrder):
    """(rank, variables of the bucket) per elimination step."""
    adj = {v: set(lg.adjacency[v]) for v in lg.vertices}
    out = []
    for v in order.sequence:
        nb = adj.pop(v)
        for a in nb:
            adj[a].discard(v)
            adj[a] |= nb - {a}
        out.append((len(nb), nb | {v}))
    return out


def remove_vertices(lg: LineGraph, gone) -> LineGraph:
    """Line graph of the network with `gone` additionally fixed."""
    gone = set(gone)
    edges = [tuple(u for u in he if u not in gone) for he in lg.hyperedges]
    return LineGraph.from_hyperedges([v for v in lg.vertices if v not in gone],
                                     [e for e in edges if e])


def choose_slice_vars(lg: LineGraph, order: ContractionOrder, k: int, window: int = 3):
    """Pick k variables to slice; returns (vars, sliced line graph, reduced
    order, CostReport of one slice)."""
    chosen = []
    cur_lg, cur_order = lg, order
    for _ in range(k):
        steps = _replay(cur_lg, cur_order)
        if not steps:
            break
        width = max(r for r, _ in steps)
        score = {}
        for r, members in steps:
            if r >= width - window:
                for u in members:
                    score[u] = score.get(u, 0.0) + 2.0 ** r
        best = min(score, key=lambda u: (-score[u], u))
        chosen.append(best)
        cur_lg = remove_vertices(cur_lg, [best])
        cur_order = ContractionOrder(tuple(v for v in cur_order.sequence if v != best))
    report = contraction_width(cur_lg, cur_order)
    return chosen, cur_lg, cur_order, report


def slice_assignments(variables):
    """All 2^k bit assignments, first variable most significant."""
    variables = list(variables)
    return [dict(zip(variables, bits)) for bits in itertools.product((0, 1), repeat=len(variables))]
