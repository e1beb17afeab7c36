"""Per-edge light-cone networks for QAOA MaxCut energies.

The reference has no energy path (SPEC.md:8, PAPER.md:185-187 defer it); the
north star asks for one built only from reference primitives.  For edge
(i, j) and depth p the cone is pruned round by round (PAPER.md:174-180
lightcone optimisation): with S_r the vertices within graph distance r of
{i, j}, round q (1-based) keeps ZZ(gamma_q) on every edge with an endpoint
in S_{p-q} and the mixer on S_{p-q}; H acts on S_p.  The cone qubits are S_p
relabelled 0..m-1 in ascending vertex order; edges keep the sorted order of
`random_regular_graph` (bench.py:74) and the mixer runs in ascending qubit
order (circuit.py:243-249).  The observable Z_i Z_j is ZPow(pi) on both
qubits (circuit.py:195-196: ZPow(pi) = diag(1, -1)), followed by the
inverse cone.  Then

    <Z_i Z_j> = <0| U_cone^dag Z_i Z_j U_cone |0>
              = contract(circuit_to_network(cone, mode, "0"*m), order)

with the reference `circuit_to_network` (network.py:93-150) and
`rgreedy_order` (ordering.py:154-189) unchanged.  The phase is exactly 1
(U's phase times its conjugate).

Angles enter the cone only through the gate parameters, so the network
STRUCTURE — and hence the order and the compiled plan — depends on (graph,
edge, p, mode) only.  `EnergyTemplate` records, per tensor, which gate and
which angle produce its data, so new angles only re-run the on-device
generator (csrc tensorgen_kernel), not the host pipeline.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .circuit import Circuit, Gate, GateKind, ProblemGraph, QaoaParams
from .network import LineGraph, TensorNetwork, circuit_to_network
from .pipeline import get_mode

__all__ = [
    "SymbolicGate",
    "edge_lightcone_gates",
    "build_edge_lightcone_circuit",
    "build_energy_network",
    "EnergyTemplate",
    "energy_template",
]


@dataclass(frozen=True)
class SymbolicGate:
    """A gate whose angle is `scale * angles[angle] + offset` (angle = -1:
    constant `offset`); angles = [gamma_1..gamma_p, beta_1..beta_p]."""

    kind: GateKind
    qubits: tuple
    angle: int = -1
    scale: float = 0.0
    offset: float = 0.0

    @property
    def parametric(self) -> bool:
        return self.kind in (GateKind.ZPOW, GateKind.XPOW, GateKind.ZZ)

    def value(self, angles) -> float | None:
        if not self.parametric:
            return None
        if self.angle < 0:
            return self.offset
        return self.scale * float(angles[self.angle]) + self.offset

    def inverse(self) -> "SymbolicGate":
        if not self.parametric:
            return self
        return SymbolicGate(self.kind, self.qubits, self.angle, -self.scale, -self.offset)

    def instantiate(self, angles) -> Gate:
        return Gate(self.kind, self.qubits, self.value(angles))


def _shells(graph: ProblemGraph, edge, p):
    adj = [set() for _ in range(graph.node_count)]
    for a, b in graph.edges:
        adj[a].add(b)
        adj[b].add(a)
    shells = [set(edge)]
    for _ in range(p):
        nxt = set(shells[-1])
        for v in shells[-1]:
            nxt |= adj[v]
        shells.append(nxt)
    return shells


def edge_lightcone_gates(graph: ProblemGraph, edge, p: int, fused: bool):
    """Symbolic gate list of U^dag Z_i Z_j U for one edge.

    Returns (m, gates, cone_vertices)."""
    edge = (int(edge[0]), int(edge[1]))
    shells = _shells(graph, edge, p)
    cone = sorted(shells[p])
    loc = {v: k for k, v in enumerate(cone)}
    u = [SymbolicGate(GateKind.H, (loc[v],)) for v in cone]
    for q in range(p):
        live = shells[p - 1 - q]
        for i, j in graph.edges:
            if i not in live and j not in live:
                continue
            a, b = loc[i], loc[j]
            if fused:
                u.append(SymbolicGate(GateKind.ZZ, (a, b), q, 1.0))
            else:
                u += [SymbolicGate(GateKind.CNOT, (a, b)),
                      SymbolicGate(GateKind.ZPOW, (b,), q, 2.0),
                      SymbolicGate(GateKind.CNOT, (a, b))]
        for v in sorted(live):
            k = loc[v]
            if fused:
                u.append(SymbolicGate(GateKind.XPOW, (k,), p + q, 2.0))
            else:
                u += [SymbolicGate(GateKind.H, (k,)),
                      SymbolicGate(GateKind.ZPOW, (k,), p + q, 2.0),
                      SymbolicGate(GateKind.H, (k,))]
    obs = [SymbolicGate(GateKind.ZPOW, (loc[edge[0]],), -1, 0.0, math.pi),
           SymbolicGate(GateKind.ZPOW, (loc[edge[1]],), -1, 0.0, math.pi)]
    return len(cone), u + obs + [g.inverse() for g in reversed(u)], cone


def _angle_vector(params: QaoaParams):
    return list(params.gammas) + list(params.betas)


def build_edge_lightcone_circuit(graph: ProblemGraph, edge, params: QaoaParams,
                                 fused: bool) -> Circuit:
    m, gates, _ = edge_lightcone_gates(graph, edge, params.p, fused)
    vec = _angle_vector(params)
    return Circuit(m, tuple(g.instantiate(vec) for g in gates), 1.0)


def build_energy_network(graph: ProblemGraph, edge, params: QaoaParams, mode) -> TensorNetwork:
    """The <Z_iZ_j> network of one edge (all-zeros output), mirroring
    `build_network` (pipeline.py:70-81)."""
    md = get_mode(mode)
    circ = build_edge_lightcone_circuit(graph, edge, params, md.fused)
    return circuit_to_network(circ, md.network_mode, "0" * circ.qubit_count)


_KIND_FULL = {GateKind.H: N.GATE_H, GateKind.ZPOW: N.GATE_ZPOW, GateKind.XPOW: N.GATE_XPOW,
              GateKind.CNOT: N.GATE_CNOT, GateKind.ZZ: N.GATE_ZZ}
_KIND_DIAG = {GateKind.ZPOW: N.GATE_ZPOW_DIAG, GateKind.ZZ: N.GATE_ZZ_DIAG}


@dataclass
class EnergyTemplate:
    """Angle-independent description of one edge's energy network.

    `tensors` keeps the unsliced description (full variables, gate kind,
    angle slot, scale, offset); `structure` / `recipes` are its slicing by
    `fixed` (network.py:153-165).  `resliced` adds more fixed variables —
    the 2^k slices of §8(e) — without re-walking the circuit."""

    edge: tuple
    m: int
    variable_count: int
    fixed: dict
    structure: list            # sliced variable tuples, network order
    recipes: np.ndarray        # RECIPE_DTYPE, out_offset relative to the network
    unfixed: tuple
    tensors: list = None       # (full vars, kind, angle, scale, offset)

    def line_graph(self) -> LineGraph:
        return LineGraph.from_hyperedges(self.unfixed, [s for s in self.structure if len(s) >= 1])

    def resliced(self, assignment: dict) -> "EnergyTemplate":
        """The same network with extra variables fixed to 0/1."""
        fixed = dict(self.fixed)
        for v, bit in assignment.items():
            if v in fixed:
                raise ValueError(f"variable {v} is already fixed")
            if bit not in (0, 1):
                raise ValueError("slice bits must be 0 or 1")
            fixed[int(v)] = int(bit)
        return _slice(self.edge, self.m, self.variable_count, fixed, self.tensors)


def _slice(edge, m, nvar, fixed, tens) -> EnergyTemplate:
    rec = np.zeros(len(tens), dtype=N.RECIPE_DTYPE)
    structure = []
    off = 0
    for k, (vs, kind, ang, sc, of) in enumerate(tens):
        keep = 0
        fbits = 0
        kept = []
        for pos, v in enumerate(vs):
            if v in fixed:
                fbits |= fixed[v] << pos
            else:
                keep |= 1 << pos
                kept.append(v)
        structure.append(tuple(kept))
        rec[k] = (off, sc, of, ang, kind, len(vs), keep, fbits)
        off += 1 << len(kept)
    unfixed = tuple(v for v in range(nvar) if v not in fixed)
    return EnergyTemplate((int(edge[0]), int(edge[1])), m, nvar, fixed, structure, rec, unfixed,
                          tens)


def energy_template(graph: ProblemGraph, edge, p: int, mode) -> EnergyTemplate:
    """Walk the symbolic cone exactly like `circuit_to_network` and record,
    per tensor, its variables and the recipe that generates its data."""
    md = get_mode(mode)
    m, gates, _ = edge_lightcone_gates(graph, edge, p, md.fused)
    tens = []  # (full vars, kind code, angle, scale, offset)
    wire = list(range(m))
    nvar = m
    for q in range(m):
        tens.append(((q,), N.GATE_INIT, -1, 0.0, 0.0))
    for g in gates:
        if md.diagonal and g.kind in _KIND_DIAG:
            tens.append((tuple(wire[q] for q in g.qubits), _KIND_DIAG[g.kind], g.angle, g.scale,
                         g.offset))
        elif len(g.qubits) == 1:
            (q,) = g.qubits
            tens.append(((nvar, wire[q]), _KIND_FULL[g.kind], g.angle, g.scale, g.offset))
            wire[q] = nvar
            nvar += 1
        else:
            a, b = g.qubits
            tens.append(((nvar, nvar + 1, wire[a], wire[b]), _KIND_FULL[g.kind], g.angle,
                         g.scale, g.offset))
            wire[a], wire[b] = nvar, nvar + 1
            nvar += 2
    fixed = {wire[q]: 0 for q in range(m)}
    tens.append(((), N.GATE_SCALAR, -1, 1.0, 0.0))  # phase exactly 1
    return _slice(edge, m, nvar, fixed, tens)
