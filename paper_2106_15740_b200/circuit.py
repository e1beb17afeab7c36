"""Gate-level circuit IR — host-side mirror of the reference vocabulary.

Mirrors the public names and conventions of
/root/reference/pkg/src/qtnsim/circuit.py (ProblemGraph 45-69, QaoaParams
72-90, GateKind/Gate 93-152, Circuit 155-176, gate_matrix 186-205,
is_diagonal 208-214, build_qaoa_maxcut_circuit 217-250)
so that networks built here are identical, tensor for tensor, to the
reference's.  The ZZ-fusion pass (circuit.py:253-318) and the text formats
(circuit.py:321-450) are out of scope: the fused ansatz is built
directly, as the reference's pipeline does (circuit.py:236-245).
"""

from __future__ import annotations

import cmath
import math
from dataclasses import dataclass
from enum import Enum

import numpy as np

__all__ = [
    "GateKind",
    "Gate",
    "Circuit",
    "ProblemGraph",
    "QaoaParams",
    "gate_matrix",
    "is_diagonal",
    "build_qaoa_maxcut_circuit",
]


@dataclass(frozen=True)
class ProblemGraph:
    """Undirected simple graph of a MaxCut instance (0-indexed nodes)."""

    node_count: int
    edges: tuple

    def __post_init__(self):
        edges = tuple((int(a), int(b)) for a, b in self.edges)
        object.__setattr__(self, "edges", edges)
        if self.node_count < 1:
            raise ValueError("node_count must be >= 1")
        keys = set()
        for a, b in edges:
            if a == b:
                raise ValueError(f"self-loop on node {a}")
            if min(a, b) < 0 or max(a, b) >= self.node_count:
                raise ValueError(f"edge ({a}, {b}) out of range for {self.node_count} nodes")
            k = (min(a, b), max(a, b))
            if k in keys:
                raise ValueError(f"duplicate edge ({a}, {b})")
            keys.add(k)

    @property
    def edge_count(self) -> int:
        return len(self.edges)


@dataclass(frozen=True)
class QaoaParams:
    """Cost (gamma) and mixer (beta) angles in radians, one per round."""

    gammas: tuple
    betas: tuple

    def __post_init__(self):
        object.__setattr__(self, "gammas", tuple(float(x) for x in self.gammas))
        object.__setattr__(self, "betas", tuple(float(x) for x in self.betas))
        if len(self.gammas) != len(self.betas):
            raise ValueError(
                f"angle vectors must have equal length, got {len(self.gammas)} gammas "
                f"and {len(self.betas)} betas"
            )

    @property
    def p(self) -> int:
        return len(self.gammas)

    def as_vector(self) -> np.ndarray:
        """[gamma_1..gamma_p, beta_1..beta_p] — the device angle layout."""
        return np.asarray(self.gammas + self.betas, dtype=np.float64)


class GateKind(Enum):
    H = "H"
    ZPOW = "ZPOW"
    XPOW = "XPOW"
    CNOT = "CNOT"
    ZZ = "ZZ"


_ARITY = {GateKind.H: 1, GateKind.ZPOW: 1, GateKind.XPOW: 1, GateKind.CNOT: 2, GateKind.ZZ: 2}
_HAS_PARAM = {GateKind.ZPOW, GateKind.XPOW, GateKind.ZZ}
_DIAGONAL = {GateKind.ZPOW, GateKind.ZZ}


@dataclass(frozen=True)
class Gate:
    kind: GateKind
    qubits: tuple
    param: float | None = None

    def __post_init__(self):
        qs = tuple(int(q) for q in self.qubits)
        object.__setattr__(self, "qubits", qs)
        if self.param is not None:
            object.__setattr__(self, "param", float(self.param))
        if len(qs) != _ARITY[self.kind]:
            raise ValueError(f"{self.kind.value} acts on {_ARITY[self.kind]} qubit(s), got {qs}")
        if len(set(qs)) != len(qs):
            raise ValueError(f"repeated qubit in {self.kind.value} gate: {qs}")
        if any(q < 0 for q in qs):
            raise ValueError(f"negative qubit index in {qs}")
        if (self.param is None) == (self.kind in _HAS_PARAM):
            raise ValueError(f"{self.kind.value} parameter mismatch")

    @staticmethod
    def h(q):
        return Gate(GateKind.H, (q,))

    @staticmethod
    def zpow(q, t):
        return Gate(GateKind.ZPOW, (q,), t)

    @staticmethod
    def xpow(q, t):
        return Gate(GateKind.XPOW, (q,), t)

    @staticmethod
    def cnot(control, target):
        return Gate(GateKind.CNOT, (control, target))

    @staticmethod
    def zz(q1, q2, gamma):
        return Gate(GateKind.ZZ, (q1, q2), gamma)

    def inverse(self) -> "Gate":
        """H and CNOT are self-inverse; the rotations negate their angle."""
        return self if self.param is None else Gate(self.kind, self.qubits, -self.param)


@dataclass(frozen=True)
class Circuit:
    """Gate list over `qubit_count` qubits with an exact global phase."""

    qubit_count: int
    gates: tuple = ()
    phase: complex = 1.0 + 0.0j

    def __post_init__(self):
        object.__setattr__(self, "gates", tuple(self.gates))
        object.__setattr__(self, "phase", complex(self.phase))
        if self.qubit_count < 1:
            raise ValueError("qubit_count must be >= 1")
        if abs(abs(self.phase) - 1.0) > 1e-12:
            raise ValueError(f"phase must have unit modulus, got |phase| = {abs(self.phase)}")
        for g in self.gates:
            if max(g.qubits) >= self.qubit_count:
                raise ValueError(f"gate {g} out of range for {self.qubit_count} qubits")

    @property
    def gate_count(self) -> int:
        return len(self.gates)


_R2 = 1.0 / math.sqrt(2.0)
_HMAT = np.array([[1, 1], [1, -1]], dtype=complex) * _R2


def gate_matrix(gate: Gate) -> np.ndarray:
    """Computational-basis matrix (row = output, first qubit = MSB).

    ZPow(t) = diag(1, e^{-it}); XPow(t) = H ZPow(t) H; ZZ(g) =
    diag(e^{ig}, e^{-ig}, e^{-ig}, e^{ig}) — the reference conventions.
    """
    k = gate.kind
    if k is GateKind.H:
        return _HMAT.copy()
    if k is GateKind.ZPOW or k is GateKind.XPOW:
        z = np.array([[1, 0], [0, cmath.exp(-1j * gate.param)]], dtype=complex)
        return z if k is GateKind.ZPOW else _HMAT @ z @ _HMAT
    if k is GateKind.CNOT:
        m = np.zeros((4, 4), dtype=complex)
        m[0, 0] = m[1, 1] = m[2, 3] = m[3, 2] = 1.0
        return m
    if k is GateKind.ZZ:
        r = cmath.exp(1j * gate.param)
        return np.diag([r, r.conjugate(), r.conjugate(), r]).astype(complex)
    raise ValueError(f"unknown gate kind {k}")


def is_diagonal(gate: Gate) -> bool:
    return gate.kind in _DIAGONAL


def build_qaoa_maxcut_circuit(graph: ProblemGraph, params: QaoaParams, fused: bool = False) -> Circuit:
    """H on every qubit, then per round the edge layer and the mixer layer."""
    gates = [Gate.h(q) for q in range(graph.node_count)]
    phase = 1.0 + 0.0j
    for gamma, beta in zip(params.gammas, params.betas):
        for i, j in graph.edges:
            if fused:
                gates.append(Gate.zz(i, j, gamma))
                phase *= cmath.exp(-1j * gamma)
            else:
                gates += [Gate.cnot(i, j), Gate.zpow(j, 2.0 * gamma), Gate.cnot(i, j)]
        for q in range(graph.node_count):
            if fused:
                gates.append(Gate.xpow(q, 2.0 * beta))
            else:
                gates += [Gate.h(q), Gate.zpow(q, 2.0 * beta), Gate.h(q)]
    return Circuit(graph.node_count, tuple(gates), phase)
