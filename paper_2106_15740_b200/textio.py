"""Graph and circuit text formats — the reference's file front end.

Restates the formats of /root/reference/pkg/src/qtnsim/circuit.py:321-450
(the `qtnsim` CLI reads them, cli.py:74-96):

* graph file: a header line "<node_count> <edge_count>", then one "u v" line
  per edge;
* circuit file: a header "qubits <N>", an optional "phase <re> <im>" line,
  then one gate per line — "H q", "ZPOW q t", "XPOW q t", "CNOT c t",
  "ZZ q1 q2 gamma".

Text after '#' is a comment; blank lines are skipped; keywords are
case-insensitive.  Malformed input raises ParseError (a ValueError naming the
file and line), which the CLI maps to exit code 1 like the reference.
"""

from __future__ import annotations

from .circuit import Circuit, Gate, GateKind, ProblemGraph

__all__ = ["ParseError", "read_graph", "write_graph", "read_circuit", "write_circuit"]


class ParseError(ValueError):
    """Malformed graph / circuit / spec file (path, 1-based line, reason)."""

    def __init__(self, path, line: int, message: str):
        super().__init__(f"{path}:{line}: {message}")
        self.path = str(path)
        self.line = line


def _lines(path):
    """(line number, tokens) of every non-empty, comment-stripped line."""
    out = []
    with open(path, "r", encoding="utf-8") as fh:
        for no, text in enumerate(fh, start=1):
            body = text.split("#", 1)[0].strip()
            if body:
                out.append((no, body.split()))
    return out


def _int(path, no, tok, what):
    try:
        return int(tok)
    except ValueError:
        raise ParseError(path, no, f"expected integer {what}, got {tok!r}") from None


def _float(path, no, tok, what):
    try:
        return float(tok)
    except ValueError:
        raise ParseError(path, no, f"expected number {what}, got {tok!r}") from None


def read_graph(path) -> ProblemGraph:
    lines = _lines(path)
    if not lines:
        raise ParseError(path, 1, "empty graph file")
    hno, head = lines[0]
    if len(head) != 2:
        raise ParseError(path, hno, "header must be '<node_count> <edge_count>'")
    n = _int(path, hno, head[0], "node count")
    m = _int(path, hno, head[1], "edge count")
    if len(lines) - 1 != m:
        raise ParseError(path, hno, f"expected {m} edge lines, found {len(lines) - 1}")
    edges = []
    for no, toks in lines[1:]:
        if len(toks) != 2:
            raise ParseError(path, no, "edge line must be 'u v'")
        edges.append((_int(path, no, toks[0], "node"), _int(path, no, toks[1], "node")))
    try:
        return ProblemGraph(n, tuple(edges))
    except ValueError as exc:
        raise ParseError(path, hno, str(exc)) from None


def write_graph(graph: ProblemGraph, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(f"{graph.node_count} {graph.edge_count}\n")
        fh.writelines(f"{u} {v}\n" for u, v in graph.edges)


# keyword -> (kind, number of qubits, has an angle)
_GATES = {
    "H": (GateKind.H, 1, False),
    "ZPOW": (GateKind.ZPOW, 1, True),
    "XPOW": (GateKind.XPOW, 1, True),
    "CNOT": (GateKind.CNOT, 2, False),
    "ZZ": (GateKind.ZZ, 2, True),
}


def read_circuit(path) -> Circuit:
    lines = _lines(path)
    if not lines:
        raise ParseError(path, 1, "empty circuit file")
    hno, head = lines[0]
    if len(head) != 2 or head[0].lower() != "qubits":
        raise ParseError(path, hno, "header must be 'qubits <N>'")
    nq = _int(path, hno, head[1], "qubit count")
    if nq < 1:
        raise ParseError(path, hno, "qubit count must be >= 1")
    body = lines[1:]
    phase = 1.0 + 0.0j
    if body and body[0][1][0].lower() == "phase":
        no, toks = body[0]
        if len(toks) != 3:
            raise ParseError(path, no, "phase line must be 'phase <re> <im>'")
        phase = complex(_float(path, no, toks[1], "phase real part"),
                        _float(path, no, toks[2], "phase imaginary part"))
        body = body[1:]
    gates = []
    for no, toks in body:
        key = toks[0].upper()
        if key not in _GATES:
            raise ParseError(path, no, f"unknown gate {toks[0]!r}")
        kind, arity, has_angle = _GATES[key]
        if len(toks) != 1 + arity + (1 if has_angle else 0):
            raise ParseError(path, no, f"{key} line needs {arity + (1 if has_angle else 0)} argument(s)")
        qubits = tuple(_int(path, no, t, "qubit index") for t in toks[1:1 + arity])
        angle = _float(path, no, toks[-1], "angle") if has_angle else None
        try:
            gate = Gate(kind, qubits, angle)
        except ValueError as exc:
            raise ParseError(path, no, str(exc)) from None
        if max(qubits) >= nq:
            raise ParseError(path, no, f"qubit index out of range for {nq} qubits")
        gates.append(gate)
    try:
        return Circuit(nq, tuple(gates), phase)
    except ValueError as exc:
        raise ParseError(path, hno, str(exc)) from None


def write_circuit(circuit: Circuit, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(f"qubits {circuit.qubit_count}\n")
        if circuit.phase != 1.0 + 0.0j:
            fh.write(f"phase {circuit.phase.real!r} {circuit.phase.imag!r}\n")
        for g in circuit.gates:
            qs = " ".join(str(q) for q in g.qubits)
            fh.write(f"{g.kind.value} {qs}\n" if g.param is None else f"{g.kind.value} {qs} {g.param!r}\n")
