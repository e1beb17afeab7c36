"""CPU oracle for the bucket-elimination hot path — TEST INFRASTRUCTURE ONLY.

This module is a compact numpy restatement of the reference `qtnsim`
algorithms that the B200 path replaces or feeds.  It exists so that the
tests (`tests/`), `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
reference arm can check and time the CUDA path against an independent CPU
computation on the same inputs.  Nothing in the product package imports it,
and the product path never falls back to it.

Parity pin: every function here is checked against golden vectors produced
by importing the real reference package (`/root/reference/pkg/src/qtnsim`)
in the build container — see `tests/golden/make_golden.py` and
`tests/test_oracle_golden.py`.  Paths below are relative to
`/root/reference/pkg/src/qtnsim/`.

Conventions (identical to the reference):
  * tensor data has shape (2,)*rank, axis k <-> variables[k], C order, so the
    first variable is the most significant bit of the flat index;
  * gate matrices: row = output, column = input, first qubit most significant.
"""

from __future__ import annotations

import cmath
import math

import numpy as np

# ----------------------------------------------------------------------------
# graphs  (bench.py:48-78)
# ----------------------------------------------------------------------------


def random_regular_graph(n: int, d: int, seed: int):
    """Configuration-model d-regular graph; follows bench.py:48-78.

    Returns the sorted edge list [(lo, hi), ...].  Same RNG stream
    (`default_rng(seed).permutation`) and rejection rule as the reference.
    """
    if n < 1 or d < 0 or d >= n or (n * d) % 2:
        raise ValueError("infeasible regular graph")
    rng = np.random.default_rng(seed)
    stubs = np.repeat(np.arange(n), d)
    for _ in range(100_000):
        perm = rng.permutation(stubs)
        a, b = perm[0::2], perm[1::2]
        if (a == b).any():
            continue
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        if np.unique(lo.astype(np.int64) * n + hi).size != lo.size:
            continue
        return sorted(zip(lo.tolist(), hi.tolist()))
    raise RuntimeError("no simple pairing found")


def seeded_angles(p: int, seed: int = 0):
    """SURVEY §8(d) convention: gammas then betas, uniform [0, pi)."""
    rng = np.random.default_rng(seed)
    g = rng.uniform(0.0, math.pi, p)
    b = rng.uniform(0.0, math.pi, p)
    return [float(x) for x in g], [float(x) for x in b]


# ----------------------------------------------------------------------------
# gates and circuits  (circuit.py:186-250)
# ----------------------------------------------------------------------------

_S = 1.0 / math.sqrt(2.0)
_H = np.array([[_S, _S], [_S, -_S]], dtype=complex)


def gate_matrix(kind: str, param=None) -> np.ndarray:
    """Dense gate matrix; conventions of circuit.py:186-205."""
    if kind == "H":
        return np.array([[1, 1], [1, -1]], dtype=complex) * _S
    if kind == "ZPOW":
        return np.array([[1, 0], [0, cmath.exp(-1j * param)]], dtype=complex)
    if kind == "XPOW":
        z = np.array([[1, 0], [0, cmath.exp(-1j * param)]], dtype=complex)
        h = np.array([[1, 1], [1, -1]], dtype=complex) * _S
        return h @ z @ h
    if kind == "CNOT":
        m = np.eye(4, dtype=complex)
        m[2:, 2:] = [[0, 1], [1, 0]]
        return m
    if kind == "ZZ":
        r = cmath.exp(1j * param)
        return np.diag([r, r.conjugate(), r.conjugate(), r]).astype(complex)
    raise ValueError(kind)


DIAGONAL_KINDS = ("ZPOW", "ZZ")


def qaoa_gates(n, edges, gammas, betas, fused):
    """Ansatz gate list + phase; circuit.py:217-250 (H layer, then per round
    the edge layer in listed order and the mixer in ascending qubit order)."""
    gates = [("H", (q,), None) for q in range(n)]
    phase = 1.0 + 0.0j
    for g, b in zip(gammas, betas):
        for (i, j) in edges:
            if fused:
                gates.append(("ZZ", (i, j), g))
                phase *= cmath.exp(-1j * g)
            else:
                gates += [("CNOT", (i, j), None), ("ZPOW", (j,), 2.0 * g), ("CNOT", (i, j), None)]
        for k in range(n):
            if fused:
                gates.append(("XPOW", (k,), 2.0 * b))
            else:
                gates += [("H", (k,), None), ("ZPOW", (k,), 2.0 * b), ("H", (k,), None)]
    return gates, phase


def _inverse(gate):
    kind, qs, t = gate
    return (kind, qs, None if t is None else -t)


def edge_cone_gates(n, edges, edge, gammas, betas, fused):
    """Per-round pruned light cone of Z_i Z_j (SURVEY §8a row A14').

    There is no reference function for this (SPEC.md:8 puts energies out of
    scope); it is composed only from reference gate vocabulary
    (circuit.py:134-152) so that the reference `circuit_to_network` /
    `contract` evaluate <psi|Z_i Z_j|psi> = <0|U^dag Z_i Z_j U|0>.
    Returns (m, gates, phase, cone_vertices).
    """
    p = len(gammas)
    adj = {v: set() for v in range(n)}
    for a, b in edges:
        adj[a].add(b)
        adj[b].add(a)
    shells = [set(edge)]
    for _ in range(p):
        grown = set(shells[-1])
        for v in shells[-1]:
            grown |= adj[v]
        shells.append(grown)
    cone = sorted(shells[p])
    loc = {v: k for k, v in enumerate(cone)}
    u = [("H", (loc[v],), None) for v in cone]
    phase = 1.0 + 0.0j
    for q in range(p):
        live = shells[p - 1 - q]
        g, b = gammas[q], betas[q]
        for (i, j) in edges:
            if i in live or j in live:
                a, c = loc[i], loc[j]
                if fused:
                    u.append(("ZZ", (a, c), g))
                    phase *= cmath.exp(-1j * g)
                else:
                    u += [("CNOT", (a, c), None), ("ZPOW", (c,), 2.0 * g), ("CNOT", (a, c), None)]
        for v in sorted(live):
            k = loc[v]
            if fused:
                u.append(("XPOW", (k,), 2.0 * b))
            else:
                u += [("H", (k,), None), ("ZPOW", (k,), 2.0 * b), ("H", (k,), None)]
    obs = [("ZPOW", (loc[edge[0]],), math.pi), ("ZPOW", (loc[edge[1]],), math.pi)]
    gates = u + obs + [_inverse(g) for g in reversed(u)]
    # U carries `phase`, U^dag carries its conjugate: the product is exactly 1.
    return len(cone), gates, 1.0 + 0.0j, cone


# ----------------------------------------------------------------------------
# tensor network  (network.py:93-165, 168-218)
# ----------------------------------------------------------------------------


def circuit_tensors(m, gates, phase, diagonal, bits):
    """Circuit -> (tensors, n_vars, fixed); network.py:93-150.

    tensors: list of (variables tuple, complex128 ndarray of shape (2,)*rank).
    """
    tensors = []
    cur = list(range(m))
    nv = m
    for q in range(m):
        tensors.append(((q,), np.array([1.0, 0.0], dtype=complex)))
    for kind, qs, t in gates:
        mat = gate_matrix(kind, t)
        if diagonal and kind in DIAGONAL_KINDS:
            d = np.diagonal(mat).copy()
            if len(qs) == 1:
                tensors.append(((cur[qs[0]],), d))
            else:
                tensors.append(((cur[qs[0]], cur[qs[1]]), d.reshape(2, 2)))
        elif len(qs) == 1:
            tensors.append(((nv, cur[qs[0]]), mat))
            cur[qs[0]] = nv
            nv += 1
        else:
            a, b = qs
            tensors.append(((nv, nv + 1, cur[a], cur[b]), mat.reshape(2, 2, 2, 2)))
            cur[a], cur[b] = nv, nv + 1
            nv += 2
    fixed = {cur[q]: int(bits[q]) for q in range(m)}
    tensors.append(((), np.asarray(phase, dtype=complex)))
    return tensors, nv, fixed


def slice_fixed(tensors, fixed):
    """Pin fixed variables by basic indexing; network.py:153-165."""
    out = []
    for vs, data in tensors:
        if any(v in fixed for v in vs):
            idx = tuple(fixed[v] if v in fixed else slice(None) for v in vs)
            out.append((tuple(v for v in vs if v not in fixed), np.asarray(data[idx])))
        else:
            out.append((vs, data))
    return out


def hyperedges(tensors, fixed):
    """Line-graph hyperedges (network.py:210-218): unfixed vars of rank>=1
    sliced tensors."""
    return [vs for vs, _ in slice_fixed(tensors, fixed) if len(vs) >= 1]


# ----------------------------------------------------------------------------
# ordering  (ordering.py:46-189)
# ----------------------------------------------------------------------------


def _adjacency(vertices, edges):
    index = {v: k for k, v in enumerate(vertices)}
    adj = [set() for _ in vertices]
    for e in edges:
        for x in e:
            for y in e:
                if x != y:
                    adj[index[x]].add(index[y])
    return adj


def _elim(adj, v):
    nb = adj[v]
    for a in nb:
        adj[a].discard(v)
        adj[a] |= nb - {a}
    adj[v] = set()
    return len(nb)


def width_of(vertices, edges, order):
    """Step ranks along `order`; ordering.py:79-100."""
    vertices = sorted(vertices)
    index = {v: k for k, v in enumerate(vertices)}
    adj = _adjacency(vertices, edges)
    return [_elim(adj, index[v]) for v in order]


def rgreedy(vertices, edges, n_repeats=10, temp=0.02, seed=0):
    """Randomized greedy, best of n passes; ordering.py:106-189.

    Pass 0 is min-degree (first minimum); pass k samples with Boltzmann
    weights from default_rng(seed + k).  Best by (width, flops_sum, pass).
    Returns (order, step_ranks).
    """
    vertices = sorted(vertices)
    dead = np.iinfo(np.int64).max
    best = None
    for rep in range(n_repeats):
        adj = _adjacency(vertices, edges)
        deg = np.array([len(s) for s in adj], dtype=np.int64)
        rng = np.random.default_rng(seed + rep) if rep else None
        seq, ranks = [], []
        for _ in range(len(vertices)):
            if rep == 0:
                v = int(deg.argmin())
            else:
                alive = deg != dead
                low = deg[alive].min()
                if temp == 0.0:
                    w = (alive & (deg == low)).astype(np.float64)
                else:
                    w = np.exp(-(deg - low) / temp, where=alive, out=np.zeros(len(deg)))
                c = np.cumsum(w)
                v = int(np.searchsorted(c, rng.random() * c[-1], side="right"))
            nb = list(adj[v])
            ranks.append(_elim(adj, v))
            for a in nb:
                deg[a] = len(adj[a])
            deg[v] = dead
            seq.append(v)
        width = max(ranks, default=0)
        flops = float(sum(2.0 ** (r + 1) for r in ranks))
        key = (width, flops, rep)
        if best is None or key < best[0]:
            best = (key, seq, ranks)
    _, seq, ranks = best
    return [vertices[i] for i in seq], ranks


# ----------------------------------------------------------------------------
# contraction  (contraction.py:42-123)
# ----------------------------------------------------------------------------


class RankCap(RuntimeError):
    def __init__(self, rank, cap):
        super().__init__(f"intermediate of rank {rank} exceeds rank cap {cap}")
        self.rank, self.cap = rank, cap


def pair_product(va, da, vb, db):
    """Broadcast product on the union (a's vars first); contraction.py:42-54."""
    out = tuple(va) + tuple(v for v in vb if v not in set(va))
    lab = {v: k for k, v in enumerate(out)}
    d = np.einsum(da, [lab[v] for v in va], db, [lab[v] for v in vb], list(range(len(out))))
    return out, d


def bucket_eliminate(operands, v):
    """One bucket: product chain in the given order, then sum over v;
    contraction.py:90-96.  operands: list of (vars, data)."""
    va, da = operands[0]
    for vb, db in operands[1:]:
        va, da = pair_product(va, da, vb, db)
    ax = va.index(v)
    return va[:ax] + va[ax + 1:], da.sum(axis=ax)


def contract(tensors, n_vars, fixed, order, rank_cap=30, cast=None):
    """Bucket elimination along `order`; contraction.py:57-111.

    `cast`, if given, is applied to every bucket output (used only by the
    precision-emulation tests).  Returns (value, step_ranks).
    """
    unfixed = [v for v in range(n_vars) if v not in fixed]
    if sorted(order) != unfixed:
        raise ValueError("order is not a permutation of the network's unfixed variables")
    live = {}
    by_var = {v: set() for v in unfixed}
    for k, (vs, d) in enumerate(slice_fixed(tensors, fixed)):
        live[k] = (vs, d)
        for v in vs:
            by_var[v].add(k)
    nid = len(live)
    scalar = 1.0 + 0.0j
    ranks = []
    for v in order:
        ids = sorted(by_var.pop(v))
        if not ids:
            scalar *= 2.0
            ranks.append(0)
            continue
        union = set()
        for k in ids:
            union.update(live[k][0])
        r = len(union) - 1
        if r > rank_cap:
            raise RankCap(r, rank_cap)
        ranks.append(r)
        vs, d = bucket_eliminate([live[k] for k in ids], v)
        if cast is not None:
            d = cast(d)
        for k in ids:
            for u in live.pop(k)[0]:
                if u != v:
                    by_var[u].discard(k)
        live[nid] = (vs, d)
        for u in vs:
            by_var[u].add(nid)
        nid += 1
    for vs, d in live.values():
        assert vs == ()
        scalar *= complex(d)
    return scalar, ranks


def direct_sum(tensors, n_vars, fixed):
    """Feynman-path enumeration (contraction.py:126-152), q <= 22 here."""
    unfixed = [v for v in range(n_vars) if v not in fixed]
    q = len(unfixed)
    if q > 22:
        raise ValueError("too many variables")
    pos = {v: q - 1 - k for k, v in enumerate(unfixed)}
    codes = np.arange(1 << q, dtype=np.int64)
    vals = np.ones(1 << q, dtype=complex)
    for vs, d in slice_fixed(tensors, fixed):
        idx = np.zeros(1 << q, dtype=np.int64)
        for v in vs:
            idx = (idx << 1) | ((codes >> pos[v]) & 1)
        vals *= np.asarray(d).reshape(-1)[idx]
    return complex(vals.sum())


def statevector(m, gates, phase):
    """Dense evolution from |0..0>; contraction.py:155-176."""
    if m > 24:
        raise ValueError("too many qubits")
    psi = np.zeros((2,) * m, dtype=complex)
    psi[(0,) * m] = 1.0
    for kind, qs, t in gates:
        mat = gate_matrix(kind, t)
        if len(qs) == 1:
            psi = np.moveaxis(np.tensordot(mat, psi, axes=([1], [qs[0]])), 0, qs[0])
        else:
            psi = np.tensordot(mat.reshape(2, 2, 2, 2), psi, axes=([2, 3], list(qs)))
            psi = np.moveaxis(psi, (0, 1), qs)
    return psi * phase


def zz_from_state(psi, i, j):
    """<Z_i Z_j> from |psi|^2."""
    prob = np.abs(psi) ** 2
    m = psi.ndim
    zi = np.array([1.0, -1.0]).reshape([2 if k == i else 1 for k in range(m)])
    zj = np.array([1.0, -1.0]).reshape([2 if k == j else 1 for k in range(m)])
    return float((prob * zi * zj).sum())


# ----------------------------------------------------------------------------
# end-to-end helpers used by the tests / bench reference arm
# ----------------------------------------------------------------------------

MODES = {
    "default": (False, False),
    "diagonal": (False, True),
    "zz": (True, False),
    "zz+diagonal": (True, True),
}  # name -> (fused, diagonal); pipeline.py:38-43


def edge_network(n, edges, edge, gammas, betas, mode):
    fused, diagonal = MODES[mode]
    m, gates, phase, _ = edge_cone_gates(n, edges, edge, gammas, betas, fused)
    return circuit_tensors(m, gates, phase, diagonal, "0" * m)


def edge_zz(n, edges, edge, gammas, betas, mode, order=None, rank_cap=30):
    """<Z_i Z_j> for one edge through the restated bucket elimination."""
    tensors, nv, fixed = edge_network(n, edges, edge, gammas, betas, mode)
    if order is None:
        verts = [v for v in range(nv) if v not in fixed]
        order, _ = rgreedy(verts, hyperedges(tensors, fixed))
    val, _ = contract(tensors, nv, fixed, order, rank_cap)
    return val


def energy_from_zz(zz_values):
    """MaxCut cost expectation E = sum_e (1 - <Z_iZ_j>)/2."""
    return float(sum((1.0 - complex(z).real) / 2.0 for z in zz_values))


def synthetic_bucket(w, m_small, seed, dtype=np.complex64):
    """Config-5 synthetic bucket: variables 0 = v, 1..w = x.

    Large operand: rank w+1 over a seeded permutation of (v, x_1..x_w).
    m_small operands, each rank-1 on (v,) or rank-2 on (v, x_r).
    Entries: re, im ~ N(0, 1) from default_rng(seed).
    Returns list of (vars, data) with the large operand first.
    """
    rng = np.random.default_rng(seed)
    perm = [int(x) for x in rng.permutation(w + 1)]
    def draw(shape):
        return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(dtype)
    ops = [(tuple(perm), draw((2,) * (w + 1)))]
    for _ in range(m_small):
        if rng.random() < 0.5:
            ops.append(((0,), draw((2,))))
        else:
            r = int(rng.integers(1, w + 1))
            ops.append(((0, r), draw((2, 2))))
    return ops


def bucket_sampled(outs, out_vars, operands_vars, fetch, v=0):
    """Selected outputs of one bucket, float64: for each flat output index o
    in `outs`, sum over the eliminated variable v of the product of every
    operand's entry at idx_t(o, v) — contraction.py:82-96 (the `_product`
    chain then `.sum`) evaluated only where asked, for buckets too large to
    materialise on the host (config 5 at w > 28).  Index maps follow the
    reference's C order (first variable = most significant bit,
    network.py:36-61).  fetch(t, flat_indices) returns operand t's entries."""
    outs = np.asarray(outs, dtype=np.int64)
    r = len(out_vars)
    val = {int(x): (outs >> (r - 1 - k)) & 1 for k, x in enumerate(out_vars)}
    acc = np.zeros(len(outs), dtype=np.complex128)
    for bit in (0, 1):
        val[v] = np.full(len(outs), bit, dtype=np.int64)
        prod = np.ones(len(outs), dtype=np.complex128)
        for t, vs in enumerate(operands_vars):
            idx = np.zeros(len(outs), dtype=np.int64)
            for pos, x in enumerate(vs):
                idx |= val[int(x)] << (len(vs) - 1 - pos)
            prod *= np.asarray(fetch(t, idx), dtype=np.complex128)
        acc += prod
    return acc
