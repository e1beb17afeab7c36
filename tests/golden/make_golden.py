"""Generate golden vectors by running the REAL reference package.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

Writes tests/golden/*.json.  The cone circuits are composed from reference
gate objects (`qtnsim.Gate`, circuit.py:134-152); everything downstream —
`circuit_to_network` (network.py:93-150), `line_graph` (network.py:210-218),
`rgreedy_order` (ordering.py:154-189), `contract` (contraction.py:114-123),
`statevector` (contraction.py:155-176), `random_regular_graph`
(bench.py:48-78) — is the unmodified reference code.
"""

from __future__ import annotations

import cmath
import json
import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import qtnsim as Q  # noqa: E402
from qtnsim.contraction import _contract_with_ranks, _product  # noqa: E402


def seeded_angles(p, seed=0):
    rng = np.random.default_rng(seed)
    g = rng.uniform(0.0, math.pi, p)
    b = rng.uniform(0.0, math.pi, p)
    return [float(x) for x in g], [float(x) for x in b]


def cone_circuit(graph, edge, gammas, betas, fused):
    """Per-round pruned light cone of Z_iZ_j built from reference Gates."""
    p = len(gammas)
    adj = {v: set() for v in range(graph.node_count)}
    for a, b in graph.edges:
        adj[a].add(b)
        adj[b].add(a)
    shells = [set(edge)]
    for _ in range(p):
        s = set(shells[-1])
        for v in shells[-1]:
            s |= adj[v]
        shells.append(s)
    cone = sorted(shells[p])
    loc = {v: k for k, v in enumerate(cone)}
    u = [Q.Gate.h(loc[v]) for v in cone]
    for q in range(p):
        live = shells[p - 1 - q]
        for (i, j) in graph.edges:
            if i in live or j in live:
                if fused:
                    u.append(Q.Gate.zz(loc[i], loc[j], gammas[q]))
                else:
                    u += [Q.Gate.cnot(loc[i], loc[j]), Q.Gate.zpow(loc[j], 2 * gammas[q]),
                          Q.Gate.cnot(loc[i], loc[j])]
        for v in sorted(live):
            if fused:
                u.append(Q.Gate.xpow(loc[v], 2 * betas[q]))
            else:
                u += [Q.Gate.h(loc[v]), Q.Gate.zpow(loc[v], 2 * betas[q]), Q.Gate.h(loc[v])]
    inv = []
    for g in reversed(u):
        inv.append(g if g.param is None else Q.Gate(g.kind, g.qubits, -g.param))
    obs = [Q.Gate.zpow(loc[edge[0]], math.pi), Q.Gate.zpow(loc[edge[1]], math.pi)]
    return Q.Circuit(len(cone), tuple(u + obs + inv), 1.0)


def structure_sig(net):
    """Order-sensitive description of the network: per tensor its variables."""
    return [list(t.variables) for t in net.tensors]


def data_checksum(net):
    acc = 0j
    for k, t in enumerate(net.tensors):
        flat = t.data.reshape(-1)
        w = 1.0 + 1e-3 * k + 1e-6 * np.arange(flat.size)
        acc += complex((flat * w).sum())
    return [acc.real, acc.imag]


def one_edge(graph, e_idx, gammas, betas, mode_name, keep_structure):
    mode = Q.get_mode(mode_name)
    edge = graph.edges[e_idx]
    circ = cone_circuit(graph, edge, gammas, betas, mode.fused)
    net = Q.circuit_to_network(circ, mode.network_mode, "0" * circ.qubit_count)
    lg = Q.line_graph(net)
    t0 = time.perf_counter()
    order, report = Q.rgreedy_order(lg, n_repeats=10, temp=0.02, seed=0)
    t_order = time.perf_counter() - t0
    t0 = time.perf_counter()
    val, ranks = _contract_with_ranks(net, order, Q.DEFAULT_RANK_CAP)
    t_con = time.perf_counter() - t0
    assert tuple(ranks) == report.step_ranks
    rec = {
        "edge_index": e_idx,
        "edge": list(edge),
        "m": circ.qubit_count,
        "gate_count": circ.gate_count,
        "n_vars": net.variable_count,
        "n_tensors": len(net.tensors),
        "fixed": sorted([int(k), int(v)] for k, v in net.fixed.items()),
        "order": list(order.sequence),
        "width": report.width,
        "flops_sum": report.flops_sum,
        "value": [val.real, val.imag],
        "data_checksum": data_checksum(net),
        "t_order_s": t_order,
        "t_contract_s": t_con,
    }
    if keep_structure:
        rec["structure"] = structure_sig(net)
    return rec


def config_block(n, p, modes, edge_subset=None, keep_structure=False):
    graph = Q.random_regular_graph(n, 3, 0)
    gammas, betas = seeded_angles(p, 0)
    out = {"n": n, "d": 3, "graph_seed": 0, "p": p, "gammas": gammas, "betas": betas,
           "edges": [list(e) for e in graph.edges], "modes": {}}
    idx = range(len(graph.edges)) if edge_subset is None else edge_subset
    for mode in modes:
        recs = [one_edge(graph, k, gammas, betas, mode, keep_structure) for k in idx]
        out["modes"][mode] = recs
        print(f"  N={n} p={p} {mode}: {len(recs)} edges, widths "
              f"{min(r['width'] for r in recs)}-{max(r['width'] for r in recs)}", flush=True)
    return out


def kats():
    """SPEC.md example values, computed with the reference."""
    res = {}
    g4 = Q.random_regular_graph(4, 3, 0)
    amp = {}
    for mname in Q.MODE_ORDER:
        net = Q.build_network(g4, 1, mname)
        order, rep = Q.rgreedy_order(Q.line_graph(net))
        amp[mname] = {"value": [Q.contract(net, order).real, Q.contract(net, order).imag],
                      "width": rep.width}
    res["k4_p1_default_angles"] = amp
    two = Q.ProblemGraph(2, ((0, 1),))
    circ = Q.build_qaoa_maxcut_circuit(two, Q.QaoaParams((0.4,), (0.7,)), fused=True)
    sv = Q.statevector_amplitude(circ, "00")
    res["n2_p1_g0.4_b0.7"] = [sv.real, sv.imag]
    circ0 = Q.build_qaoa_maxcut_circuit(Q.ProblemGraph(4, ()), Q.QaoaParams((), ()))
    res["p0_n4"] = Q.statevector_amplitude(circ0, "0000").real
    # statevector energy for config 1 (full N=20 circuit)
    g20 = Q.random_regular_graph(20, 3, 0)
    gam, bet = seeded_angles(1, 0)
    psi = Q.statevector(Q.build_qaoa_maxcut_circuit(g20, Q.QaoaParams(gam, bet), fused=True))
    prob = np.abs(psi) ** 2
    zz = []
    for i, j in g20.edges:
        z = np.ones((2,) * 20)
        sl = [slice(None)] * 20
        sl[i] = 1
        z[tuple(sl)] *= -1
        sl = [slice(None)] * 20
        sl[j] = 1
        z[tuple(sl)] *= -1
        zz.append(float((prob * z).sum()))
    res["config1_statevector_zz"] = zz
    return res


def synthetic_buckets():
    """Config-5-shaped buckets at small w through the reference bucket ops
    (`_product` chain + `.sum`, contraction.py:42-54, 90-96)."""
    out = []
    for w, m, seed in [(6, 4, 1), (8, 8, 2), (10, 16, 3), (9, 4, 4)]:
        rng = np.random.default_rng(seed)
        perm = [int(x) for x in rng.permutation(w + 1)]

        def draw(shape):
            return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)

        ops = [(tuple(perm), draw((2,) * (w + 1)))]
        for _ in range(m):
            if rng.random() < 0.5:
                ops.append(((0,), draw((2,))))
            else:
                ops.append(((0, int(rng.integers(1, w + 1))), draw((2, 2))))
        va, da = ops[0]
        for vb, db in ops[1:]:
            va, da = _product(va, da, vb, db)
        ax = va.index(0)
        res = da.sum(axis=ax)
        vs = va[:ax] + va[ax + 1:]
        out.append({
            "w": w, "m": m, "seed": seed,
            "operands": [{"vars": list(v), "re": d.real.reshape(-1).tolist(),
                          "im": d.imag.reshape(-1).tolist()} for v, d in ops],
            "out_vars": list(vs),
            "out_re": res.real.reshape(-1).tolist(),
            "out_im": res.imag.reshape(-1).tolist(),
        })
    return out


def amplitude_path():
    """Front end of the amplitude path: the reference's
    text formats, ZZ fusion, `cost`/`amplitude` CLI output and run_benchmark
    rows, on small instances."""
    import contextlib
    import io
    import tempfile

    from qtnsim.bench import BenchSpec, run_benchmark
    from qtnsim.cli import main as cli_main

    out = {"circuits": [], "cli": [], "bench": []}
    gate = lambda g: [g.kind.value, list(g.qubits), g.param]
    for n, p in ((4, 1), (6, 2), (8, 1)):
        graph = Q.random_regular_graph(n, 3, 0)
        params = Q.default_angles(p)
        raw = Q.build_qaoa_maxcut_circuit(graph, params, fused=False)
        fused = Q.fuse_zz(raw)
        with tempfile.TemporaryDirectory() as d:
            gp, cp = os.path.join(d, "g.txt"), os.path.join(d, "c.txt")
            Q.write_graph(graph, gp)
            Q.write_circuit(raw, cp)
            graph_text, circ_text = open(gp).read(), open(cp).read()
            rec = {"n": n, "p": p, "graph_text": graph_text, "circuit_text": circ_text,
                   "raw_gates": [gate(g) for g in raw.gates],
                   "fused_gates": [gate(g) for g in fused.gates],
                   "fused_phase": [fused.phase.real, fused.phase.imag]}
            out["circuits"].append(rec)
            for mode in Q.MODE_ORDER:
                for cmd in ("cost", "amplitude"):
                    buf = io.StringIO()
                    with contextlib.redirect_stdout(buf):
                        rc = cli_main([cmd, "--circuit", cp, "--mode", mode])
                    lines = [l for l in buf.getvalue().splitlines() if not l.startswith("order_seconds")]
                    out["cli"].append({"n": n, "p": p, "mode": mode, "cmd": cmd, "rc": rc,
                                       "stdout": lines})
    spec = BenchSpec(ns=(4, 6), ps=(1, 2), seeds=(0, 1), contract=True)
    for r in run_benchmark(spec):
        out["bench"].append({"graph_seed": r.graph_seed, "n": r.n, "p": r.p, "mode": r.mode,
                             "width": r.width, "memory_bytes": r.memory_bytes,
                             "contracted": r.contracted, "amp": [r.amp_re, r.amp_im]})
    return out


def main():
    which = set(sys.argv[1:]) or {"kat", "c1", "c2", "c3", "c4", "synth", "amp"}
    if "amp" in which:
        with open(os.path.join(HERE, "amplitude_path.json"), "w") as f:
            json.dump(amplitude_path(), f)
        print("amplitude path done", flush=True)
    if "kat" in which:
        with open(os.path.join(HERE, "kat.json"), "w") as f:
            json.dump(kats(), f)
        print("kat done", flush=True)
    if "synth" in which:
        with open(os.path.join(HERE, "synthetic_buckets.json"), "w") as f:
            json.dump(synthetic_buckets(), f)
        print("synth done", flush=True)
    if "c1" in which:
        blk = config_block(20, 1, list(Q.MODE_ORDER), keep_structure=True)
        with open(os.path.join(HERE, "config1.json"), "w") as f:
            json.dump(blk, f)
    if "c2" in which:
        blk = config_block(100, 2, ["zz+diagonal"])
        blk2 = config_block(100, 2, ["default"], edge_subset=list(range(0, 150, 10)))
        blk["modes"].update(blk2["modes"])
        with open(os.path.join(HERE, "config2.json"), "w") as f:
            json.dump(blk, f)
    if "c3" in which:
        blk = config_block(244, 3, ["zz+diagonal"])
        blk2 = config_block(244, 3, ["default"])  # all 366 edges: the energy is asserted
        blk["modes"].update(blk2["modes"])
        with open(os.path.join(HERE, "config3.json"), "w") as f:
            json.dump(blk, f)
    if "c4" in which:
        blk = config_block(1000, 5, ["zz+diagonal"], edge_subset=[0, 8, 16, 1058])
        with open(os.path.join(HERE, "config4.json"), "w") as f:
            json.dump(blk, f)


if __name__ == "__main__":
    main()
