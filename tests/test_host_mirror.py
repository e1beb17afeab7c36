"""CPU tests of the host side: reference-API mirror, native ordering passes,
plan compiler and C-ABI surface (no compute calls that need a GPU)."""

import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import paper_2106_15740_b200 as Q
from paper_2106_15740_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _checksum(net):
    acc = 0j
    for k, t in enumerate(net.tensors):
        flat = t.data.reshape(-1)
        acc += complex((flat * (1.0 + 1e-3 * k + 1e-6 * np.arange(flat.size))).sum())
    return acc


# ------------------------------------------------------------ C-ABI surface
def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "qtn_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(qtn_\w+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    lib = C.CDLL(N.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(N.EXPORTED)
    assert N.lib.qtn_version() >= 1


def test_no_cuda_is_loud():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    net = Q.build_network(Q.random_regular_graph(4, 3, 0), 1, "zz+diagonal")
    order = Q.greedy_order(Q.line_graph(net))
    with pytest.raises(RuntimeError):
        Q.contract(net, order)


# ------------------------------------------------------------ host mirror
@pytest.mark.parametrize("mode", list(Q.MODE_ORDER))
def test_config1_networks_identical_to_reference(golden, mode):
    G = golden("config1.json")
    graph = Q.random_regular_graph(20, 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    for r in G["modes"][mode]:
        net = Q.build_energy_network(graph, graph.edges[r["edge_index"]], params, mode)
        assert [list(t.variables) for t in net.tensors] == r["structure"]
        assert net.variable_count == r["n_vars"]
        assert sorted([k, v] for k, v in net.fixed.items()) == r["fixed"]
        cs = _checksum(net)
        assert abs(cs - complex(*r["data_checksum"])) < 1e-9


def _check_orders(G, cfg):
    graph = Q.random_regular_graph(G["n"], 3, 0)
    n = 0
    for mode, recs in G["modes"].items():
        for r in recs:
            tpl = Q.energy_template(graph, graph.edges[r["edge_index"]], G["p"], mode)
            order, rep = Q.rgreedy_order(tpl.line_graph())
            assert list(order.sequence) == r["order"], (cfg, mode, r["edge_index"])
            assert rep.width == r["width"] and rep.flops_sum == r["flops_sum"]
            assert Q.contraction_width(tpl.line_graph(), order) == rep
            n += 1
    return n


@pytest.mark.parametrize("cfg", ["config1.json", "config2.json", "config3.json", "config4.json"])
def test_orders_identical_to_reference(golden, cfg):
    _check_orders(golden(cfg), cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["config1.json", "config2.json", "config3.json", "config4.json"])
def test_orders_identical_to_reference_on_gpu_host(golden, cfg):
    """The same check on the B200 box's host: bench.py and EnergyPlan order
    there with the native rgreedy fed numpy variates and an exp table
    (ordering.py); the reference draws with a masked np.exp (ordering.py:146).
    Bit-identity must hold on that host's numpy/libm, not only here."""
    assert _check_orders(golden(cfg), cfg) > 0


def test_template_matches_circuit_to_network(golden):
    """The angle-free template (structure + recipes) describes exactly the
    network circuit_to_network builds; recipes re-evaluated on the host."""
    G = golden("config2.json")
    graph = Q.random_regular_graph(100, 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    vec = params.as_vector()
    for mode in Q.MODE_ORDER:
        for e in (0, 77):
            tpl = Q.energy_template(graph, graph.edges[e], 2, mode)
            net = Q.build_energy_network(graph, graph.edges[e], params, mode)
            sl = Q.sliced_tensors(net)
            assert [t.variables for t in sl] == tpl.structure
            assert tpl.fixed == net.fixed and tpl.variable_count == net.variable_count
            for t, rec in zip(sl, tpl.recipes):
                got = _eval_recipe(rec, vec)
                assert np.allclose(got, t.data.reshape(-1), atol=1e-15), (mode, e, rec)


def _eval_recipe(rec, angles):
    """Host re-statement of csrc tensorgen_kernel, for the test above."""
    kind, fr = int(rec["kind"]), int(rec["full_rank"])
    t = rec["scale"] * angles[rec["angle"]] + rec["offset"] if rec["angle"] >= 0 else rec["offset"]
    e = complex(math.cos(t), -math.sin(t))
    s = 1 / math.sqrt(2)
    if kind == N.GATE_INIT:
        full = np.array([1, 0], complex)
    elif kind == N.GATE_H:
        full = np.array([s, s, s, -s], complex)
    elif kind == N.GATE_ZPOW:
        full = np.array([1, 0, 0, e])
    elif kind == N.GATE_ZPOW_DIAG:
        full = np.array([1, e])
    elif kind == N.GATE_XPOW:
        full = 0.5 * np.array([1 + e, 1 - e, 1 - e, 1 + e])
    elif kind == N.GATE_CNOT:
        full = np.eye(4, dtype=complex)[[0, 1, 3, 2]].reshape(-1)
    elif kind == N.GATE_ZZ:
        r = complex(math.cos(t), math.sin(t))
        full = np.diag([r, r.conjugate(), r.conjugate(), r]).reshape(-1)
    elif kind == N.GATE_ZZ_DIAG:
        r = complex(math.cos(t), math.sin(t))
        full = np.array([r, r.conjugate(), r.conjugate(), r])
    elif kind == N.GATE_SCALAR:
        return np.array([complex(rec["scale"], rec["offset"])])
    full = full.reshape((2,) * fr)
    idx = tuple(slice(None) if (rec["keep_mask"] >> q) & 1 else (rec["fixed_bits"] >> q) & 1
                for q in range(fr))
    return np.asarray(full[idx]).reshape(-1)


def test_lightcone_sizes(golden):
    """Cone qubit counts: config 1: 5-6, config 2: 14 (SURVEY §8a A14')."""
    G = golden("config2.json")
    graph = Q.random_regular_graph(100, 3, 0)
    ms = {Q.energy_template(graph, e, 2, "zz+diagonal").m for e in graph.edges}
    assert ms <= set(range(10, 15)) and 14 in ms
    G1 = golden("config1.json")
    assert {r["m"] for r in G1["modes"]["zz+diagonal"]} <= {5, 6}


# ------------------------------------------------------------ plan compiler
def test_plan_peak_rank_equals_width_and_executor_choice(golden):
    G = golden("config3.json")
    graph = Q.random_regular_graph(244, 3, 0)
    for mode, want_exec in (("zz+diagonal", N.EXEC_SMEM), ("default", N.EXEC_HBM)):
        for r in G["modes"][mode][:4]:
            tpl = Q.energy_template(graph, graph.edges[r["edge_index"]], 3, mode)
            plan = Q.ContractionPlan(tpl.structure, tpl.variable_count, tpl.fixed, r["order"],
                                     dtype="complex64")
            assert plan.width == r["width"] == max(plan.step_ranks)
            assert plan.executor == want_exec
            assert plan.input_elems == sum(1 << len(s) for s in tpl.structure)
            if want_exec == N.EXEC_HBM:
                assert plan.workspace_bytes > 0
            else:
                assert plan.smem_bytes <= Q.contraction.DEFAULT_SMEM_BUDGET
            # forcing the HBM executor is always possible
            hb = Q.ContractionPlan(tpl.structure, tpl.variable_count, tpl.fixed, r["order"],
                                   smem_budget=0)
            assert hb.executor == N.EXEC_HBM


def test_plan_errors_before_allocation():
    graph = Q.random_regular_graph(20, 3, 0)
    params = Q.seeded_angles(1)
    net = Q.build_energy_network(graph, graph.edges[3], params, "default")
    order, rep = Q.rgreedy_order(Q.line_graph(net))
    sl = Q.sliced_tensors(net)
    st = [t.variables for t in sl]
    with pytest.raises(ValueError):
        Q.ContractionPlan(st, net.variable_count, net.fixed, order.sequence[:-1])
    bad = list(order.sequence)
    bad[0] = max(net.fixed)  # a fixed variable
    with pytest.raises(ValueError):
        Q.ContractionPlan(st, net.variable_count, net.fixed, bad)
    with pytest.raises(Q.RankCapExceeded) as ei:
        Q.ContractionPlan(st, net.variable_count, net.fixed, order.sequence, rank_cap=rep.width - 1)
    assert isinstance(ei.value, RuntimeError)
    # first offending bucket, reference semantics (contraction.py:85-87)
    first = next(x for x in rep.step_ranks if x > rep.width - 1)
    assert ei.value.rank == first and ei.value.cap == rep.width - 1
    # contract() itself raises ValueError for a non-permutation before touching CUDA
    with pytest.raises(ValueError):
        Q.contract(net, Q.ContractionOrder(order.sequence[:-1]))


def test_empty_buckets_and_scalars():
    """A variable in no tensor gives a factor 2 (contraction.py:77-81); a
    network with only scalars compiles to zero buckets."""
    t0 = Q.Tensor(0, (0,), np.array([1.0, 2.0]))
    net = Q.TensorNetwork((t0, Q.Tensor(1, (), np.array(3.0))), 3, {2: 0})
    plan, _ = Q.ContractionPlan.from_network(net, Q.ContractionOrder((1, 0)))
    assert plan.n_empty_buckets == 1 and plan.n_buckets == 1
    assert plan.step_ranks == (0, 0)
    only = Q.TensorNetwork((Q.Tensor(0, (), np.array(2.0)),), 1, {0: 1})
    plan2, _ = Q.ContractionPlan.from_network(only, Q.ContractionOrder(()))
    assert plan2.n_buckets == 0


def test_rgreedy_argument_errors_and_determinism():
    lg = Q.LineGraph.from_edges(range(6), [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 0), (0, 3)])
    with pytest.raises(ValueError):
        Q.rgreedy_order(lg, n_repeats=0)
    with pytest.raises(ValueError):
        Q.rgreedy_order(lg, temp=-1.0)
    a = Q.rgreedy_order(lg, 10, 0.02, 3)
    b = Q.rgreedy_order(lg, 10, 0.02, 3)
    assert a == b
    one = Q.rgreedy_order(lg, n_repeats=1)
    assert one[0] == Q.greedy_order(lg)
    z = Q.rgreedy_order(lg, 5, 0.0, 1)  # temp = 0: uniform among min-degree
    assert sorted(z[0].sequence) == list(range(6))


def test_rgreedy_matches_oracle_on_random_graphs():
    import qtn_oracle as O

    rng = np.random.default_rng(11)
    for trial in range(25):
        nv = int(rng.integers(3, 30))
        edges = []
        for _ in range(int(rng.integers(nv, 3 * nv))):
            k = int(rng.integers(1, 5))
            edges.append(tuple(int(x) for x in rng.choice(nv, size=min(k, nv), replace=False)))
        temp = [0.02, 0.5, 0.0][trial % 3]
        lg = Q.LineGraph.from_hyperedges(range(nv), edges)
        order, rep = Q.rgreedy_order(lg, 6, temp, trial)
        o2, r2 = O.rgreedy(list(range(nv)), edges, 6, temp, trial)
        assert list(order.sequence) == o2 and list(rep.step_ranks) == r2


def test_spec_examples_contraction_width():
    # SPEC: path a-b-c, order (b,a,c) -> ranks (2,1,0), width 2
    lg = Q.LineGraph.from_edges((0, 1, 2), [(0, 1), (1, 2)])
    rep = Q.contraction_width(lg, Q.ContractionOrder((1, 0, 2)))
    assert rep.step_ranks == (2, 1, 0) and rep.width == 2
    # star K_{1,3}: greedy eliminates leaves first, width 1
    star = Q.LineGraph.from_edges(range(4), [(0, 1), (0, 2), (0, 3)])
    o = Q.greedy_order(star)
    assert Q.contraction_width(star, o).width == 1
    with pytest.raises(ValueError):
        Q.contraction_width(lg, Q.ContractionOrder((0, 1)))


def test_shard_edges_lpt():
    costs = [5.0, 1.0, 1.0, 4.0, 3.0, 3.0]
    sh = Q.shard_edges(costs, 2)
    assert sorted(sum(sh, [])) == list(range(6))
    loads = [sum(costs[i] for i in s) for s in sh]
    assert max(loads) - min(loads) <= 1.0
    assert Q.shard_edges(costs, 2) == sh  # deterministic
    assert Q.shard_edges(costs, 8)[7] == []


# ------------------------------------------------------------------ slicing
def test_slices_sum_to_unsliced_value(golden):
    """2^k slices (extra fixed variables, reduced reference order) add up to
    the unsliced contraction (oracle contraction of each slice)."""
    import qtn_oracle as O
    from paper_2106_15740_b200.slicing import choose_slice_vars, slice_assignments

    G = golden("config2.json")
    graph = Q.random_regular_graph(100, 3, 0)
    edges = [tuple(e) for e in G["edges"]]
    for r in G["modes"]["zz+diagonal"][:3]:
        tpl = Q.energy_template(graph, graph.edges[r["edge_index"]], 2, "zz+diagonal")
        order, rep = Q.rgreedy_order(tpl.line_graph())
        for k in (1, 3):
            svars, lg2, o2, rep2 = choose_slice_vars(tpl.line_graph(), order, k)
            assert len(svars) == k and rep2.width <= rep.width
            tens, nv, fixed = O.edge_network(100, edges, edges[r["edge_index"]], G["gammas"],
                                             G["betas"], "zz+diagonal")
            total = 0j
            for a in slice_assignments(svars):
                t2 = tpl.resliced(a)
                assert sorted(o2.sequence) == list(t2.unfixed)
                val, ranks = O.contract(tens, nv, {**fixed, **a}, list(o2.sequence))
                assert max(ranks) == rep2.width
                total += val
            assert abs(total - complex(*r["value"])) < 1e-12


def test_slice_choice_config4_widths():
    """Edge #1058 (width 26): k=3 -> 23, k=6 -> 20."""
    from paper_2106_15740_b200.slicing import choose_slice_vars

    graph = Q.random_regular_graph(1000, 3, 0)
    tpl = Q.energy_template(graph, graph.edges[1058], 5, "zz+diagonal")
    order, rep = Q.rgreedy_order(tpl.line_graph())
    assert rep.width == 26
    assert choose_slice_vars(tpl.line_graph(), order, 3)[3].width == 23
    _, lg6, o6, rep6 = choose_slice_vars(tpl.line_graph(), order, 6)
    assert rep6.width == 20
    assert Q.contraction_width(lg6, o6) == rep6


def test_sliced_jobs_share_one_plan():
    graph = Q.random_regular_graph(100, 3, 0)
    jobs = Q.plan_edges(graph, 2, "zz+diagonal", [5], slice_k=2)
    assert len(jobs) == 4 and len({id(j.plan) for j in jobs}) == 1
    assert sum(j.weight for j in jobs) == 1.0
    assert all(j.template.structure == jobs[0].template.structure for j in jobs)
    assert len({tuple(j.template.recipes["fixed_bits"]) for j in jobs}) == 4


def test_threaded_planning_matches_serial():
    """plan_edges on a thread pool (native ordering + plan compiler release
    the GIL) gives the same jobs, orders and plans as the serial loop."""
    g = Q.random_regular_graph(100, 3, 0)
    ids = list(range(0, 150, 7))
    a = Q.plan_edges(g, 2, "zz+diagonal", ids, workers=1)
    b = Q.plan_edges(g, 2, "zz+diagonal", ids, workers=4)
    assert [j.index for j in a] == [j.index for j in b] == ids
    for x, y in zip(a, b):
        assert x.order.sequence == y.order.sequence
        assert x.report == y.report
        assert x.plan.step_ranks == y.plan.step_ranks
        assert x.plan.program_bytes == y.plan.program_bytes
        assert x.plan.alg_bytes == y.plan.alg_bytes


def test_plan_pack_layout_matches_input_offsets():
    """ContractionPlan.pack (one concatenate when the inputs lie back to back)
    places tensor k at input_offsets[k], sliced data included
    (network.py:153-165 slicing, contraction.py:66-73 input list)."""
    g = Q.random_regular_graph(20, 3, 0)
    net = Q.build_energy_network(g, g.edges[0], Q.seeded_angles(1, 0), "zz+diagonal")
    order, _ = Q.rgreedy_order(Q.line_graph(net))
    plan, sl = Q.ContractionPlan.from_network(net, order)
    datas = [t.data for t in sl]
    buf = plan.pack(datas)
    assert buf.shape == (plan.input_elems,)
    for off, d in zip(plan.input_offsets, datas):
        flat = np.asarray(d, dtype=np.complex128).reshape(-1)
        assert np.array_equal(buf[off: off + flat.size], flat)
