"""GPU parity: the sm_100a path (through the C ABI) against the oracle and
the golden vectors produced by the real reference (tests/golden)."""

import math

import numpy as np
import pytest

import paper_2106_15740_b200 as Q
import qtn_oracle as O

pytestmark = pytest.mark.gpu


def _net_from_oracle(tensors, nv, fixed):
    ts = [Q.Tensor(k, vs, d) for k, (vs, d) in enumerate(tensors)]
    return Q.TensorNetwork(tuple(ts), nv, fixed)


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("mode", list(Q.MODE_ORDER))
def test_config1_contract_all_modes_c128(golden, mode):
    G = golden("config1.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    nets, orders, want = [], [], []
    for r in G["modes"][mode]:
        net = Q.build_energy_network(graph, graph.edges[r["edge_index"]], params, mode)
        order = Q.ContractionOrder(r["order"])
        nets.append(net)
        orders.append(order)
        want.append(complex(*r["value"]))
    got = Q.contract_many(nets, orders, dtype="complex128")
    for g, w in zip(got, want):
        assert abs(g - w) < 1e-12
    # and single-network entry point, with step ranks
    v, ranks = Q.contraction._contract_with_ranks(nets[0], orders[0], 30)
    assert abs(v - want[0]) < 1e-12
    assert max(ranks) == G["modes"][mode][0]["width"]


def test_config1_energy_matches_statevector(golden):
    G = golden("config1.json")
    kat = golden("kat.json")
    graph = Q.random_regular_graph(20, 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    want = sum((1 - z) / 2 for z in kat["config1_statevector_zz"])
    for mode in Q.MODE_ORDER:
        e = Q.energy_expectation(graph, params, mode=mode, dtype="complex128")
        assert abs(e - want) < 1e-10, (mode, e, want)


def test_config2_energy_and_edges(golden):
    G = golden("config2.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    plan = Q.EnergyPlan(graph, G["p"], "zz+diagonal", dtype="complex64")
    zz = plan.zz_values(params)
    recs = G["modes"]["zz+diagonal"]
    for r in recs:
        w = complex(*r["value"])
        assert abs(zz[r["edge_index"]] - w) < 1e-10
    want = sum((1 - r["value"][0]) / 2 for r in recs)
    e = plan.energies(params)[0]
    assert abs(e - want) / abs(want) < 1e-12


def test_config2_angle_batch_vs_oracle(golden):
    """Several angle sets in one launch, each against the oracle at its angles."""
    G = golden("config2.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    edges = [tuple(e) for e in G["edges"]]
    plan = Q.EnergyPlan(graph, 2, "zz+diagonal", edge_ids=list(range(0, 150, 15)))
    rng = np.random.default_rng(7)
    sets = rng.uniform(0, math.pi, (5, 4))
    got = plan.energies(sets)
    for s in range(5):
        g, b = list(sets[s, :2]), list(sets[s, 2:])
        zz = [O.edge_zz(100, edges, edges[e], g, b, "zz+diagonal") for e in plan.edge_ids]
        assert abs(got[s] - O.energy_from_zz(zz)) < 1e-10


@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-11), ("complex64", 1e-5)])
def test_config3_default_hbm_path(golden, dtype, tol):
    G = golden("config3.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    recs = G["modes"]["default"][:6]
    plan = Q.EnergyPlan(graph, G["p"], "default", dtype=dtype,
                        edge_ids=[r["edge_index"] for r in recs])
    assert plan.hbm_jobs, "config 3 default networks must take the HBM executor"
    zz = plan.zz_values(params)
    for r in recs:
        w = complex(*r["value"])
        assert abs(zz[r["edge_index"]] - w) <= tol * abs(w) + 1e-12


def test_config3_zzdiag_energy(golden):
    G = golden("config3.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    recs = G["modes"]["zz+diagonal"]
    plan = Q.EnergyPlan(graph, G["p"], "zz+diagonal", dtype="complex64")
    want = sum((1 - r["value"][0]) / 2 for r in recs)
    e = plan.energies(params)[0]
    assert abs(e - want) / abs(want) < 1e-10


@pytest.mark.parametrize("edge_index,tol", [(16, 1e-5), (1058, 1e-5)])
def test_config4_single_edge_c64(golden, edge_index, tol):
    G = golden("config4.json")
    rec = [r for r in G["modes"]["zz+diagonal"] if r["edge_index"] == edge_index][0]
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    plan = Q.EnergyPlan(graph, G["p"], "zz+diagonal", dtype="complex64", edge_ids=[edge_index])
    zz = plan.zz_values(params)[edge_index]
    w = complex(*rec["value"])
    assert abs(zz - w) / abs(w) < tol


def test_config4_edge16_c128(golden):
    G = golden("config4.json")
    rec = [r for r in G["modes"]["zz+diagonal"] if r["edge_index"] == 16][0]
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    plan = Q.EnergyPlan(graph, G["p"], "zz+diagonal", dtype="complex128", edge_ids=[16])
    zz = plan.zz_values(params)[16]
    w = complex(*rec["value"])
    assert abs(zz - w) / abs(w) < 1e-11


def test_synthetic_buckets_c_abi(golden):
    """qtn_bucket_contract on config-5-shaped buckets vs the reference bucket ops."""
    import ctypes as C

    import torch

    from paper_2106_15740_b200 import _native as N

    for case in golden("synthetic_buckets.json"):
        ops = case["operands"]
        datas = [np.asarray(o["re"]) + 1j * np.asarray(o["im"]) for o in ops]
        for c64 in (False, True):
            dt = torch.complex64 if c64 else torch.complex128
            dev = [torch.from_numpy(d).to(dt).cuda() for d in datas]
            ranks = np.asarray([len(o["vars"]) for o in ops], dtype=np.int32)
            offs = np.zeros(len(ops) + 1, dtype=np.int32)
            offs[1:] = np.cumsum(ranks)
            flat = np.asarray([v for o in ops for v in o["vars"]], dtype=np.int32)
            ptrs = (C.c_void_p * len(ops))(*[d.data_ptr() for d in dev])
            flags = np.full(len(ops), 1 if c64 else 0, dtype=np.uint8)
            ov = np.asarray(case["out_vars"], dtype=np.int32)
            out = torch.empty(1 << len(ov), dtype=dt, device="cuda")
            N.check(N.lib.qtn_bucket_contract(len(ops), N.i32(ranks), N.i32(offs), N.i32(flat),
                                              ptrs, N.u8(flags), 0, len(ov), N.i32(ov),
                                              1 if c64 else 0, out.data_ptr(),
                                              torch.cuda.current_stream().cuda_stream))
            got = out.cpu().numpy().astype(np.complex128)
            want = np.asarray(case["out_re"]) + 1j * np.asarray(case["out_im"])
            if c64:
                # operands rounded to complex64 first: compare against that
                ref_ops = [(tuple(o["vars"]), d.astype(np.complex64).astype(np.complex128))
                           for o, d in zip(ops, datas)]
                vs, ref = O.bucket_eliminate(
                    [(v, d.reshape((2,) * len(v))) for v, d in ref_ops], 0)
                assert list(vs) == case["out_vars"]
                want = ref.reshape(-1)
                tol = 1e-5
            else:
                tol = 1e-12
            err = np.abs(got - want).max() / np.abs(want).max()
            assert err < tol, (case["w"], case["m"], c64, err)
            if not c64:
                # a non-preferred output layout (reversed) takes the generic
                # gather kernel; compare against the transposed golden
                rv = ov[::-1].copy()
                out2 = torch.empty(1 << len(ov), dtype=dt, device="cuda")
                N.check(N.lib.qtn_bucket_contract(len(ops), N.i32(ranks), N.i32(offs),
                                                  N.i32(flat), ptrs, N.u8(flags), 0, len(rv),
                                                  N.i32(rv), 0, out2.data_ptr(),
                                                  torch.cuda.current_stream().cuda_stream))
                got2 = out2.cpu().numpy().reshape((2,) * len(ov))
                want2 = want.reshape((2,) * len(ov)).transpose(list(range(len(ov)))[::-1])
                assert np.abs(got2 - want2).max() / np.abs(want2).max() < 1e-12


def test_rank_cap_raised_before_execution():
    graph = Q.random_regular_graph(100, 3, 0)
    tpl = Q.energy_template(graph, graph.edges[0], 2, "default")
    order, rep = Q.rgreedy_order(tpl.line_graph())
    with pytest.raises(Q.RankCapExceeded) as ei:
        Q.ContractionPlan(tpl.structure, tpl.variable_count, tpl.fixed, order.sequence,
                          rank_cap=rep.width - 1)
    assert ei.value.cap == rep.width - 1


@pytest.mark.parametrize("edge_index,k", [(16, 3), (1058, 3)])
def test_config4_sliced_c64(golden, edge_index, k):
    """2^k slices of the config-4 network, one batch, summed on device."""
    G = golden("config4.json")
    rec = [r for r in G["modes"]["zz+diagonal"] if r["edge_index"] == edge_index][0]
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    plan = Q.EnergyPlan(graph, G["p"], "zz+diagonal", dtype="complex64", edge_ids=[edge_index],
                        slice_k=k)
    assert len(plan.jobs) == 2 ** k
    assert max(j.report.width for j in plan.jobs) < rec["width"]
    zz = plan.zz_values(params)[edge_index]
    w = complex(*rec["value"])
    assert abs(zz - w) / abs(w) < 1e-5
    e = plan.energies(params)[0]
    assert abs(e - (1 - w.real) / 2) < 1e-5


def test_config2_sliced_energy_c128(golden):
    G = golden("config2.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    plan = Q.EnergyPlan(graph, 2, "zz+diagonal", dtype="complex128", slice_k=1)
    want = sum((1 - r["value"][0]) / 2 for r in G["modes"]["zz+diagonal"])
    assert abs(plan.energies(params)[0] - want) < 1e-10


def test_fused_and_unfused_generation_agree(golden):
    """In-executor tensor generation (fused) == tensorgen + executor."""
    G = golden("config2.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    rng = np.random.default_rng(3)
    sets = rng.uniform(0, math.pi, (7, 4))
    plan = Q.EnergyPlan(graph, 2, "zz+diagonal", edge_ids=list(range(0, 150, 5)))
    fused = plan.energies(sets)
    plan.fused = False
    plan._bufs.clear()
    unfused = plan.energies(sets)
    assert np.allclose(fused, unfused, rtol=0, atol=1e-12)
    # default mode (FULL networks: H/CNOT/XPOW... all gate kinds), mixed executors
    G3 = golden("config3.json")
    g3 = Q.random_regular_graph(244, 3, 0)
    p3 = Q.EnergyPlan(g3, 3, "default", dtype="complex128", edge_ids=[0, 23])
    s3 = rng.uniform(0, math.pi, (3, 6))
    f3 = p3.energies(s3)
    p3.fused = False
    p3._bufs.clear()
    u3 = p3.energies(s3)
    assert np.allclose(f3, u3, rtol=0, atol=1e-11)


@pytest.fixture
def setmajor_min_sets(monkeypatch):
    """Switch the set-major executor threshold (read per call by the library)."""
    def set_(n):
        monkeypatch.setenv("QTN_SETMAJOR_MIN_SETS", str(n))
    return set_


@pytest.mark.parametrize("mode,slice_k", [("zz+diagonal", 0), ("zz+diagonal", 1), ("default", 0)])
def test_setmajor_matches_warp_executor(golden, setmajor_min_sets, mode, slice_k):
    """Set-major streaming executor (many angle sets) == warp-resident SMEM
    executor, every gate kind, sliced networks with rank-0 gate inputs."""
    rng = np.random.default_rng(11)
    if mode == "default":
        graph, p, ids = Q.random_regular_graph(244, 3, 0), 3, None
        # default-mode config-3 networks that fit the warp executor
        sets = rng.uniform(0, math.pi, (70, 6))
        plan = Q.EnergyPlan(graph, p, mode, dtype="complex128", edge_ids=list(range(0, 366, 7)))
    else:
        graph, p = Q.random_regular_graph(100, 3, 0), 2
        sets = rng.uniform(0, math.pi, (70, 4))
        plan = Q.EnergyPlan(graph, p, mode, dtype="complex128", slice_k=slice_k)
    setmajor_min_sets(0)
    warp = plan.energies(sets)
    plan._bufs.clear()
    setmajor_min_sets(1)
    sm = plan.energies(sets)
    assert plan.launches == plan.launches_per_eval(len(sets))
    assert np.allclose(sm, warp, rtol=1e-12, atol=1e-11), np.abs(sm - warp).max()


def test_setmajor_vs_oracle(golden, setmajor_min_sets):
    """Set-major executor against the oracle at each angle set, including a
    set count that is not a multiple of 32."""
    setmajor_min_sets(1)
    G = golden("config2.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    edges = [tuple(e) for e in G["edges"]]
    plan = Q.EnergyPlan(graph, 2, "zz+diagonal", dtype="complex128",
                        edge_ids=list(range(0, 150, 15)))
    plan._prepare()
    assert plan._batch.setmajor_elem_bytes(37) == 16
    rng = np.random.default_rng(17)
    sets = rng.uniform(0, math.pi, (37, 4))
    got = plan.energies(sets)
    for s in (0, 1, 31, 32, 36):
        g, b = list(sets[s, :2]), list(sets[s, 2:])
        zz = [O.edge_zz(100, edges, edges[e], g, b, "zz+diagonal") for e in plan.edge_ids]
        assert abs(got[s] - O.energy_from_zz(zz)) < 1e-10


# ---------------------------------------------------------------- amplitudes
def test_reference_amplitude_path_k4(golden):
    """The reference's own workload: build_network amplitudes (pipeline.py:70-81)
    of K4 at default_angles, all four modes (SPEC.md examples)."""
    kat = golden("kat.json")["k4_p1_default_angles"]
    graph = Q.random_regular_graph(4, 3, 0)
    for mode in Q.MODE_ORDER:
        net = Q.build_network(graph, 1, mode)
        order, rep = Q.rgreedy_order(Q.line_graph(net))
        assert rep.width == kat[mode]["width"]
        for dt, tol in (("complex128", 1e-13), ("complex64", 1e-6)):
            v = Q.contract(net, order, dtype=dt)
            assert abs(v - complex(*kat[mode]["value"])) < tol


def test_random_circuits_vs_statevector():
    """Random small circuits over the whole gate set, both network modes,
    greedy and rgreedy orders, SMEM and forced-HBM executors, against the
    oracle statevector amplitude."""
    rng = np.random.default_rng(5)
    kinds = ["H", "ZPOW", "XPOW", "CNOT", "ZZ"]
    for trial in range(12):
        n = int(rng.integers(2, 7))
        gates, ogates = [], []
        for _ in range(int(rng.integers(5, 25))):
            k = kinds[int(rng.integers(0, 5))]
            if k in ("CNOT", "ZZ"):
                a, b = (int(x) for x in rng.choice(n, 2, replace=False))
                qs = (a, b)
            else:
                qs = (int(rng.integers(0, n)),)
            t = float(rng.uniform(-3, 3)) if k in ("ZPOW", "XPOW", "ZZ") else None
            gates.append(Q.Gate(Q.GateKind[k], qs, t))
            ogates.append((k, qs, t))
        circ = Q.Circuit(n, tuple(gates), complex(np.exp(1j * rng.uniform(0, 6))))
        bits = "".join(str(int(x)) for x in rng.integers(0, 2, n))
        psi = O.statevector(n, ogates, circ.phase)
        want = complex(psi[tuple(int(c) for c in bits)])
        for mode in (Q.NetworkMode.FULL, Q.NetworkMode.DIAGONAL):
            net = Q.circuit_to_network(circ, mode, bits)
            lg = Q.line_graph(net)
            for order in (Q.greedy_order(lg), Q.rgreedy_order(lg, 4, 0.5, trial)[0]):
                for budget in (Q.contraction.DEFAULT_SMEM_BUDGET, 0):
                    v = Q.contract(net, order, smem_budget=budget)
                    assert abs(v - want) < 1e-12, (trial, mode, budget)


def test_contract_cached_structure_other_outputs_and_data():
    """One structure, many calls: contract() keeps the compiled plan of a
    structure and pins the fixed variables on the data only
    (network.py:153-165).  Every output bitstring of one circuit (same
    structure, other fixed values) and other gate angles (same structure,
    other data) against the oracle statevector."""
    from paper_2106_15740_b200 import contraction as CT

    rng = np.random.default_rng(11)
    n = 4
    for rep in range(2):
        gates, ogates = [], []
        for k, qs in (("H", (0,)), ("H", (1,)), ("H", (2,)), ("H", (3,)), ("ZZ", (0, 1)), ("ZZ", (1, 2)),
                      ("CNOT", (2, 3)), ("XPOW", (0,)), ("ZPOW", (3,)), ("ZZ", (0, 3)), ("XPOW", (2,))):
            t = float(rng.uniform(-3, 3)) if k in ("ZPOW", "XPOW", "ZZ") else None
            gates.append(Q.Gate(Q.GateKind[k], qs, t))
            ogates.append((k, qs, t))
        circ = Q.Circuit(n, tuple(gates), 1.0 + 0.0j)
        psi = O.statevector(n, ogates, circ.phase)
        for mode in (Q.NetworkMode.FULL, Q.NetworkMode.DIAGONAL):
            order = None
            n_runs = None
            for b in range(1 << n):
                bits = format(b, f"0{n}b")
                net = Q.circuit_to_network(circ, mode, bits)
                if order is None:
                    order = Q.greedy_order(Q.line_graph(net))
                v = Q.contract(net, order)
                assert abs(v - complex(psi[tuple(int(c) for c in bits)])) < 1e-12, (rep, mode, bits)
                if n_runs is None:
                    n_runs = set(CT._RUNS)
            assert set(CT._RUNS) == n_runs  # the 16 outputs share one compiled plan


def test_degenerate_networks():
    """Empty buckets (factor 2), scalar-only networks, a single variable."""
    t0 = Q.Tensor(0, (0,), np.array([1.0, 2.0 + 1j]))
    net = Q.TensorNetwork((t0, Q.Tensor(1, (), np.array(3.0))), 3, {2: 0})
    v = Q.contract(net, Q.ContractionOrder((1, 0)))
    assert abs(v - 2 * 3 * (3.0 + 1j)) < 1e-12
    only = Q.TensorNetwork((Q.Tensor(0, (), np.array(2.0 - 1j)),), 1, {0: 1})
    assert abs(Q.contract(only, Q.ContractionOrder(())) - (2.0 - 1j)) < 1e-15
    for budget in (Q.contraction.DEFAULT_SMEM_BUDGET, 0):
        assert abs(Q.contract(net, Q.ContractionOrder((0, 1)), smem_budget=budget)
                   - 6 * (3.0 + 1j)) < 1e-12


def test_hbm_small_bucket_kernel_matches_stream_kernel(golden, monkeypatch):
    """HBM networks: buckets of output rank <= 9 on the warp/CTA-per-bucket
    kernel give the same values as the tile pipeline (QTN_SMALL_R=-1), and
    both match the reference values."""
    G = golden("config3.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    recs = G["modes"]["default"][:8]
    ids = [r["edge_index"] for r in recs]
    vals = {}
    for small_r in ("-1", "9", "12"):
        monkeypatch.setenv("QTN_SMALL_R", small_r)
        plan = Q.EnergyPlan(graph, G["p"], "default", dtype="complex128", edge_ids=ids)
        vals[small_r] = plan.zz_values(params)
    for r in recs:
        w = complex(*r["value"])
        for small_r, zz in vals.items():
            assert abs(zz[r["edge_index"]] - w) <= 1e-11 * abs(w) + 1e-12, (small_r, r["edge_index"])


def test_setmajor_large_batch_and_graph_replay(golden, setmajor_min_sets):
    """Set-major at 1100 angle sets (2 sets per thread, partial last pass,
    split tail levels) equals the warp-resident executor; replaying the
    captured evaluation with new angles in the same buffers gives the new
    energies (graph reads the buffer contents, not captured values)."""
    graph = Q.random_regular_graph(100, 3, 0)
    plan = Q.EnergyPlan(graph, 2, "zz+diagonal", dtype="complex128",
                        edge_ids=list(range(0, 150, 6)))
    rng = np.random.default_rng(23)
    s1 = rng.uniform(0, math.pi, (1100, 4))
    s2 = rng.uniform(0, math.pi, (1100, 4))
    setmajor_min_sets(0)
    w1, w2 = plan.energies(s1), plan.energies(s2)
    plan._bufs.clear()
    setmajor_min_sets(1)
    assert plan._batch.uses_setmajor(1100)
    g1 = plan.energies(s1)
    g2 = plan.energies(s2)   # same buffers: replay of the captured graph
    g1b = plan.energies(s1)
    assert np.allclose(g1, w1, rtol=1e-12, atol=1e-11)
    assert np.allclose(g2, w2, rtol=1e-12, atol=1e-11)
    assert np.array_equal(g1, g1b)
    assert not np.allclose(g1, g2)


@pytest.mark.parametrize("min_r,max_k", [("0", "8"), ("18", "4")])
def test_fused_reduction_chains(golden, monkeypatch, min_r, max_k):
    """Chains of single-operand buckets as one multi-variable sum
    (reduce_kernel, default on for chains into rank >= 18): same values as
    the unfused buckets (QTN_FUSE_REDUCE=0) and the reference; loosened
    filters (min_r 0, max_k 8) fuse every chain, including those summing
    bit 0 of their source."""
    monkeypatch.setenv("QTN_FUSE_MIN_R", min_r)
    monkeypatch.setenv("QTN_FUSE_MAX_K", max_k)
    G = golden("config3.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    recs = G["modes"]["default"][:8]
    G4 = golden("config4.json")
    rec4 = complex(*[r for r in G4["modes"]["zz+diagonal"] if r["edge_index"] == 16][0]["value"])
    g4 = Q.random_regular_graph(G4["n"], 3, 0)
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("QTN_FUSE_REDUCE", flag)
        for dt in ("complex128", "complex64"):
            plan = Q.EnergyPlan(graph, G["p"], "default", dtype=dt,
                                edge_ids=[r["edge_index"] for r in recs])
            p4 = Q.EnergyPlan(g4, G4["p"], "zz+diagonal", dtype=dt, edge_ids=[16])
            out[flag, dt] = (plan.zz_values(params),
                             p4.zz_values(Q.QaoaParams(G4["gammas"], G4["betas"]))[16])
            assert plan.launches == plan.launches_per_eval(1)
    for dt, tol in (("complex128", 1e-11), ("complex64", 1e-5)):
        for r in recs:
            w = complex(*r["value"])
            e = r["edge_index"]
            assert abs(out["1", dt][0][e] - w) <= tol * abs(w) + 1e-12
            assert abs(out["1", dt][0][e] - out["0", dt][0][e]) <= tol * abs(w) + 1e-12
        assert abs(out["1", dt][1] - rec4) <= tol * abs(rec4)


def test_setmajor_limit_falls_back_to_warp_executor():
    """Complete graph K8 at p=1: buckets with 9 operands exceed the set-major
    form (<= 8); a 200-set evaluation then runs on the warp-resident executor
    and still matches the oracle."""
    import itertools

    graph = Q.ProblemGraph(8, tuple(itertools.combinations(range(8), 2)))
    plan = Q.EnergyPlan(graph, 1, "zz+diagonal", dtype="complex128")
    rng = np.random.default_rng(5)
    sets = rng.uniform(0, math.pi, (200, 2))
    got = plan.energies(sets)
    assert not plan._batch.uses_setmajor(200)
    edges = [tuple(e) for e in graph.edges]
    for s in (0, 199):
        zz = [O.edge_zz(8, edges, e, [sets[s, 0]], [sets[s, 1]], "zz+diagonal") for e in edges]
        assert abs(got[s] - O.energy_from_zz(zz)) < 1e-10


def test_contract_plan_cache_reuses_structure_with_new_data(golden):
    """contract() caches the compiled plan and device program per (sliced
    structure, order); a second network with the same structure but other
    tensor data (new angles) must give its own value."""
    graph = Q.random_regular_graph(20, 3, 0)
    edges = [tuple(e) for e in graph.edges]
    rng = np.random.default_rng(31)
    order = None
    for _ in range(3):
        g, b = list(rng.uniform(0, math.pi, 1)), list(rng.uniform(0, math.pi, 1))
        net = Q.build_energy_network(graph, graph.edges[3], Q.QaoaParams(g, b), "default")
        if order is None:
            order, _ = Q.rgreedy_order(Q.line_graph(net))
        got = Q.contract(net, order)
        tensors, nv, fixed = O.edge_network(20, edges, edges[3], g, b, "default")
        want, _ = O.contract(tensors, nv, fixed, list(order.sequence))
        assert abs(got - want) < 1e-12


# ------------------------------------------------ complex64 set-major rows
def _setmajor_values(plan, sets):
    """(energies, per-job values) of one set-major evaluation of `sets`."""
    import torch

    b = plan.launch(torch.from_numpy(np.ascontiguousarray(sets)).cuda())
    torch.cuda.synchronize()
    return b["energy"].cpu().numpy().copy(), b["res"].cpu().numpy().copy()


@pytest.mark.parametrize("n_sets", [37, 1024, 1100])
def test_setmajor_c64_config2_vs_oracle(golden, setmajor_min_sets, n_sets):
    """complex64 set-major rows (config 2's dtype): every edge value within
    1e-5 (abs, |<ZZ>| <= 1) and every energy within 1e-5 relative of the
    complex128 executor; sampled sets against the oracle.  37 sets: odd count
    (padded row stride); 1024: the full-pass kernel; 1100: partial passes."""
    setmajor_min_sets(1)
    G = golden("config2.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    edges = [tuple(e) for e in G["edges"]]
    rng = np.random.default_rng(29)
    sets = rng.uniform(0, math.pi, (n_sets, 4))
    sets[0] = list(G["gammas"]) + list(G["betas"])
    p64 = Q.EnergyPlan(graph, 2, "zz+diagonal", dtype="complex64")
    p128 = Q.EnergyPlan(graph, 2, "zz+diagonal", dtype="complex128")
    p64._prepare()
    p128._prepare()
    assert p64._batch.setmajor_elem_bytes(n_sets) == 8
    assert p128._batch.setmajor_elem_bytes(n_sets) == 16
    e64, r64 = _setmajor_values(p64, sets)
    e128, r128 = _setmajor_values(p128, sets)
    assert np.abs(r64 - r128).max() < 1e-5
    assert np.all(np.abs(e64 - e128) <= 1e-5 * np.abs(e128))
    # set 0 = the config's seeded angles: the golden energy of the reference
    want = sum((1 - r["value"][0]) / 2 for r in G["modes"]["zz+diagonal"])
    assert abs(e64[0] - want) / abs(want) < 1e-5
    for s in (1, n_sets - 1):
        g, b = list(sets[s, :2]), list(sets[s, 2:])
        zz = [O.edge_zz(100, edges, edges[e], g, b, "zz+diagonal") for e in range(0, 150, 10)]
        got = [r64[s, p64.jobs.index(next(j for j in p64.jobs if j.index == e))]
               for e in range(0, 150, 10)]
        assert np.abs(np.asarray(got) - np.asarray(zz)).max() < 1e-5
    # the public host-to-host call (captured graph) gives the same energies
    assert np.allclose(p64.energies(sets), e64, rtol=0, atol=1e-9)


def test_setmajor_c64_config3_zzdiag(golden, setmajor_min_sets):
    """Config 3 zz+diagonal (p=3, deeper networks) on complex64 set-major
    rows: energy at the seeded angles within 1e-5 of the reference golden,
    all 256 sets within 1e-5 relative of the complex128 rows."""
    setmajor_min_sets(1)
    G = golden("config3.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    rng = np.random.default_rng(31)
    sets = rng.uniform(0, math.pi, (256, 6))
    sets[0] = list(G["gammas"]) + list(G["betas"])
    p64 = Q.EnergyPlan(graph, 3, "zz+diagonal", dtype="complex64")
    p128 = Q.EnergyPlan(graph, 3, "zz+diagonal", dtype="complex128")
    p64._prepare()
    assert p64._batch.setmajor_elem_bytes(256) == 8
    e64, r64 = _setmajor_values(p64, sets)
    e128, r128 = _setmajor_values(p128, sets)
    assert np.abs(r64 - r128).max() < 1e-5
    assert np.all(np.abs(e64 - e128) <= 1e-5 * np.abs(e128))
    want = sum((1 - r["value"][0]) / 2 for r in G["modes"]["zz+diagonal"])
    assert abs(e64[0] - want) / abs(want) < 1e-5
    assert abs(e128[0] - want) / abs(want) < 1e-10


# ------------------------------------------------- expanding-bucket kernel
@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-11), ("complex64", 1e-5)])
def test_expand_kernel_config4(golden, monkeypatch, dtype, tol):
    """Config 4 edges #16 and #1058 (expanding buckets [2,17,17]->25,
    [1,22,21]->26, ...) on the outer-product kernel equal the streaming
    kernel (QTN_EXPAND=0) and the reference values; one angle set and a
    batch of 3 (grid.y over sets)."""
    G = golden("config4.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    ids = [16, 1058]
    recs = {r["edge_index"]: complex(*r["value"]) for r in G["modes"]["zz+diagonal"]
            if r["edge_index"] in ids}
    rng = np.random.default_rng(41)
    sets = rng.uniform(0, math.pi, (3, 2 * G["p"]))
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("QTN_EXPAND", flag)
        plan = Q.EnergyPlan(graph, G["p"], "zz+diagonal", dtype=dtype, edge_ids=ids)
        out[flag] = (plan.zz_values(params), plan.energies(sets))
        assert plan.launches == plan.launches_per_eval(3)
    for e in ids:
        assert abs(out["1"][0][e] - recs[e]) <= tol * abs(recs[e])
        assert abs(out["1"][0][e] - out["0"][0][e]) <= tol * abs(recs[e])
    assert np.allclose(out["1"][1], out["0"][1], rtol=tol, atol=0)


def test_expand_kernel_config3_default(golden, monkeypatch):
    """Config 3 default-mode networks (H/CNOT, 2-operand buckets): the
    outer-product kernel wherever it applies equals the streaming kernel and
    the reference values (complex128)."""
    G = golden("config3.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    recs = G["modes"]["default"][:12]
    ids = [r["edge_index"] for r in recs]
    vals = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("QTN_EXPAND", flag)
        monkeypatch.setenv("QTN_EXPAND_MIN_R", "12")
        plan = Q.EnergyPlan(graph, G["p"], "default", dtype="complex128", edge_ids=ids)
        vals[flag] = plan.zz_values(params)
    for r in recs:
        w = complex(*r["value"])
        assert abs(vals["1"][r["edge_index"]] - w) <= 1e-11 * abs(w) + 1e-13
        assert abs(vals["1"][r["edge_index"]] - vals["0"][r["edge_index"]]) <= 1e-11 * abs(w) + 1e-13


def test_chain_kernel_opt_in(golden, monkeypatch):
    """Tiny-level chains in one cluster launch (QTN_CHAIN=1, cluster barriers
    between levels) equal the per-level small_kernel launches (config 4 edge
    #16 and config 3 default networks, complex128), with fewer launches."""
    monkeypatch.setenv("QTN_SUBTREE", "0")  # tiny levels must exist for the chains
    G4 = golden("config4.json")
    g4 = Q.random_regular_graph(G4["n"], 3, 0)
    p4 = Q.QaoaParams(G4["gammas"], G4["betas"])
    G3 = golden("config3.json")
    g3 = Q.random_regular_graph(G3["n"], 3, 0)
    p3 = Q.QaoaParams(G3["gammas"], G3["betas"])
    ids3 = [r["edge_index"] for r in G3["modes"]["default"][:10]]
    monkeypatch.setenv("QTN_TINY_LEVEL", str(1 << 17))  # tiny levels exist
    monkeypatch.setenv("QTN_SMALL_R", "9")
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("QTN_CHAIN", flag)
        a = Q.EnergyPlan(g4, G4["p"], "zz+diagonal", dtype="complex128", edge_ids=[16])
        b = Q.EnergyPlan(g3, G3["p"], "default", dtype="complex128", edge_ids=ids3)
        out[flag] = (a.zz_values(p4)[16], b.zz_values(p3), a.launches_per_eval(1))
    assert abs(out["1"][0] - out["0"][0]) <= 1e-12 * abs(out["0"][0])
    for e in ids3:
        assert abs(out["1"][1][e] - out["0"][1][e]) <= 1e-12 * abs(out["0"][1][e]) + 1e-14
    assert out["1"][2] < out["0"][2]


@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-12), ("complex64", 1e-6)])
def test_trace_kernel_matches_stream_kernel(golden, monkeypatch, dtype, tol):
    """Single-operand buckets (partial traces, 59 % of config 3 default's
    bytes) on trace_kernel equal the streaming kernel (QTN_TRACE=0) and the
    reference values; config 3 default networks and config 4 edge #16."""
    G3 = golden("config3.json")
    g3 = Q.random_regular_graph(G3["n"], 3, 0)
    p3 = Q.QaoaParams(G3["gammas"], G3["betas"])
    recs = G3["modes"]["default"][:10]
    ids3 = [r["edge_index"] for r in recs]
    G4 = golden("config4.json")
    g4 = Q.random_regular_graph(G4["n"], 3, 0)
    p4 = Q.QaoaParams(G4["gammas"], G4["betas"])
    w4 = complex(*[r for r in G4["modes"]["zz+diagonal"] if r["edge_index"] == 16][0]["value"])
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("QTN_TRACE", flag)
        a = Q.EnergyPlan(g3, G3["p"], "default", dtype=dtype, edge_ids=ids3)
        b = Q.EnergyPlan(g4, G4["p"], "zz+diagonal", dtype=dtype, edge_ids=[16])
        out[flag] = (a.zz_values(p3), b.zz_values(p4)[16])
        assert a.launches == a.launches_per_eval(1)
    ref_tol = 1e-11 if dtype == "complex128" else 1e-5
    for r in recs:
        w = complex(*r["value"])
        e = r["edge_index"]
        assert abs(out["1"][0][e] - w) <= ref_tol * abs(w) + 1e-13
        assert abs(out["1"][0][e] - out["0"][0][e]) <= tol * abs(w) + 1e-13
    assert abs(out["1"][1] - w4) <= ref_tol * abs(w4)
    assert abs(out["1"][1] - out["0"][1]) <= tol * abs(w4)


@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-12), ("complex64", 1e-6)])
def test_trace_kernel_every_eligible_bucket(golden, monkeypatch, dtype, tol):
    """QTN_TRACE_MIN_MB=0 sends every eligible bucket to trace_kernel,
    including complex128 primaries/outputs and outputs wider than the
    primary (new bits from staged operands): same values as the streaming
    kernel and the reference (config 3 default networks)."""
    monkeypatch.setenv("QTN_TRACE_MIN_MB", "0")
    G3 = golden("config3.json")
    g3 = Q.random_regular_graph(G3["n"], 3, 0)
    p3 = Q.QaoaParams(G3["gammas"], G3["betas"])
    recs = G3["modes"]["default"][10:18]
    ids3 = [r["edge_index"] for r in recs]
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("QTN_TRACE", flag)
        a = Q.EnergyPlan(g3, G3["p"], "default", dtype=dtype, edge_ids=ids3)
        out[flag] = a.zz_values(p3)
    ref_tol = 1e-11 if dtype == "complex128" else 1e-5
    for r in recs:
        w = complex(*r["value"])
        e = r["edge_index"]
        assert abs(out["1"][e] - w) <= ref_tol * abs(w) + 1e-13
        assert abs(out["1"][e] - out["0"][e]) <= tol * abs(w) + 1e-13


@pytest.mark.parametrize("fwarp", ["1", "0"])
@pytest.mark.parametrize("min_r", ["0", "10"])
def test_fused_product_chains(golden, monkeypatch, min_r, fwarp):
    """Product buckets followed by their partial traces as one contraction
    (every chain here, whatever the default window): equal to the unfused
    bucket-by-bucket evaluation (QTN_FUSE_CHAIN=0) and to the reference
    values, on config 3 default (GEMM-shaped chains, dot-product chains into
    scalars) and config 4 edge #16 (wide streaming chains), complex128 and
    complex64, at 1 and 3 angle sets.  min_r 0 also fuses the tiny chains of
    the first levels.  fwarp 1: chains of output rank >= 5 on the
    warp-granular kernel (fusedw_kernel, qtn_fusedw.cu), the rest on the CTA
    kernel; 0: every chain on the CTA kernel (fused_kernel, qtn_fused.cu)."""
    monkeypatch.setenv("QTN_FWARP", fwarp)
    monkeypatch.setenv("QTN_FCHAIN_MIN_R", min_r)
    monkeypatch.setenv("QTN_FCHAIN_MIN_OUT", "0")   # every chain: dot products,
    monkeypatch.setenv("QTN_FCHAIN_MAX_OUT", "64")  # wide streaming chains too
    G = golden("config3.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    recs = G["modes"]["default"][:10]
    G4 = golden("config4.json")
    rec4 = complex(*[r for r in G4["modes"]["zz+diagonal"] if r["edge_index"] == 16][0]["value"])
    g4 = Q.random_regular_graph(G4["n"], 3, 0)
    p4v = Q.QaoaParams(G4["gammas"], G4["betas"])
    rng = np.random.default_rng(3)
    sets3 = np.vstack([params.as_vector(), rng.uniform(0, math.pi, (2, 2 * G["p"]))])
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("QTN_FUSE_CHAIN", flag)
        for dt in ("complex128", "complex64"):
            plan = Q.EnergyPlan(graph, G["p"], "default", dtype=dt,
                                edge_ids=[r["edge_index"] for r in recs])
            p4 = Q.EnergyPlan(g4, G4["p"], "zz+diagonal", dtype=dt, edge_ids=[16])
            nf = sum(j.plan.n_fused_chains for j in plan.jobs + p4.jobs)
            assert (nf > 0) == (flag == "1")
            out[flag, dt] = (plan.zz_values(params), p4.zz_values(p4v)[16], plan.energies(sets3))
            assert plan.launches == plan.launches_per_eval(1)
    for dt, tol in (("complex128", 1e-11), ("complex64", 1e-5)):
        for r in recs:
            w = complex(*r["value"])
            e = r["edge_index"]
            assert abs(out["1", dt][0][e] - w) <= tol * abs(w) + 1e-12, (dt, e)
            assert abs(out["1", dt][0][e] - out["0", dt][0][e]) <= tol * abs(w) + 1e-12
        assert abs(out["1", dt][1] - rec4) <= tol * abs(rec4)
        assert np.allclose(out["1", dt][2], out["0", dt][2], rtol=tol, atol=tol)


@pytest.mark.parametrize("min_r", ["14", "10"])
def test_expand_consumer_pairs(golden, monkeypatch, min_r):
    """An expanding bucket and its consumer as one pass (xt_kernel,
    qtn_xt.cu; contraction.py:90-96 twice without storing the union-size
    result): equal to the bucket-by-bucket evaluation (QTN_XT=0) and to the
    reference values, complex64 at 1e-5, on config 4 edges #16 and #1058 (the
    rank-25/26 pairs, with and without a staged consumer operand) and on
    config 3 default edges, at 1 and 3 angle sets.  min_r 10 also pairs the
    small expanding buckets (few tiles, h = 1..2)."""
    monkeypatch.setenv("QTN_XT_MIN_R", min_r)
    monkeypatch.setenv("QTN_EXPAND_MIN_R", min_r)
    G = golden("config3.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    recs = G["modes"]["default"][:12]
    G4 = golden("config4.json")
    rec4 = {r["edge_index"]: complex(*r["value"]) for r in G4["modes"]["zz+diagonal"]
            if r["edge_index"] in (16, 1058)}
    g4 = Q.random_regular_graph(G4["n"], 3, 0)
    p4v = Q.QaoaParams(G4["gammas"], G4["betas"])
    rng = np.random.default_rng(5)
    sets3 = np.vstack([params.as_vector(), rng.uniform(0, math.pi, (2, 2 * G["p"]))])
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("QTN_XT", flag)
        plan = Q.EnergyPlan(graph, G["p"], "default", dtype="complex64",
                            edge_ids=[r["edge_index"] for r in recs])
        p4 = Q.EnergyPlan(g4, G4["p"], "zz+diagonal", dtype="complex64", edge_ids=sorted(rec4))
        npairs = sum(j.plan.n_pairs for j in plan.jobs), sum(j.plan.n_pairs for j in p4.jobs)
        assert (npairs[0] > 0 and npairs[1] >= 4) if flag == "1" else npairs == (0, 0)
        out[flag] = (plan.zz_values(params), p4.zz_values(p4v), plan.energies(sets3))
        assert plan.launches == plan.launches_per_eval(1)
    tol = 1e-5
    for r in recs:
        w = complex(*r["value"])
        e = r["edge_index"]
        assert abs(out["1"][0][e] - w) <= tol * abs(w) + 1e-12, e
        assert abs(out["1"][0][e] - out["0"][0][e]) <= tol * abs(w) + 1e-12
    for e, w in rec4.items():
        assert abs(out["1"][1][e] - w) <= tol * abs(w), e
        assert abs(out["1"][1][e] - out["0"][1][e]) <= tol * abs(w), e
    assert np.allclose(out["1"][2], out["0"][2], rtol=tol, atol=tol)


def test_device_memory_fit_check():
    """an evaluation whose buffers exceed the free device memory
    raises MemoryError before allocating (config 4 edge #16 at 2^20 angle
    sets needs ~100 TB of arena)."""
    g4 = Q.random_regular_graph(1000, 3, 0)
    plan = Q.EnergyPlan(g4, 5, "zz+diagonal", dtype="complex64", edge_ids=[16])
    with pytest.raises(MemoryError):
        plan.energies(np.zeros((1 << 20, 10)))
    # and a normal call still works afterwards
    z = plan.energies(np.zeros((1, 10)))
    assert np.isfinite(z).all()


def test_repeatable_bitwise_results():
    """Every kernel path is deterministic (fixed reduction orders, no atomics
    on data): repeated evaluations of HBM-executor networks (config 3 default
    edges 0-7: small, stream, trace, expand, reduce and fused-chain kernels
    with split-K; config 4 edge #16) and of the set-major executor give
    bit-identical energies — a data race in a cp.async / mbarrier pipeline
    would show up as run-to-run differences.  (compute-sanitizer is not
    available on the build's GPU pool.)"""
    import os

    os.environ["QTN_GRAPHS"] = "0"
    try:
        g3 = Q.random_regular_graph(244, 3, 0)
        p3 = Q.EnergyPlan(g3, 3, "default", dtype="complex64", edge_ids=list(range(8)))
        g4 = Q.random_regular_graph(1000, 3, 0)
        p4 = Q.EnergyPlan(g4, 5, "zz+diagonal", dtype="complex64", edge_ids=[16])
        g2 = Q.random_regular_graph(100, 3, 0)
        p2 = Q.EnergyPlan(g2, 2, "zz+diagonal", dtype="complex64")
        rng = np.random.default_rng(11)
        a3, a4, a2 = (rng.uniform(0, math.pi, (2, 6)), rng.uniform(0, math.pi, (1, 10)),
                      rng.uniform(0, math.pi, (256, 4)))
        ref = (p3.energies(a3), p4.energies(a4), p2.energies(a2))
        for _ in range(4):
            got = (p3.energies(a3), p4.energies(a4), p2.energies(a2))
            for x, y in zip(got, ref):
                assert np.array_equal(x, y)
    finally:
        del os.environ["QTN_GRAPHS"]


@pytest.mark.parametrize("sub_r", ["9", "12"])
def test_tiny_subtrees(golden, monkeypatch, sub_r):
    """Tiny subtrees (subtree_kernel: a connected set of small buckets
    evaluated by one CTA with its intermediates in shared memory): equal to
    the level-by-level buckets (QTN_SUBTREE=0) and to the reference on
    config 3 default (10 edges) and config 4 edge #16, complex128 and
    complex64; QTN_SUBTREE_R=12 also takes larger buckets."""
    monkeypatch.setenv("QTN_SUBTREE_R", sub_r)
    G = golden("config3.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    recs = G["modes"]["default"][:10]
    G4 = golden("config4.json")
    rec4 = complex(*[r for r in G4["modes"]["zz+diagonal"] if r["edge_index"] == 16][0]["value"])
    g4 = Q.random_regular_graph(G4["n"], 3, 0)
    p4v = Q.QaoaParams(G4["gammas"], G4["betas"])
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("QTN_SUBTREE", flag)
        for dt in ("complex128", "complex64"):
            plan = Q.EnergyPlan(graph, G["p"], "default", dtype=dt,
                                edge_ids=[r["edge_index"] for r in recs])
            p4 = Q.EnergyPlan(g4, G4["p"], "zz+diagonal", dtype=dt, edge_ids=[16])
            out[flag, dt] = (plan.zz_values(params), p4.zz_values(p4v)[16])
            assert plan.launches == plan.launches_per_eval(1)
    for dt, tol in (("complex128", 1e-11), ("complex64", 1e-5)):
        for r in recs:
            w = complex(*r["value"])
            e = r["edge_index"]
            assert abs(out["1", dt][0][e] - w) <= tol * abs(w) + 1e-12, (dt, e)
            assert abs(out["1", dt][0][e] - out["0", dt][0][e]) <= tol * abs(w) + 1e-12
        assert abs(out["1", dt][1] - rec4) <= tol * abs(rec4)


def test_tail_chains(golden, monkeypatch):
    """Tail chains (wsum_kernel, DESIGN 3.9): the linear chain from the last
    wide intermediate to the scalar (contraction.py:90-96 once per remaining
    variable) as one weighted full sum.  Equal to the bucket-by-bucket
    evaluation (QTN_WSUM=0) and to the reference values at 1e-5 on config 4
    edges #16 / #1058 (unsliced and in 2^3 slices) and on config 3 default
    networks, for several angle sets; repeated evaluations are bitwise equal
    (fixed summation order)."""
    G = golden("config3.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    recs = G["modes"]["default"][:12]
    G4 = golden("config4.json")
    rec4 = {r["edge_index"]: complex(*r["value"]) for r in G4["modes"]["zz+diagonal"]
            if r["edge_index"] in (16, 1058)}
    g4 = Q.random_regular_graph(G4["n"], 3, 0)
    p4v = Q.QaoaParams(G4["gammas"], G4["betas"])
    rng = np.random.default_rng(7)
    sets3 = np.vstack([params.as_vector(), rng.uniform(0, math.pi, (2, 2 * G["p"]))])
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("QTN_WSUM", flag)
        plan = Q.EnergyPlan(graph, G["p"], "default", dtype="complex64",
                            edge_ids=[r["edge_index"] for r in recs])
        p4 = Q.EnergyPlan(g4, G4["p"], "zz+diagonal", dtype="complex64", edge_ids=sorted(rec4))
        p4s = Q.EnergyPlan(g4, G4["p"], "zz+diagonal", dtype="complex64", edge_ids=[1058], slice_k=3)
        nt = sum(j.plan.n_tails for j in plan.jobs), sum(j.plan.n_tails for j in p4.jobs), \
            sum(j.plan.n_tails for j in p4s.jobs)
        assert (nt[0] > 0 and nt[1] >= 1 and nt[2] >= 1) if flag == "1" else nt == (0, 0, 0)
        out[flag] = (plan.zz_values(params), p4.zz_values(p4v), plan.energies(sets3), p4s.zz_values(p4v))
        assert plan.launches == plan.launches_per_eval(1)
        again = p4.zz_values(p4v)
        assert all(again[e] == out[flag][1][e] for e in rec4)
    tol = 1e-5
    for r in recs:
        w = complex(*r["value"])
        e = r["edge_index"]
        assert abs(out["1"][0][e] - w) <= tol * abs(w) + 1e-12, e
        assert abs(out["1"][0][e] - out["0"][0][e]) <= tol * abs(w) + 1e-12
    for e, w in rec4.items():
        assert abs(out["1"][1][e] - w) <= tol * abs(w), e
        assert abs(out["1"][1][e] - out["0"][1][e]) <= tol * abs(w), e
    w = rec4[1058]
    assert abs(out["1"][3][1058] - w) <= tol * abs(w)
    assert np.allclose(out["1"][2], out["0"][2], rtol=tol, atol=tol)



