"""Pin the CPU oracle (oracle/qtn_oracle.py) to the golden vectors produced
by the real reference (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import qtn_oracle as O


def test_graph_generator_matches_reference(golden):
    for name in ("config1.json", "config2.json", "config3.json", "config4.json"):
        G = golden(name)
        assert [list(e) for e in O.random_regular_graph(G["n"], 3, 0)] == G["edges"]


def test_seeded_angles(golden):
    G = golden("config2.json")
    g, b = O.seeded_angles(G["p"], 0)
    assert g == G["gammas"] and b == G["betas"]


@pytest.mark.parametrize("mode", ["default", "diagonal", "zz", "zz+diagonal"])
def test_config1_networks_orders_values(golden, mode):
    G = golden("config1.json")
    edges = [tuple(e) for e in G["edges"]]
    for r in G["modes"][mode]:
        tens, nv, fixed = O.edge_network(G["n"], edges, edges[r["edge_index"]], G["gammas"],
                                         G["betas"], mode)
        assert nv == r["n_vars"] and len(tens) == r["n_tensors"]
        assert [list(vs) for vs, _ in tens] == r["structure"]
        assert sorted([k, v] for k, v in fixed.items()) == r["fixed"]
        verts = [v for v in range(nv) if v not in fixed]
        order, ranks = O.rgreedy(verts, O.hyperedges(tens, fixed))
        assert order == r["order"]
        assert max(ranks) == r["width"]
        val, sr = O.contract(tens, nv, fixed, order)
        assert abs(val - complex(*r["value"])) < 1e-13
        assert sr == ranks  # SPEC.md:311 peak-rank invariant


def test_config1_statevector_energy(golden):
    G = golden("config1.json")
    kat = golden("kat.json")
    edges = [tuple(e) for e in G["edges"]]
    gates, ph = O.qaoa_gates(20, edges, G["gammas"], G["betas"], True)
    psi = O.statevector(20, gates, ph)
    zz = [O.zz_from_state(psi, i, j) for i, j in edges]
    assert np.allclose(zz, kat["config1_statevector_zz"], atol=1e-12)
    # per-edge cone values equal the full-circuit statevector values
    for r in G["modes"]["zz+diagonal"]:
        assert abs(r["value"][0] - zz[r["edge_index"]]) < 1e-12


def test_config2_values_and_orders(golden):
    G = golden("config2.json")
    edges = [tuple(e) for e in G["edges"]]
    for r in G["modes"]["zz+diagonal"][::7]:
        tens, nv, fixed = O.edge_network(G["n"], edges, edges[r["edge_index"]], G["gammas"],
                                         G["betas"], "zz+diagonal")
        verts = [v for v in range(nv) if v not in fixed]
        order, ranks = O.rgreedy(verts, O.hyperedges(tens, fixed))
        assert order == r["order"]
        val, _ = O.contract(tens, nv, fixed, order)
        assert abs(val - complex(*r["value"])) < 1e-12


def test_kats(golden):
    kat = golden("kat.json")
    # N=2, p=1, gamma=0.4, beta=0.7 frozen regression constant
    gates, ph = O.qaoa_gates(2, [(0, 1)], [0.4], [0.7], True)
    psi = O.statevector(2, gates, ph)
    assert abs(psi[0, 0] - complex(*kat["n2_p1_g0.4_b0.7"])) < 1e-15
    # p=0, N=4 -> 0.25
    gates, ph = O.qaoa_gates(4, [], [], [], False)
    assert abs(O.statevector(4, gates, ph)[0, 0, 0, 0] - kat["p0_n4"]) < 1e-15


def test_synthetic_bucket_ops(golden):
    for case in golden("synthetic_buckets.json"):
        ops = [(tuple(o["vars"]),
                (np.asarray(o["re"]) + 1j * np.asarray(o["im"])).reshape((2,) * len(o["vars"])))
               for o in case["operands"]]
        vs, out = O.bucket_eliminate(ops, 0)
        assert list(vs) == case["out_vars"]
        want = np.asarray(case["out_re"]) + 1j * np.asarray(case["out_im"])
        assert np.allclose(out.reshape(-1), want, rtol=0, atol=1e-12)


def test_direct_sum_agrees_with_contract(golden):
    G = golden("config1.json")
    edges = [tuple(e) for e in G["edges"]]
    for r in G["modes"]["zz+diagonal"][:5]:
        tens, nv, fixed = O.edge_network(G["n"], edges, edges[r["edge_index"]], G["gammas"],
                                         G["betas"], "zz+diagonal")
        assert abs(O.direct_sum(tens, nv, fixed) - complex(*r["value"])) < 1e-12


def test_rank_cap_and_permutation_errors():
    tens = [((0, 1), np.ones((2, 2), complex)), ((1, 2), np.ones((2, 2), complex))]
    with pytest.raises(ValueError):
        O.contract(tens, 3, {}, [0, 1])
    with pytest.raises(O.RankCap) as ei:
        O.contract(tens, 3, {}, [1, 0, 2], rank_cap=1)
    assert ei.value.rank == 2
