"""Plan-compiler checks of the fused product chains (host only, no GPU):
which buckets fuse, what the fused descriptors cover, and that the
reference's invariants survive (step ranks = CostReport)."""

import paper_2106_15740_b200 as Q


def test_fused_chain_census_and_levels(golden):
    """Config 4 edge #1058: with every chain fused (QTN_FCHAIN_MAX_OUT=64)
    the product chains fuse (fewer levels, fewer bytes moved than the
    reference's per-bucket bytes); with QTN_FUSE_CHAIN=0
    none do; the width invariant holds either way."""
    import os

    G4 = golden("config4.json")
    g4 = Q.random_regular_graph(G4["n"], 3, 0)
    os.environ["QTN_FCHAIN_MAX_OUT"] = "64"  # every chain, wide streaming ones too
    os.environ["QTN_WSUM"] = "0"             # (the tail chain would take the last product chains)
    try:
        j = Q.plan_edges(g4, G4["p"], "zz+diagonal", [1058], dtype="complex64")[0]
    finally:
        del os.environ["QTN_FCHAIN_MAX_OUT"]
        del os.environ["QTN_WSUM"]
    assert j.plan.n_fused_chains >= 5
    assert j.plan.exec_bytes < 0.8 * j.plan.alg_bytes
    assert max(j.plan.step_ranks) == j.report.width
    os.environ["QTN_FUSE_CHAIN"] = "0"
    os.environ["QTN_WSUM"] = "0"
    try:
        k = Q.plan_edges(g4, G4["p"], "zz+diagonal", [1058], dtype="complex64")[0]
    finally:
        del os.environ["QTN_FUSE_CHAIN"]
        del os.environ["QTN_WSUM"]
    assert k.plan.n_fused_chains == 0
    assert k.plan.n_levels > j.plan.n_levels
    assert k.plan.alg_bytes == j.plan.alg_bytes
    assert k.plan.step_ranks == j.plan.step_ranks


def test_fused_chains_config3_default_every_network(golden):
    """Config 3 default networks compile with fused chains by default (the
    output-rank window 1..15); the deepest elimination tree gets shorter
    (70 levels unfused) and the executed bytes drop."""
    import os

    G = golden("config3.json")
    graph = Q.random_regular_graph(G["n"], 3, 0)
    jobs = Q.plan_edges(graph, G["p"], "default", range(0, 366, 3), dtype="complex64")  # default window
    assert sum(j.plan.n_fused_chains for j in jobs) > 100
    assert max(j.plan.n_levels for j in jobs) <= 55
    assert sum(j.plan.exec_bytes for j in jobs) < 0.8 * sum(j.plan.alg_bytes for j in jobs)


def test_expand_consumer_pairs_config4(golden):
    """Config 4 edge #1058: the three wide expanding buckets ([2,17,17]->25,
    [2,16,19]->25, [1,22,21]->26) pair with their consumers (xt_kernel), so
    the rank-25/26 results are never stored: executed bytes fall below half of
    the reference's per-bucket bytes; QTN_XT=0 keeps every bucket on its own
    kernel; complex128 plans have no pairs (float math only); step ranks and
    the algorithmic bytes are those of the reference either way."""
    import os

    G4 = golden("config4.json")
    g4 = Q.random_regular_graph(G4["n"], 3, 0)
    j = Q.plan_edges(g4, G4["p"], "zz+diagonal", [1058], dtype="complex64")[0]
    assert j.plan.n_pairs >= 3
    assert j.plan.exec_bytes < 0.5 * j.plan.alg_bytes
    assert max(j.plan.step_ranks) == j.report.width
    os.environ["QTN_XT"] = "0"
    try:
        k = Q.plan_edges(g4, G4["p"], "zz+diagonal", [1058], dtype="complex64")[0]
    finally:
        del os.environ["QTN_XT"]
    assert k.plan.n_pairs == 0
    assert k.plan.n_levels > j.plan.n_levels
    assert k.plan.exec_bytes > j.plan.exec_bytes
    assert k.plan.alg_bytes == j.plan.alg_bytes
    assert k.plan.step_ranks == j.plan.step_ranks
    d = Q.plan_edges(g4, G4["p"], "zz+diagonal", [16], dtype="complex128")[0]
    assert d.plan.n_pairs == 0


def test_tail_chain_config4(golden):
    """Config 4 edge #1058: after the last wide chain the elimination order is
    a linear chain from a rank-22 intermediate to the scalar (22 buckets whose
    other operands are rank-1/2 gates): one weighted full sum (wsum_kernel),
    so the tail's levels and intermediates disappear; QTN_WSUM=0 keeps them;
    complex128 plans have no tail chain (their intermediates are complex128);
    step ranks and algorithmic bytes are the reference's either way."""
    import os

    G4 = golden("config4.json")
    g4 = Q.random_regular_graph(G4["n"], 3, 0)
    j = Q.plan_edges(g4, G4["p"], "zz+diagonal", [1058], dtype="complex64")[0]
    assert j.plan.n_tails == 1
    assert max(j.plan.step_ranks) == j.report.width
    os.environ["QTN_WSUM"] = "0"
    try:
        k = Q.plan_edges(g4, G4["p"], "zz+diagonal", [1058], dtype="complex64")[0]
    finally:
        del os.environ["QTN_WSUM"]
    assert k.plan.n_tails == 0
    assert k.plan.n_levels >= j.plan.n_levels + 10
    assert k.plan.exec_bytes > j.plan.exec_bytes
    assert k.plan.alg_bytes == j.plan.alg_bytes
    assert k.plan.step_ranks == j.plan.step_ranks
    d = Q.plan_edges(g4, G4["p"], "zz+diagonal", [16], dtype="complex128")[0]
    assert d.plan.n_tails == 0
