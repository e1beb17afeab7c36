"""Amplitude path: the reference's own workload,
`build_network` (pipeline.py:70-81) -> `rgreedy_order` -> `contract`,
through the B200 backend, against outputs of the real reference
(tests/golden/amplitude_path.json, made by tests/golden/make_golden.py from
`qtnsim.bench.run_benchmark` rows and `qtnsim amplitude` output).

The reference's text formats, ZZ-fusion pass, sweep/CSV harness and CLI are
out of scope; only the contraction they call is replaced."""

import pytest

import paper_2106_15740_b200 as Q


@pytest.fixture(scope="module")
def amp(golden):
    return golden("amplitude_path.json")


def _cases(amp):
    """(graph seed, n, p, mode, golden width, golden amplitude) per record:
    run_benchmark rows (bench.py:209-256) and `amplitude` CLI lines for the
    default-angle circuits (cli.py:105-116; the CLI fuses the raw circuit,
    which yields the directly built fused ansatz, circuit.py:236-245)."""
    out = []
    for r in amp["bench"]:
        out.append((r["graph_seed"], r["n"], r["p"], r["mode"], r["width"], complex(*r["amp"])))
    for r in amp["cli"]:
        if r["cmd"] != "amplitude":
            continue
        width = int(r["stdout"][1].split()[-1])
        val = complex(*map(float, r["stdout"][2].split()[1:]))
        out.append((0, r["n"], r["p"], r["mode"], width, val))
    return out


def test_amplitude_widths_match_reference(amp):
    """Host side only: network build + reference rgreedy give the reference's
    widths (CostReport.width, ordering.py:46-68)."""
    for seed, n, p, mode, width, _ in _cases(amp):
        net = Q.build_network(Q.random_regular_graph(n, 3, seed), p, mode)
        _, rep = Q.rgreedy_order(Q.line_graph(net))
        assert rep.width == width, (seed, n, p, mode)


def test_amplitude_rank_cap_before_device_work(amp):
    """RankCapExceeded is raised at plan time, before any allocation
    (contraction.py:85-87) — no GPU needed."""
    net = Q.build_network(Q.random_regular_graph(8, 3, 0), 1, "default")
    order, rep = Q.rgreedy_order(Q.line_graph(net))
    sl = Q.sliced_tensors(net)
    with pytest.raises(Q.RankCapExceeded) as ei:
        Q.ContractionPlan([t.variables for t in sl], net.variable_count, net.fixed,
                          order.sequence, rank_cap=rep.width - 1)
    assert ei.value.rank == rep.width and ei.value.cap == rep.width - 1


@pytest.mark.gpu
def test_amplitude_path_on_gpu(amp):
    for seed, n, p, mode, width, want in _cases(amp):
        net = Q.build_network(Q.random_regular_graph(n, 3, seed), p, mode)
        order, rep = Q.rgreedy_order(Q.line_graph(net))
        got = Q.contract(net, order)
        assert abs(got - want) < 1e-12, (seed, n, p, mode, got, want)
