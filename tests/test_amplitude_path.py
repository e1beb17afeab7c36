"""Amplitude path front end: text formats, ZZ fusion,
the CLI and the run_benchmark sweep, against outputs of the real reference
(tests/golden/amplitude_path.json, made by tests/golden/make_golden.py)."""

import contextlib
import io

import pytest

import paper_2106_15740_b200 as Q
from paper_2106_15740_b200.cli import main as cli_main


@pytest.fixture(scope="module")
def amp(golden):
    return golden("amplitude_path.json")


def _gates(c):
    return [[g.kind.value, list(g.qubits), g.param] for g in c.gates]


def _run_cli(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = cli_main(argv)
    return rc, out.getvalue().splitlines(), err.getvalue()


def test_text_formats_match_reference(amp, tmp_path):
    for rec in amp["circuits"]:
        graph = Q.random_regular_graph(rec["n"], 3, 0)
        raw = Q.build_qaoa_maxcut_circuit(graph, Q.default_angles(rec["p"]), fused=False)
        gp, cp = tmp_path / "g.txt", tmp_path / "c.txt"
        Q.write_graph(graph, gp)
        Q.write_circuit(raw, cp)
        assert gp.read_text() == rec["graph_text"]
        assert cp.read_text() == rec["circuit_text"]
        # the reference's files read back into identical objects
        (tmp_path / "rg.txt").write_text(rec["graph_text"])
        (tmp_path / "rc.txt").write_text(rec["circuit_text"])
        assert Q.read_graph(tmp_path / "rg.txt") == graph
        assert _gates(Q.read_circuit(tmp_path / "rc.txt")) == rec["raw_gates"]


def test_fuse_zz_matches_reference(amp):
    for rec in amp["circuits"]:
        graph = Q.random_regular_graph(rec["n"], 3, 0)
        raw = Q.build_qaoa_maxcut_circuit(graph, Q.default_angles(rec["p"]), fused=False)
        fused = Q.fuse_zz(raw)
        assert _gates(fused) == rec["fused_gates"]
        assert abs(fused.phase - complex(*rec["fused_phase"])) < 1e-15
        # idempotent, and equal to the directly-built fused ansatz
        assert _gates(Q.fuse_zz(fused)) == rec["fused_gates"]
        direct = Q.build_qaoa_maxcut_circuit(graph, Q.default_angles(rec["p"]), fused=True)
        assert _gates(direct) == rec["fused_gates"]


def test_parse_errors(tmp_path):
    bad = tmp_path / "bad.txt"
    for text in ("qubits 2\nH 5\n", "qubits 2\nFOO 0\n", "qubits x\n", "", "qubits 2\nZZ 0 1\n"):
        bad.write_text(text)
        with pytest.raises(Q.ParseError):
            Q.read_circuit(bad)
    for text in ("3 1\n0 1\n1 2\n", "3\n", "2 1\n0 0\n"):
        bad.write_text(text)
        with pytest.raises(Q.ParseError):
            Q.read_graph(bad)
    bad.write_text("n = 4\np = 1\n")
    with pytest.raises(Q.ParseError):
        Q.parse_bench_spec(bad)
    bad.write_text("n = 5\np = 1\nseeds = 0\n")  # infeasible regular graph
    with pytest.raises(Q.ParseError):
        Q.parse_bench_spec(bad)


def test_cli_cost_and_errors(amp, tmp_path):
    for rec in amp["circuits"]:
        cp = tmp_path / f"c{rec['n']}.txt"
        cp.write_text(rec["circuit_text"])
    for want in amp["cli"]:
        if want["cmd"] != "cost":
            continue
        rc, lines, _ = _run_cli(["cost", "--circuit", str(tmp_path / f"c{want['n']}.txt"),
                                 "--mode", want["mode"]])
        assert rc == want["rc"] == 0
        assert [l for l in lines if not l.startswith("order_seconds")] == want["stdout"]
    # exit codes: malformed file -> 1; bad flag -> 1; rank cap -> 2 (raised
    # at plan time, before any device work)
    (tmp_path / "bad.txt").write_text("qubits 2\nNOPE 0\n")
    assert _run_cli(["amplitude", "--circuit", str(tmp_path / "bad.txt")])[0] == 1
    with pytest.raises(SystemExit) as ei:
        _run_cli(["amplitude"])
    assert ei.value.code == 1
    rc, _, err = _run_cli(["amplitude", "--circuit", str(tmp_path / "c8.txt"), "--rank-cap", "2"])
    assert rc == 2 and "infeasible" in err


def test_cli_gen_graph_and_circuit(tmp_path):
    g = tmp_path / "g.txt"
    c = tmp_path / "c.txt"
    assert _run_cli(["gen-graph", "--n", "6", "--d", "3", "--seed", "1", "-o", str(g)])[0] == 0
    assert Q.read_graph(g) == Q.random_regular_graph(6, 3, 1)
    assert _run_cli(["circuit", "--graph", str(g), "--p", "2", "--fused", "-o", str(c)])[0] == 0
    want = Q.build_qaoa_maxcut_circuit(Q.random_regular_graph(6, 3, 1), Q.default_angles(2), fused=True)
    got = Q.read_circuit(c)
    assert _gates(got) == _gates(want) and abs(got.phase - want.phase) < 1e-15
    assert _run_cli(["circuit", "--graph", str(g), "--p", "2", "--gamma", "0.1", "-o", str(c)])[0] == 1


@pytest.mark.gpu
def test_cli_amplitude_on_gpu(amp, tmp_path):
    for rec in amp["circuits"]:
        (tmp_path / f"c{rec['n']}.txt").write_text(rec["circuit_text"])
    for want in amp["cli"]:
        if want["cmd"] != "amplitude":
            continue
        rc, lines, _ = _run_cli(["amplitude", "--circuit", str(tmp_path / f"c{want['n']}.txt"),
                                 "--mode", want["mode"]])
        assert rc == 0
        assert lines[:2] == want["stdout"][:2]  # bits, width
        got = complex(*map(float, lines[2].split()[1:]))
        ref = complex(*map(float, want["stdout"][2].split()[1:]))
        assert abs(got - ref) < 1e-12, (want["n"], want["mode"], got, ref)


@pytest.mark.gpu
def test_run_benchmark_on_gpu(amp, tmp_path):
    spec = Q.BenchSpec(ns=(4, 6), ps=(1, 2), seeds=(0, 1), contract=True)
    rows = Q.run_benchmark(spec)
    assert len(rows) == len(amp["bench"])
    for r, w in zip(rows, amp["bench"]):
        assert (r.graph_seed, r.n, r.p, r.mode) == (w["graph_seed"], w["n"], w["p"], w["mode"])
        assert r.width == w["width"] and r.memory_bytes == w["memory_bytes"]
        assert r.contracted and w["contracted"]
        assert abs(complex(r.amp_re, r.amp_im) - complex(*w["amp"])) < 1e-12
        assert r.contract_seconds is not None and r.contract_seconds > 0
    out = tmp_path / "rows.csv"
    Q.sweep.write_csv(rows, out)
    lines = out.read_text().splitlines()
    assert lines[0] == ",".join(Q.sweep.CSV_HEADER) and len(lines) == len(rows) + 1
