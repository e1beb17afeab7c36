"""Amplitude sweep through the B200 backend — the reference's run_benchmark.

Mirrors /root/reference/pkg/src/qtnsim/bench.py:80-270 for the part on the
contraction path: the sweep spec (`BenchSpec`,
`parse_bench_spec`), one `BenchRow` per (graph seed, n, p, mode) cell in the
reference's order, the ordering time, the CostReport figures and — when the
spec asks for it and the width fits the rank cap — the all-zeros amplitude of
`build_network(graph, p, mode, default_angles)` contracted on the GPU, with
its wall time in `contract_seconds`.  The CSV columns are the reference's
(bench.py:141-157).  The summary/plot stage of the reference harness is not
on the path and is not mirrored.
"""

from __future__ import annotations

import io
import time
from dataclasses import dataclass

from .contraction import DEFAULT_RANK_CAP, RankCapExceeded, contract
from .network import line_graph
from .ordering import rgreedy_order
from .pipeline import MODE_ORDER, build_network, default_angles, get_mode, random_regular_graph
from .textio import ParseError

__all__ = ["BenchSpec", "BenchRow", "CSV_HEADER", "parse_bench_spec", "run_benchmark",
           "rows_to_csv", "write_csv"]


@dataclass(frozen=True)
class BenchSpec:
    """Cross product of graph seeds, sizes, depths and modes (bench.py:80-104)."""

    ns: tuple
    ps: tuple
    seeds: tuple
    modes: tuple = MODE_ORDER
    degree: int = 3
    n_repeats: int = 10
    temp: float = 0.02
    order_seed: int = 0
    contract: bool = False
    rank_cap: int = DEFAULT_RANK_CAP

    def __post_init__(self):
        for m in self.modes:
            get_mode(m)
        for n in self.ns:
            if (n * self.degree) % 2 or self.degree >= n:
                raise ValueError(f"infeasible regular graph: n={n}, d={self.degree}")


_LISTS = {"n": "ns", "p": "ps", "seeds": "seeds"}
_INTS = {"d": "degree", "n_repeats": "n_repeats", "order_seed": "order_seed",
         "rank_cap": "rank_cap"}


def parse_bench_spec(path) -> BenchSpec:
    """key = value lines (comma-separated lists), '#' comments (bench.py:107-138)."""
    vals = {}
    with open(path, "r", encoding="utf-8") as fh:
        raw = fh.readlines()
    for no, text in enumerate(raw, start=1):
        body = text.split("#", 1)[0].strip()
        if not body:
            continue
        if "=" not in body:
            raise ParseError(path, no, f"expected 'key = value', got {body!r}")
        key, _, val = body.partition("=")
        key, val = key.strip().lower(), val.strip()
        try:
            if key in _LISTS:
                vals[_LISTS[key]] = tuple(int(x) for x in val.split(","))
            elif key in _INTS:
                vals[_INTS[key]] = int(val)
            elif key == "temp":
                vals["temp"] = float(val)
            elif key == "modes":
                vals["modes"] = tuple(m.strip() for m in val.split(","))
            elif key == "contract":
                if val.lower() not in ("true", "false"):
                    raise ValueError(f"expected true/false, got {val!r}")
                vals["contract"] = val.lower() == "true"
            else:
                raise ValueError(f"unknown key {key!r}")
        except ValueError as exc:
            raise ParseError(path, no, str(exc)) from None
    for req in ("ns", "ps", "seeds"):
        if req not in vals:
            raise ParseError(path, len(raw) or 1, f"missing required key {req!r}")
    try:
        return BenchSpec(**vals)
    except ValueError as exc:
        raise ParseError(path, len(raw) or 1, str(exc)) from None


CSV_HEADER = ("graph_seed", "n", "degree", "p", "mode", "n_repeats", "temp", "order_seconds",
              "width", "log2_flops_2c", "memory_bytes", "contracted", "amp_re", "amp_im",
              "contract_seconds")


@dataclass
class BenchRow:
    graph_seed: int
    n: int
    degree: int
    p: int
    mode: str
    n_repeats: int
    temp: float
    order_seconds: float
    width: int
    log2_flops_2c: int
    memory_bytes: float
    contracted: bool
    amp_re: float | None = None
    amp_im: float | None = None
    contract_seconds: float | None = None

    def to_csv_fields(self) -> tuple:
        opt = lambda x, f: "" if x is None else f(x)
        return (str(self.graph_seed), str(self.n), str(self.degree), str(self.p), self.mode,
                str(self.n_repeats), repr(self.temp), f"{self.order_seconds:.6f}",
                str(self.width), str(self.log2_flops_2c), f"{self.memory_bytes:.0f}",
                "true" if self.contracted else "false", opt(self.amp_re, repr),
                opt(self.amp_im, repr), opt(self.contract_seconds, lambda v: f"{v:.6f}"))


def _mode_key(m: str) -> int:
    return MODE_ORDER.index(m) if m in MODE_ORDER else len(MODE_ORDER)


def run_benchmark(spec: BenchSpec, dtype="complex128") -> list:
    """One row per (seed, n, p, mode) cell, in the reference's nesting order
    (bench.py:209-256); contraction on the B200 backend when spec.contract
    and the width fits the rank cap.  A cell whose contraction still exceeds
    the cap is recorded with contracted=false, as in the reference."""
    rows = []
    for seed in spec.seeds:
        for n in spec.ns:
            graph = random_regular_graph(n, spec.degree, seed)
            for p in sorted(spec.ps):
                for name in sorted(spec.modes, key=_mode_key):
                    mode = get_mode(name)
                    network = build_network(graph, p, mode, default_angles)
                    lg = line_graph(network)
                    t0 = time.perf_counter()
                    order, rep = rgreedy_order(lg, n_repeats=spec.n_repeats, temp=spec.temp,
                                               seed=spec.order_seed)
                    row = BenchRow(seed, n, spec.degree, p, mode.name, spec.n_repeats, spec.temp,
                                   time.perf_counter() - t0, rep.width, rep.width,
                                   rep.memory_bytes, False)
                    if spec.contract and rep.width <= spec.rank_cap:
                        t0 = time.perf_counter()
                        try:
                            amp = contract(network, order, rank_cap=spec.rank_cap, dtype=dtype)
                        except RankCapExceeded:
                            amp = None
                        if amp is not None:
                            row.contract_seconds = time.perf_counter() - t0
                            row.contracted = True
                            row.amp_re, row.amp_im = amp.real, amp.imag
                    rows.append(row)
    return rows


def rows_to_csv(rows) -> str:
    buf = io.StringIO()
    buf.write(",".join(CSV_HEADER) + "\n")
    for r in rows:
        buf.write(",".join(r.to_csv_fields()) + "\n")
    return buf.getvalue()


def write_csv(rows, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(rows_to_csv(rows))
