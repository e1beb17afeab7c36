#!/usr/bin/env python
"""GEMM census of the bucket-elimination programs (SURVEY §8(f) row 3,
VERDICT r01 "next" #8): which product buckets, fused with the single-operand
sums that follow them, form a dense (batched) GEMM, and what a tensor-core
path could save.

The symbolic loop is the reference's (contraction.py:75-106): bucket = the
live tensors holding v, in ascending id; the result gets a fresh id.  A
*chain* starts at a bucket of >= 2 operands whose result C is then consumed
only by single-operand buckets (partial traces, contraction.py:94-96) for
k more variables.  The chain computes

    out[O] = sum_{K} prod_t T_t[...]          K = {v, w_1..w_k}

Split the two largest operands A, B (the others are small gate tensors that
fold into either side): summed variables in both A and B form the GEMM's K
dimension, output variables in both form the batch, A-only / B-only output
variables form M / N.  Summed variables in only one side are pre-reductions
of that side (a bandwidth pass on a smaller tensor, not GEMM work).

For each chain the census reports batch, M, N, K and two projections:
  * today: the chain's algorithmic bytes (product bucket + every trace) at
    the HBM peak, i.e. the best the current bandwidth kernels can do;
  * GEMM: max(bytes of A + B + out at the HBM peak, flops at a tensor-core
    rate) with flops = 8 * batch * M * N * K (complex MAC); rates:
    3xTF32 ~ 370 TFLOP/s (complex64), DMMA FP64 ~ 37 TFLOP/s (complex128).
The saving is today - GEMM, summed per (M, N, K) class, as a share of the
whole evaluation's bytes at peak.

usage: python tools/gemm_census.py [config3-default|config4] [--edges a,b,..]
"""
import argparse
import collections
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

HBM = 6540.2e9
TC = {"complex64": 370e12, "complex128": 37e12}


def bucket_program(structure, order):
    """Symbolic reference bucket loop; yields (v, [(id, vars)], result vars)."""
    live = {}
    for i, vs in enumerate(structure):
        live[i] = tuple(vs)
    nxt = len(structure)
    prog = []
    for v in order:
        ids = sorted(i for i, vs in live.items() if v in vs)
        if not ids:
            prog.append((v, [], None, None))
            continue
        ops = [(i, live.pop(i)) for i in ids]
        union = []
        for _, vs in ops:
            for x in vs:
                if x not in union:
                    union.append(x)
        res = tuple(x for x in union if x != v)
        live[nxt] = res
        prog.append((v, ops, res, nxt))
        nxt += 1
    return prog


def chains(prog):
    """Product buckets followed by single-operand sums of their result."""
    consumer = {}
    for k, (v, ops, res, rid) in enumerate(prog):
        for i, _ in ops:
            consumer[i] = k
    out = []
    for k, (v, ops, res, rid) in enumerate(prog):
        if len(ops) < 2:
            continue
        summed = [v]
        bytes_chain = sum(2 ** len(vs) for _, vs in ops) + 2 ** len(res)
        cur, cid = res, rid
        while cid in consumer:
            k2 = consumer[cid]
            v2, ops2, res2, rid2 = prog[k2]
            if len(ops2) != 1:
                break
            summed.append(v2)
            bytes_chain += 2 ** len(cur) + 2 ** len(res2)
            cur, cid = res2, rid2
        ops_sorted = sorted(ops, key=lambda t: -len(t[1]))
        A, B = set(ops_sorted[0][1]), set(ops_sorted[1][1])
        for _, vs in ops_sorted[2:]:
            # small operands fold into the side they share most with
            (A if len(A & set(vs)) >= len(B & set(vs)) else B).update(vs)
        S = set(summed)
        O = set(cur)
        kk = len(S & A & B)
        bt = len(O & A & B)
        m = len(O & (A - B))
        n = len(O & (B - A))
        out.append({"batch": bt, "m": m, "n": n, "k": kk, "k_chain": len(summed) - 1,
                    "bytes_chain": bytes_chain,
                    "bytes_gemm": 2 ** len(ops_sorted[0][1]) + 2 ** len(ops_sorted[1][1]) +
                                  2 ** len(cur),
                    "ops": [len(vs) for _, vs in ops], "out_rank": len(cur)})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="config3-default")
    ap.add_argument("--edges", default=None)
    ap.add_argument("--dtype", default="complex64")
    a = ap.parse_args()
    import bench
    import paper_2106_15740_b200 as Q

    wl = dict(bench.WORKLOADS[a.workload])
    if a.edges:
        wl["edges"] = [int(x) for x in a.edges.split(",")]
    graph = Q.random_regular_graph(wl["n"], 3, 0)
    jobs = Q.plan_edges(graph, wl["p"], wl["mode"], bench.edge_ids_of(wl), compile_plans=False)
    e = 8 if a.dtype == "complex64" else 16
    total_bytes = 0.0
    cls = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    n_chain = 0
    for j in jobs:
        prog = bucket_program(j.template.structure, j.order.sequence)
        for v, ops, res, rid in prog:
            if ops:
                total_bytes += e * (sum(2 ** len(vs) for _, vs in ops) + 2 ** len(res))
        for c in chains(prog):
            n_chain += 1
            flops = 8.0 * 2 ** (c["batch"] + c["m"] + c["n"] + c["k"])
            t_now = e * c["bytes_chain"] / HBM
            t_gemm = max(e * c["bytes_gemm"] / HBM, flops / TC[a.dtype])
            key = (c["batch"], c["m"], c["n"], c["k"])
            d = cls[key]
            d[0] += 1
            d[1] += t_now
            d[2] += t_gemm
            d[3] += flops
    t_all = total_bytes / HBM
    print(f"{a.workload}: {len(jobs)} networks, {total_bytes / 1e9:.3f} GB algorithmic "
          f"({a.dtype}), {t_all * 1e3:.3f} ms at {HBM / 1e9:.0f} GB/s; {n_chain} product chains")
    print(f"{'log2 batch,M,N,K':>18s} {'chains':>7s} {'now us':>9s} {'gemm us':>9s} "
          f"{'save us':>9s} {'save %eval':>10s} {'TFLOP':>8s}")
    rows = sorted(cls.items(), key=lambda kv: -(kv[1][1] - kv[1][2]))
    save_gemm = 0.0
    for key, (cnt, tn, tg, fl) in rows[:25]:
        s = tn - tg
        print(f"{str(key):>18s} {cnt:7d} {tn * 1e6:9.1f} {tg * 1e6:9.1f} {s * 1e6:9.1f} "
              f"{100 * s / t_all:9.2f}% {fl / 1e12:8.4f}")
    for key, (cnt, tn, tg, fl) in rows:
        # a tensor-core path needs a real GEMM: M, N >= 16 and K >= 8 (tile shapes)
        if key[1] >= 4 and key[2] >= 4 and key[3] >= 3:
            save_gemm += tn - tg
    print(f"saving of the GEMM-shaped classes (M, N >= 16, K >= 8): {save_gemm * 1e6:.1f} us "
          f"= {100 * save_gemm / t_all:.2f}% of the evaluation at peak")


if __name__ == "__main__":
    main()
