#!/usr/bin/env python
"""A small workload that launches every kernel family once, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

  config 1 energy on the warp-resident and the set-major executors,
  config 3 default edges 0..5 through the HBM executor (small, stream,
  trace, expand, reduce and fused-chain kernels, split-K combine),
  config 4 edge #16 (staged trace, expanding buckets, fused chains),
  one config-5-shaped bucket (w = 18) through qtn_bucket_contract.

usage: compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("QTN_GRAPHS", "0")  # direct launches: the tools see each kernel


def main():
    import numpy as np
    import torch

    import bench
    import paper_2106_15740_b200 as Q

    torch.cuda.set_device(0)
    g1 = Q.random_regular_graph(20, 3, 0)
    p1 = Q.EnergyPlan(g1, 1, "zz+diagonal", dtype="complex128")
    e1 = p1.energies(Q.seeded_angles(1, 0))
    e1m = p1.energies(np.tile(Q.seeded_angles(1, 0).as_vector(), (128, 1)))
    g3 = Q.random_regular_graph(244, 3, 0)
    p3 = Q.EnergyPlan(g3, 3, "default", dtype="complex64", edge_ids=list(range(6)))
    e3 = p3.energies(Q.seeded_angles(3, 0))
    g4 = Q.random_regular_graph(1000, 3, 0)
    p4 = Q.EnergyPlan(g4, 5, "zz+diagonal", dtype="complex64", edge_ids=[16])
    z4 = p4.zz_values(Q.seeded_angles(5, 0))[16]
    r5 = bench.config5_bucket(torch, w=18, m=8, reps=1)
    torch.cuda.synchronize()
    print(f"sanitize workload ok: E1={e1[0]:.12f} E1[128]={e1m[-1]:.12f} E3={e3[0]:.9f} "
          f"zz4={z4.real:.9f} c5={r5['parity']} err={r5['parity_max_rel_err']:.1e}")


if __name__ == "__main__":
    main()
