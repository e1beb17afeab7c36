"""World-size-2 gloo test of the multi-rank host path: LPT edge sharding
(energy.rank_shard) + one all_reduce of partial energies
(energy.reduce_partials).  Per-edge values come from the CPU oracle here;
on GPUs the same functions wrap EnergyPlan and NCCL."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, golden_path, out_q):
    import json
    import sys

    import numpy as np
    import torch.distributed as dist

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import paper_2106_15740_b200 as Q
    import qtn_oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    G = json.load(open(golden_path))
    graph = Q.random_regular_graph(G["n"], 3, 0)
    edges = [tuple(e) for e in graph.edges]
    shard = [j.index for j in Q.energy.rank_shard(graph, G["p"], "zz+diagonal", rank, world,
                                                  compile_plans=False)]
    # two angle sets: the config's and a second one
    sets = [(G["gammas"], G["betas"]), ([0.3, 1.1], [0.9, 0.2])]
    partial = np.zeros(len(sets))
    for s, (g, b) in enumerate(sets):
        zz = [O.edge_zz(G["n"], edges, edges[e], g, b, "zz+diagonal") for e in shard]
        partial[s] = O.energy_from_zz(zz)
    total = Q.energy.reduce_partials(partial)
    all_shards = [None] * world
    dist.all_gather_object(all_shards, shard)
    out_q.put((rank, total.tolist(), all_shards))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_energy_equals_single(golden):
    G = golden("config2.json")
    want0 = sum((1 - r["value"][0]) / 2 for r in G["modes"]["zz+diagonal"])
    import qtn_oracle as O

    edges = [tuple(e) for e in G["edges"]]
    want1 = O.energy_from_zz([O.edge_zz(100, edges, e, [0.3, 1.1], [0.9, 0.2], "zz+diagonal")
                              for e in edges])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    from conftest import GOLDEN

    procs = [ctx.Process(target=_worker, args=(r, 2, port, os.path.join(GOLDEN, "config2.json"), q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, total, shards in res:
        assert abs(total[0] - want0) < 1e-9
        assert abs(total[1] - want1) < 1e-9
        assert sorted(shards[0] + shards[1]) == list(range(150))
        assert not set(shards[0]) & set(shards[1])
