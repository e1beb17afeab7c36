"""bench.py's multi-rank path on CPU (gloo, world size 2): the `--gpus N`
launcher (spawn, torchrun environment), job planning with LPT sharding and
shard-only compilation, the per-step all-reduce, max-over-ranks timing and
the JSON line — with the CPU oracle's partial energies standing in for the
GPU executor and a host rig standing in for the CUDA one.  On GPUs the same
code runs with CudaRig, EnergyPlan and NCCL."""

import json
import os
import time

import numpy as np
import pytest


class CpuRig:
    """Host stand-in for bench.CudaRig: perf_counter timing, gloo."""

    def __init__(self, local):
        import torch

        self.torch = torch
        self.device = torch.device("cpu")
        self.stream = None

    def init_dist(self):
        import torch.distributed as dist

        dist.init_process_group("gloo")
        return dist

    def flush(self):
        pass

    def sync(self):
        pass

    def start(self):
        return time.perf_counter()

    def end(self):
        return time.perf_counter()

    def elapsed(self, t0, t1):
        return t1 - t0

    def clocks(self):
        import bench

        return bench.NoClocks()


class OraclePlan:
    """EnergyPlan's bench-facing interface over the CPU oracle: per job
    (edge, or one slice of it) the restated bucket elimination along the
    job's own order, with the slice's variables fixed (network.py:153-165)."""

    def __init__(self, graph_args, jobs):
        import qtn_oracle as O

        self.O = O
        self.graph, self.p, self.mode, _ = graph_args
        self.jobs = jobs
        self.edges = [tuple(e) for e in self.graph.edges]
        self.launches = 0
        self._cache = {}

    def _partials(self, angles):
        import torch

        a = np.atleast_2d(np.asarray(angles, dtype=np.float64))
        out = np.zeros(a.shape[0])
        for s, vec in enumerate(a):
            key = vec.tobytes()
            if key not in self._cache:
                e = 0.0
                for j in self.jobs:
                    t, nv, fixed = self.O.edge_network(self.graph.node_count, self.edges,
                                                       self.edges[j.index], list(vec[:self.p]),
                                                       list(vec[self.p:]), self.mode)
                    fixed = {**fixed, **j.assignment}
                    val, _ = self.O.contract(t, nv, fixed, list(j.order.sequence))
                    e += (j.weight - complex(val).real) / 2.0
                self._cache[key] = e
            out[s] = self._cache[key]
        return out

    def launch(self, angles_dev, stream=None):
        import torch

        self.launches = 1 if self.jobs else 0
        return {"energy": torch.from_numpy(self._partials(angles_dev.numpy()))}

    def execute_only(self, angles_dev, stream=None):
        self._partials(angles_dev.numpy())

    def energies(self, angle_sets):
        return self._partials(angle_sets)

    def describe(self, n_sets):
        return {"kernel": "oracle", "dtype": "c128 (CPU oracle stand-in)"}

    def alg_bytes_eval(self, n_sets):
        return 0.0


def _target(args):
    import bench

    return bench.run_gpu(args, rig_factory=CpuRig, plan_factory=OraclePlan)


def _run(tmp_path, argv):
    import bench

    out = tmp_path / "line.json"
    args = bench.parse_args(argv + ["--no-cpu-baseline", "--no-records", "--out-json", str(out)])
    rc = bench.main_with(args, _target)
    assert rc == 0
    return json.loads(out.read_text())


def test_two_rank_bench_line(tmp_path, golden):
    """config 2 weak scaling on 2 ranks: 75 edges each, 2 angle sets per rank
    (4 in all); set 0's energy is the reference's."""
    G = golden("config2.json")
    want = sum((1 - r["value"][0]) / 2 for r in G["modes"]["zz+diagonal"])
    line = _run(tmp_path, ["--gpus", "2", "--workload", "config2", "--angle-sets", "2",
                           "--steps", "1", "--warmup", "3"])
    assert line["n_gpus"] == 2
    assert line["config"]["angle_sets_per_step"] == 4
    assert line["config"]["contractions_per_step"] == 600
    assert line["run"]["jobs_on_rank0"] == 75
    assert abs(line["run"]["energy_set0"] - want) < 1e-9
    assert line["value"] > 0 and line["e2e"]["value"] > 0


def test_two_rank_slice_sharding_equals_unsliced(tmp_path, golden):
    """Strong scaling over slices: config 4 edge #0 in 2^2 slices striped
    over 2 ranks (2 slices each); the all-reduced energy equals the unsliced
    reference value."""
    G = golden("config4.json")
    rec = [r for r in G["modes"]["zz+diagonal"] if r["edge_index"] == 0][0]
    want = (1 - rec["value"][0]) / 2
    line = _run(tmp_path, ["--gpus", "2", "--workload", "config4", "--edge-ids", "0",
                           "--slices", "2", "--scaling", "strong", "--steps", "1",
                           "--warmup", "3"])
    assert line["n_gpus"] == 2
    assert line["config"]["slices_per_edge"] == 4
    assert line["run"]["jobs_on_rank0"] == 2
    assert abs(line["run"]["energy_set0"] - want) < 1e-10


def test_empty_shard_rank(tmp_path, golden):
    """More ranks than jobs: config 4 edge #0 unsliced on 2 ranks — rank 1
    has no job, contributes zeros, and nobody hangs in the all-reduce."""
    G = golden("config4.json")
    rec = [r for r in G["modes"]["zz+diagonal"] if r["edge_index"] == 0][0]
    line = _run(tmp_path, ["--gpus", "2", "--workload", "config4", "--edge-ids", "0",
                           "--scaling", "strong", "--steps", "1", "--warmup", "3"])
    assert line["n_gpus"] == 2
    assert abs(line["run"]["energy_set0"] - (1 - rec["value"][0]) / 2) < 1e-10
