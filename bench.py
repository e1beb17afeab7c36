#!/usr/bin/env python
"""Benchmark: QAOA edge-energy contractions/sec and bucket-kernel HBM GB/s.

Default workload (BASELINE.json configs[1], "config 2"): QAOA p=2 MaxCut
energy on the seeded random 3-regular graph N=100 (graph seed 0), all 150
per-edge light-cone networks in zz+diagonal mode, orders from the reference
rgreedy(10, 0.02, seed 0), plans cached.  One step evaluates the energy for
a batch of A angle sets (set 0 is the config's seeded angles, the rest are
seeded U[0, pi) draws — the parameter batch a QAOA optimiser evaluates),
i.e. 150*A edge contractions: on-device tensor generation, the set-major
executor, and the energy reduction.

Multi-GPU (`--gpus N`; under torchrun, or spawned here when WORLD_SIZE is
unset): one process per GPU, NCCL.  Jobs (edge networks, or 2^k slices of
them with `--slices k`) are LPT-sharded over the ranks; every rank orders
every job (the partition needs all costs) but compiles only its shard; one
all-reduce of the per-set partial energies per step.  `--scaling weak`
(default): the angle-set batch is A*N (fixed work per GPU); `strong`: the
batch stays A and the jobs are split (e.g. `--workload config4 --slices 4
--scaling strong`: config 4's 16 slices striped over the ranks).

The default single-GPU run also carries sub-records for the other configs
(`records`): config 2 at one angle set and with complex128 rows, config 4
edge #1058 unsliced and in 2^3 slices, the config 3 ablation (default vs
zz+diagonal: widths and time) and the config 5 bucket (parity-checked) — each
with its roofline fraction (algorithmic and DRAM), e2e figure and a one-core
CPU baseline of the reference (bench_reference.py).

`--impl reference` times the reference's own implementation (the installed
`qtnsim` from baseline/_ref, else the oracle port) on all host cores, on the
same workload config (bench_reference.py); it never imports the B200 package.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback
METRIC = "QAOA edge-energy contractions/sec"


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None
        # in-process NVML samples taken while a timed step is executing: the
        # timed region of a fast workload is shorter than nvidia-smi's period
        self.nv = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self.nv = None

    def sample_now(self):
        """One NVML sample (clocks + event reasons) appended to rows."""
        if self.nv is None:
            return
        nv, h = self.nv
        try:
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            bits = fn(h)
            flag = lambda b: "Active" if bits & b else "Not Active"
            # hw_slowdown 0x8, hw_thermal 0x40, sw_thermal 0x20, sw_power_cap 0x4
            self.rows.append([str(sm), str(mx), flag(0x8), flag(0x40), flag(0x20), flag(0x4)])
        except Exception:
            pass

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0:  # first sample before timing
                time.sleep(0.05)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


class NoClocks:
    def sample_now(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass

    def summary(self):
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no GPU"]}


# --------------------------------------------------------------- workloads
WORKLOADS = {
    "config1": dict(n=20, p=1, mode="zz+diagonal", edges=None, dtype="complex128", sets=1024),
    "config2": dict(n=100, p=2, mode="zz+diagonal", edges=None, dtype="complex64", sets=1024),
    "config3": dict(n=244, p=3, mode="zz+diagonal", edges=None, dtype="complex64", sets=256),
    "config3-default": dict(n=244, p=3, mode="default", edges=None, dtype="complex64", sets=1),
    "config4": dict(n=1000, p=5, mode="zz+diagonal", edges=[1058], dtype="complex64", sets=1),
}
N_EDGES = {20: 30, 100: 150, 244: 366, 1000: 1500}  # 3-regular: 3N/2 edges


def seeded_angle_vector(p, seed=0):
    """Config angles: gammas then betas ~ U[0, pi) from
    default_rng(seed) (= pipeline.seeded_angles(p, seed).as_vector())."""
    rng = np.random.default_rng(seed)
    g = rng.uniform(0.0, math.pi, p)
    b = rng.uniform(0.0, math.pi, p)
    return np.concatenate([g, b])


def angle_sets(p, n_sets, seed=0):
    a = np.empty((n_sets, 2 * p), dtype=np.float64)
    a[0] = seeded_angle_vector(p, seed)
    if n_sets > 1:
        rng = np.random.default_rng(1000 + seed)
        a[1:] = rng.uniform(0.0, math.pi, (n_sets - 1, 2 * p))
    return a


def edge_ids_of(wl):
    return list(wl["edges"]) if wl["edges"] is not None else list(range(N_EDGES[wl["n"]]))


def batch_sets(args, wl, world):
    per = args.angle_sets if args.angle_sets else wl["sets"]
    return per * (world if args.scaling == "weak" else 1)


def workload_config(args, wl, world):
    """The workload description both arms print (identical by construction;
    nothing here depends on a measurement)."""
    A = batch_sets(args, wl, world)
    edges = edge_ids_of(wl)
    per = args.angle_sets if args.angle_sets else wl["sets"]
    return {
        "workload": args.workload, "n": wl["n"], "p": wl["p"], "mode": wl["mode"],
        "edges": len(edges), "edge_ids": edges if len(edges) <= 8 else f"0..{len(edges) - 1}",
        "angle_sets_per_step": A, "slices_per_edge": 2 ** args.slices,
        "contractions_per_step": len(edges) * A,
        "graph": "random_regular_graph(n, 3, seed=0)", "angles": "set 0 = seeded_angles(p, 0), "
        "others U[0, pi) seeded; re-drawn every step",
        "order": "reference rgreedy_order(n_repeats=10, temp=0.02, seed=0), cached",
        "l2": "flushed between timed steps (256 MiB write)",
        "parallelism": (f"jobs LPT-sharded over {world} GPU(s), {per} angle sets per GPU per step"
                        if args.scaling == "weak" else
                        f"jobs LPT-sharded over {world} GPU(s), {A} angle sets per step"),
    }


def profile_record(key):
    """A committed ncu summary (profiles/ncu_full_*.json, newest first) for
    "kernel@workload", or None when that pair was not captured."""
    prof = os.path.join(ROOT, "profiles")
    if not os.path.isdir(prof):
        return None
    for name in sorted(os.listdir(prof), reverse=True):
        if name.startswith("ncu_full") and name.endswith(".json"):
            try:
                with open(os.path.join(prof, name)) as f:
                    d = json.load(f)
                k = d.get("kernels", {}).get(key)
                if k and k.get("dram_bytes_per_launch"):
                    return dict(k, file=name)
            except Exception:
                pass
    return None


# -------------------------------------------------------------- launching
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_entry(rank, world, port, target, args):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    rc = target(args)
    if rc:
        raise SystemExit(rc)


def spawn_ranks(args, target, world):
    """`--gpus N` without torchrun: N processes (spawn), one per GPU, with
    the torchrun environment; returns the worst exit code."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    port = free_port()
    procs = [ctx.Process(target=_rank_entry, args=(r, world, port, target, args))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join()
    return max(abs(p.exitcode or 0) for p in procs)


# -------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's CPU implementation on all host cores, on this arm's
    config; rank 0 only under torchrun.  Never imports the B200 package."""
    apply_edge_override(args)  # spawned ranks re-import bench
    world, rank, _ = dist_env()
    world = max(world, args.gpus)
    if rank != 0:
        return 0
    import bench_reference as R

    wl = WORKLOADS[args.workload]
    cfg = workload_config(args, wl, world)
    A = cfg["angle_sets_per_step"]
    sets = angle_sets(wl["p"], max(A, 1))
    cores = os.cpu_count() or 1
    # config 4 slices spread one edge over the cores (the fixed-variable
    # mechanism, network.py:78, 153-165): 2^k >= cores, k <= 4
    slice_k = args.slices
    if wl["edges"] is not None and len(wl["edges"]) < cores:
        slice_k = max(slice_k, min(4, max(0, math.ceil(math.log2(cores)))))
    t0 = time.perf_counter()
    w = R.prepare(wl["n"], wl["p"], wl["mode"], edge_ids_of(wl), sets[0], slice_k)
    prep_s = time.perf_counter() - t0
    # each step: a bounded sample of the arm's step — S angle sets x every
    # edge network, S sized from one probe step so the whole run stays short
    probe, _, pv = R.timed_steps(w, lambda it: [sets[0]], 0, 1, cores)
    # E = sum_e (1 - <ZZ>_e)/2; the slices of an edge add up to its <ZZ>
    energy0 = 0.5 * len(w.edge_ids) - 0.5 * float(sum(complex(z).real for z in pv))
    budget = args.ref_step_seconds
    S = int(max(1, min(A, budget / max(probe[0], 1e-6))))
    step_sets = lambda it: [sets[(it * S + k) % len(sets)] for k in range(S)]
    times, per, vals = R.timed_steps(w, step_sets, args.warmup, args.steps, cores)
    total = sum(times)
    value = per * len(times) / total
    sample = (f"per step {S} of the {A} angle sets x {len(w.edge_ids)} edge network(s)"
              f"{f' in 2^{slice_k} slices' if slice_k else ''} ({per} contractions), "
              f"{cores} worker processes: " +
              ("qtnsim circuit_to_network + contract (baseline/_ref)" if w.kind == "reference"
               else "oracle port network build + bucket elimination") +
              f", complex128, orders prepared once ({prep_s:.1f}s, untimed)")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "contractions/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "c128",
        "data": "synthetic (seeded random 3-regular graph, seeded angles)",
        "config": cfg,
        "run": {"energy_set0": energy0, "prepare_seconds": prep_s,
                "modules": sorted(m for m in sys.modules if m.startswith("paper_2106"))},
        "cpu_baseline": {"value": value, "unit": "contractions/s", "cores": cores,
                         "kind": w.kind, "sample": sample, "host": R.host_cpu()},
        "e2e": {"value": value, "unit": "contractions/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ device
class CudaRig:
    """One GPU: stream, CUDA-event timing, L2 flush, NCCL."""

    def __init__(self, local):
        import torch

        self.torch = torch
        backend = os.environ.get("QTN_DIST_BACKEND", "nccl")
        # QTN_SHARE_GPU=1 (+ QTN_DIST_BACKEND=gloo): exercise the multi-rank
        # path with several ranks on one GPU; their timings mean nothing
        if os.environ.get("QTN_SHARE_GPU"):
            local = 0
        self.index = local
        torch.cuda.set_device(local)
        self.device = torch.device("cuda", local)
        self.stream = torch.cuda.current_stream(self.device)
        self.backend = backend
        self._flush = torch.empty(256 << 20, dtype=torch.uint8, device=self.device)  # > L2

    def init_dist(self):
        import torch.distributed as dist

        if self.backend == "nccl":
            dist.init_process_group("nccl", device_id=self.device)
        else:
            dist.init_process_group(self.backend)
        return dist

    def flush(self):
        self._flush.zero_()

    def sync(self):
        self.torch.cuda.synchronize(self.device)

    def start(self):
        e0 = self.torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        return e0

    def end(self):
        e1 = self.torch.cuda.Event(enable_timing=True)
        e1.record(self.stream)
        return e1

    def elapsed(self, e0, e1):
        e1.synchronize()
        return e0.elapsed_time(e1) / 1e3

    def clocks(self):
        return ClockSampler(self.index)


def make_energy_plan(graph_args, jobs):
    import paper_2106_15740_b200 as Q

    graph, p, mode, dtype = graph_args
    return Q.EnergyPlan(graph, p, mode, dtype=dtype, jobs=jobs)


def plan_jobs(wl, args, dtype, world, rank):
    """Order every job, keep this rank's LPT shard, compile only it."""
    import paper_2106_15740_b200 as Q

    graph = Q.random_regular_graph(wl["n"], 3, 0)
    ids = edge_ids_of(wl)
    alljobs = Q.plan_edges(graph, wl["p"], wl["mode"], ids, dtype=dtype, slice_k=args.slices,
                           compile_plans=False)
    widths = [j.report.width for j in alljobs]
    keep = Q.shard_edges([j.cost for j in alljobs], world)[rank] if world > 1 else \
        list(range(len(alljobs)))
    jobs = [alljobs[k] for k in keep]
    Q.compile_jobs(jobs, dtype=dtype)
    return graph, jobs, widths


def measure(rig, plan, p, A, steps, warmup, dist=None, clk=None, n_units=None, ring=4):
    """Time `steps` evaluations of A angle sets: device-timed steps (events
    on the launching stream, L2 flushed between steps), the executors alone,
    and the public host-to-host call.  Max over ranks.  Returns a dict."""
    torch = rig.torch
    sets = angle_sets(p, A)
    ring_host = [sets] + [np.random.default_rng(2000 + k).uniform(0.0, math.pi, sets.shape)
                          for k in range(1, ring)]
    ring_dev = [torch.from_numpy(h).to(rig.device) for h in ring_host]
    it = [0]

    def step():
        b = plan.launch(ring_dev[it[0] % ring], rig.stream)
        it[0] += 1
        if dist is not None:
            dist.all_reduce(b["energy"])
        return b

    for _ in range(warmup):
        step()
    rig.sync()
    if dist is not None:
        dist.barrier()
    step_t, kern_t, launches = [], [], 0
    for _ in range(steps):
        rig.flush()
        rig.sync()
        e0 = rig.start()
        step()
        e1 = rig.end()
        if clk is not None:
            clk.sample_now()  # while the step executes (outside the events)
        step_t.append(rig.elapsed(e0, e1))
        launches += plan.launches
        rig.flush()
        rig.sync()
        k0 = rig.start()
        plan.execute_only(ring_dev[it[0] % ring], rig.stream)
        kern_t.append(rig.elapsed(k0, rig.end()))
    total = sum(step_t)
    # end to end through the public API: host angles -> energies on host,
    # H2D of the angles and D2H of the energies inside the timed region
    e2e_t = []
    for k in range(warmup + steps):
        rig.flush()
        rig.sync()
        if dist is not None:
            dist.barrier()
        t1 = time.perf_counter()
        en = plan.energies(ring_host[k % ring])
        if dist is not None:
            buf = torch.from_numpy(en).to(rig.device)
            dist.all_reduce(buf)
            en = buf.cpu().numpy()
        if k >= warmup:
            e2e_t.append(time.perf_counter() - t1)
    e2e_total = sum(e2e_t)
    kt = sum(kern_t) / len(kern_t)
    if dist is not None:
        t = torch.tensor([total, e2e_total, kt], dtype=torch.float64, device=rig.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total, e2e_total, kt = (float(x) for x in t.cpu())
    en = plan.energies(sets)  # set 0 at the config's seeded angles
    if dist is not None:
        buf = torch.from_numpy(en).to(rig.device)
        dist.all_reduce(buf)
        en = buf.cpu().numpy()
    units = n_units * steps
    return {"value": units / total, "ms_per_step": 1e3 * total / steps, "kernel_s": kt,
            "e2e": units / e2e_total, "e2e_ms_per_step": 1e3 * e2e_total / steps,
            "launches": launches, "energy_set0": float(en[0]), "h2d": int(sets.nbytes),
            "d2h": 8 * A}


def roofline(plan, A, kt, key):
    peak, kind = hbm_peak()
    alg = plan.alg_bytes_eval(A)
    achieved = alg / kt / 1e9
    prof = profile_record(key)
    traffic = prof["dram_bytes_per_launch"] if prof else None
    r = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
         "frac": achieved / peak, "traffic": traffic, "kernel": key.split("@")[0],
         "peak_source": f"{kind} (MEASURED_PEAKS.json hbm_gbs)",
         "alg_bytes_per_launch": alg, "avg_launch_s": kt,
         "scope": "one evaluation of all angle sets: every executor launch (set-major: gate "
                  "rows + level launches + fold; HBM: level launches + fold), CUDA events on "
                  "the launching stream"}
    ex = plan.exec_bytes_eval(A) if hasattr(plan, "exec_bytes_eval") else alg
    if ex != alg:
        # fused chains skip the union-size products: the bytes the kernels move
        r["exec_bytes_per_launch"] = ex
        r["exec_frac"] = ex / kt / 1e9 / peak
        r["note"] = ("achieved/frac count the reference's per-bucket bytes (SURVEY 8d); fused chains "
                     "(fused_kernel, xt_kernel) never write or re-read the union-size intermediates, so "
                     "frac may exceed 1: exec_frac counts the bytes the kernels move, dram_frac the "
                     "ncu DRAM bytes of the same evaluation")
    if traffic:
        # DRAM bytes of the committed ncu capture of the same evaluation over
        # the live executor time: the fraction of HBM actually moving
        r["dram_frac"] = traffic / kt / 1e9 / peak
        r["traffic_source"] = f"profiles/{prof['file']} [{key}]"
    return r


# --------------------------------------------------------------- config 5
def config5_bucket(torch, w=30, m=16, c64=True, reps=5, seed=0, check=True, n_sample=4096):
    """Synthetic config-5 bucket: one rank-(w+1) operand over
    a seeded permutation of (v, x_1..x_w) plus m rank-1 (v) / rank-2 (v, x_r)
    operands, entries re/im ~ N(0, 1) (seeded, generated on the device),
    output rank w, through the C ABI `qtn_bucket_contract`.  Before the GB/s
    is reported, 4096 random outputs plus the first and last 4096-output
    tile are recomputed on the host in float64 from the operand entries they
    touch: out[o] = sum_v prod_t T_t[idx_t(o, v)] (contraction.py:82-96)."""
    import ctypes as C

    from paper_2106_15740_b200 import _native as N

    rng = np.random.default_rng(seed)
    perm = [int(x) for x in rng.permutation(w + 1)]
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    fdt = torch.float32 if c64 else torch.float64
    cdt = torch.complex64 if c64 else torch.complex128
    big = torch.randn(4 << w, dtype=fdt, device=dev, generator=g).view(cdt)
    ops_vars = [perm]
    datas = [big]
    for _ in range(m):
        if rng.random() < 0.5:
            ops_vars.append([0])
        else:
            ops_vars.append([0, int(rng.integers(1, w + 1))])
        datas.append(torch.randn(2 << len(ops_vars[-1]), dtype=fdt, device=dev,
                                 generator=g).view(cdt))
    ranks = np.asarray([len(v) for v in ops_vars], dtype=np.int32)
    offs = np.zeros(len(ranks) + 1, dtype=np.int32)
    offs[1:] = np.cumsum(ranks)
    flat = np.asarray([x for v in ops_vars for x in v], dtype=np.int32)
    ov = np.zeros(w, dtype=np.int32)
    r = C.c_int32()
    N.check(N.lib.qtn_bucket_layout(len(ranks), N.i32(ranks), N.i32(offs), N.i32(flat), 0,
                                    C.byref(r), N.i32(ov)))
    out = torch.empty(1 << w, dtype=cdt, device=dev)
    ptrs = (C.c_void_p * len(datas))(*[d.data_ptr() for d in datas])
    flags = np.full(len(datas), 1 if c64 else 0, dtype=np.uint8)
    st = torch.cuda.current_stream()

    def run():
        N.check(N.lib.qtn_bucket_contract(len(ranks), N.i32(ranks), N.i32(offs), N.i32(flat),
                                          ptrs, N.u8(flags), 0, w, N.i32(ov), 1 if c64 else 0,
                                          out.data_ptr(), st.cuda_stream))

    for _ in range(2):
        run()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        run()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    esz = 8 if c64 else 16
    alg = esz * ((2 << w) + sum(1 << len(v) for v in ops_vars[1:]) + (1 << w))
    t = statistics.median(ts)
    rec = {"w": w, "m": m, "dtype": "c64" if c64 else "c128", "alg_bytes": alg, "seconds": t,
           "gbs": alg / t / 1e9}
    if check:
        rec.update(sampled_bucket_check(torch, ops_vars, datas, list(ov), out, w, n_sample,
                                        seed, 1e-5 if c64 else 1e-10))
    del big, out, datas
    torch.cuda.empty_cache()
    return rec


def sampled_bucket_check(torch, ops_vars, datas, out_vars, out, w, n_sample, seed, tol):
    """float64 host recomputation of sampled outputs of one bucket from the
    operand entries they touch (index maps in the reference's C order: the
    first variable is the most significant bit, network.py:36-61)."""
    rng = np.random.default_rng(seed + 7)
    tile = min(4096, 1 << w)
    outs = np.unique(np.concatenate([
        rng.integers(0, 1 << w, n_sample, dtype=np.int64),
        np.arange(tile, dtype=np.int64), (1 << w) - 1 - np.arange(tile, dtype=np.int64)]))
    # value of each output variable at each sampled o
    val = {int(x): (outs >> (w - 1 - k)) & 1 for k, x in enumerate(out_vars)}
    acc = np.zeros(len(outs), dtype=np.complex128)
    for v in (0, 1):
        val[0] = np.full(len(outs), v, dtype=np.int64)
        prod = np.ones(len(outs), dtype=np.complex128)
        for vs, d in zip(ops_vars, datas):
            idx = np.zeros(len(outs), dtype=np.int64)
            for pos, x in enumerate(vs):
                idx |= val[int(x)] << (len(vs) - 1 - pos)
            got = d[torch.from_numpy(idx).to(d.device)].cpu().numpy().astype(np.complex128)
            prod *= got
        acc += prod
    got = out[torch.from_numpy(outs).to(out.device)].cpu().numpy().astype(np.complex128)
    err = float(np.abs(got - acc).max() / max(np.abs(acc).max(), 1e-300))
    ok = err <= tol
    if not ok:
        raise AssertionError(f"config-5 bucket parity failed: max rel err {err:.3g} > {tol}")
    return {"parity": "checked", "parity_outputs": int(len(outs)), "parity_max_rel_err": err,
            "parity_tol": tol}


# ------------------------------------------------------------ sub-records
def workload_record(rig, name, wl, A, dtype, slices, steps, warmup, cpu=None, key_name=None):
    """One config measured in this process (1 GPU): value, e2e, roofline
    (algorithmic and DRAM fractions), widths."""
    class _A:
        pass

    a = _A()
    a.slices = slices
    graph, jobs, widths = plan_jobs(wl, a, dtype, 1, 0)
    plan = make_energy_plan((graph, wl["p"], wl["mode"], dtype), jobs)
    n_units = len(edge_ids_of(wl)) * A
    m = measure(rig, plan, wl["p"], A, steps, warmup, n_units=n_units)
    desc = plan.describe(A)
    roof = roofline(plan, A, m["kernel_s"], f"{desc['kernel']}@{key_name or name}")
    rec = {"workload": name, "n": wl["n"], "p": wl["p"], "mode": wl["mode"],
           "edges": len(edge_ids_of(wl)), "angle_sets_per_step": A,
           "slices_per_edge": 2 ** slices, "dtype": desc["dtype"],
           "value": m["value"], "unit": "contractions/s", "ms_per_step": m["ms_per_step"],
           "width_max": max(widths), "width_min": min(widths),
           "width_hist": {str(k): widths.count(k) for k in sorted(set(widths))},
           "energy_set0": m["energy_set0"], "gpu_launches_per_step": m["launches"] // steps,
           "roofline": roof,
           "e2e": {"value": m["e2e"], "unit": "contractions/s", "h2d_bytes_per_step": m["h2d"],
                   "d2h_bytes_per_step": m["d2h"],
                   "api": "EnergyPlan.energies(host angles) -> host energies"},
           "cpu_baseline": cpu}
    del plan
    rig.torch.cuda.empty_cache()
    return rec


def cpu_sample(wl, sets, seconds, edge_subset=None, slice_k=0, label=None):
    import bench_reference as R

    ids = edge_ids_of(wl) if edge_subset is None else edge_subset
    try:
        r = R.sample_rate(wl["n"], wl["p"], wl["mode"], ids, sets, seconds=seconds, cores=1,
                          slice_k=slice_k)
        if label:
            r["sample"] = label + "; " + r["sample"]
        return r
    except Exception as ex:  # report, do not hide
        return {"error": repr(ex)}


def sub_records(rig, args, main_cpu):
    """The other configs, so the driver's default run carries them."""
    recs = {}
    t_all = time.perf_counter()
    c2 = WORKLOADS["config2"]
    sets2 = angle_sets(2, 4)

    def guard(name, fn):
        t0 = time.perf_counter()
        try:
            recs[name] = fn()
        except Exception as ex:
            recs[name] = {"error": repr(ex)}
        recs[name]["wall_s"] = time.perf_counter() - t0

    same = {"same_as": "top-level cpu_baseline (same workload)"} if main_cpu else None
    # config 2, one angle set per step: the sequential QAOA optimiser's call
    guard("config2_A1", lambda: workload_record(rig, "config2", c2, 1, "complex64", 0, 20,
                                                args.warmup, cpu=same, key_name="config2-A1"))
    # config 2 with complex128 rows throughout (the survey's c128 policy)
    guard("config2_c128", lambda: workload_record(rig, "config2", c2, 1024, "complex128", 0,
                                                  10, args.warmup, cpu=same,
                                                  key_name="config2-c128"))
    # config 4: edge #1058 unsliced and in 2^3 slices
    c4 = WORKLOADS["config4"]
    s4 = angle_sets(5, 2)
    cpu4 = cpu_sample(c4, s4, args.cpu_seconds / 2, slice_k=4,
                      label="slices of edge #1058 (2^4), each weighted 1/16")
    guard("config4", lambda: workload_record(rig, "config4", c4, 1, "complex64", 0, 20,
                                             args.warmup, cpu=cpu4))
    guard("config4_k3", lambda: workload_record(rig, "config4", c4, 1, "complex64", 3, 20,
                                                args.warmup, cpu=cpu4, key_name="config4-k3"))
    # config 3 ablation: default (H/CNOT) vs zz+diagonal, widths and time
    sub = list(range(0, 366, 23))
    s3 = angle_sets(3, 2)
    for name, mode, A in (("config3_default", "default", 1), ("config3_zzdiag", "zz+diagonal", 256)):
        wl = dict(WORKLOADS["config3"], mode=mode)
        cpu = cpu_sample(wl, s3, args.cpu_seconds / 2, edge_subset=sub,
                         label="edges 0, 23, .., 345 of 366")
        guard(name, lambda wl=wl, A=A, cpu=cpu, name=name: workload_record(
            rig, "config3", wl, A, "complex64", 0, 10, args.warmup, cpu=cpu,
            key_name="config3-default" if mode == "default" else "config3"))
    a3 = {}
    for k, v in (("default", recs.get("config3_default", {})),
                 ("zz+diagonal", recs.get("config3_zzdiag", {}))):
        if "value" in v:
            a3[k] = {"width_max": v["width_max"], "width_min": v["width_min"],
                     "ms_per_edge_energy_set": v["ms_per_step"] / (366 * v["angle_sets_per_step"]),
                     "contractions_per_s": v["value"], "frac": v["roofline"]["frac"]}
    recs["config3_ablation"] = a3
    # config 5: the w=30, m=16 bucket, parity-checked, with the reference
    # bucket ops on one core at w=22 as its CPU baseline
    import bench_reference as R

    def c5():
        peak, _ = hbm_peak()
        r = config5_bucket(rig.torch, w=args.c5_w, m=args.c5_m)
        r["frac"] = r["gbs"] / peak
        r["roofline"] = {"bound": "hbm", "achieved": r["gbs"], "peak": peak, "unit": "GB/s",
                         "frac": r["frac"]}
        prof = profile_record(f"stream_kernel@config5")
        if prof:
            r["roofline"]["traffic"] = prof["dram_bytes_per_launch"]
            r["roofline"]["dram_frac"] = prof["dram_bytes_per_launch"] / r["seconds"] / 1e9 / peak
        r["cpu_baseline"] = R.bucket_rate(w_bits=22, m=args.c5_m)
        r["e2e"] = None  # a device-resident microbench: no host path
        return r

    guard("config5", c5)

    # the drop-in call itself: contract(network, order) on one network, host
    # network in, host scalar out (what the reference's own callers see:
    # bench.py:247, cli.py:108), beside qtnsim.contract on the same network
    def call_latency():
        import paper_2106_15740_b200 as Q

        out = {"unit": "ms per contract() call (median of 20 after one warm call)",
               "api": "contract(network, order): host TensorNetwork -> host complex"}
        for key, name in (("config2_edge0", "config2"), ("config3_default_edge0", "config3")):
            wl = dict(WORKLOADS[name], mode="default") if name == "config3" else WORKLOADS[name]
            g = Q.random_regular_graph(wl["n"], 3, 0)
            ang = angle_sets(wl["p"], 1)[0]
            net = Q.build_energy_network(g, g.edges[0], Q.seeded_angles(wl["p"], 0), wl["mode"])
            order, _ = Q.rgreedy_order(Q.line_graph(net))
            v = Q.contract(net, order)
            ts = []
            for _ in range(20):
                t0 = time.perf_counter()
                v = Q.contract(net, order)
                ts.append(time.perf_counter() - t0)
            ts.sort()
            rec = {"ms": ts[len(ts) // 2] * 1e3, "ms_min": ts[0] * 1e3,
                   "value": [v.real, v.imag]}
            w = R.prepare(wl["n"], wl["p"], wl["mode"], [0], ang)
            cv = w.zz(0, ang[:wl["p"]], ang[wl["p"]:])
            cs = []
            for _ in range(5):
                t0 = time.perf_counter()
                cv = w.zz(0, ang[:wl["p"]], ang[wl["p"]:])
                cs.append(time.perf_counter() - t0)
            cs.sort()
            rec["cpu_baseline"] = {"ms": cs[len(cs) // 2] * 1e3, "cores": 1, "kind": w.kind,
                                   "sample": "circuit_to_network + contract on the same edge "
                                             "network, median of 5", "value": [cv.real, cv.imag]}
            rec["rel_err_vs_cpu"] = abs(v - cv) / max(abs(cv), 1e-300)
            out[key] = rec
        return out

    guard("contract_call", call_latency)
    recs["wall_s"] = time.perf_counter() - t_all
    return recs


# ------------------------------------------------------------------ GPU arm
def run_gpu(args, rig_factory=None, plan_factory=None, plan_jobs_fn=None):
    apply_edge_override(args)  # spawned ranks re-import bench
    world, rank, local = dist_env()
    rig = (rig_factory or CudaRig)(local)
    dist = rig.init_dist() if world > 1 else None
    wl = WORKLOADS[args.workload]
    dtype = args.dtype or wl["dtype"]
    t0 = time.perf_counter()
    graph, jobs, widths = (plan_jobs_fn or plan_jobs)(wl, args, dtype, world, rank)
    plan = (plan_factory or make_energy_plan)((graph, wl["p"], wl["mode"], dtype), jobs)
    plan_s = time.perf_counter() - t0
    cfg = workload_config(args, wl, world)
    A = cfg["angle_sets_per_step"]
    clk = rig.clocks().__enter__()  # sampled through warm-up, timed and e2e loops
    m = measure(rig, plan, wl["p"], A, args.steps, args.warmup, dist=dist, clk=clk,
                n_units=cfg["contractions_per_step"])
    clk.__exit__(None, None, None)
    desc = plan.describe(A)
    roof = roofline(plan, A, m["kernel_s"], f"{desc['kernel']}@{args.workload}") \
        if plan.alg_bytes_eval(A) else None
    if dist is not None:
        # the roofline is the dominant kernel's on one GPU: rank 0's shard
        pass
    out = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            cpu = cpu_sample(wl, angle_sets(wl["p"], 4), args.cpu_seconds)
        recs = None
        if world == 1 and not args.no_records and args.workload == "config2" and \
                hasattr(rig, "torch") and rig.torch.cuda.is_available():
            recs = sub_records(rig, args, cpu)
        out = {
            "metric": METRIC,
            "value": m["value"],
            "unit": "contractions/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": m["ms_per_step"],
            "higher_is_better": True,
            "scaling": args.scaling,
            "vs_baseline": None,
            "dtype": desc["dtype"],
            "data": "synthetic (seeded random 3-regular graph, seeded angles)",
            "config": cfg,
            "run": {"energy_set0": m["energy_set0"], "plan_seconds": plan_s,
                    "width_max": max(widths), "jobs_on_rank0": len(jobs)},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": m["e2e"], "unit": "contractions/s",
                    "h2d_bytes_per_step": m["h2d"], "d2h_bytes_per_step": m["d2h"],
                    "api": "EnergyPlan.energies(host angle array) -> host energies"},
            "gpu_launches": m["launches"],
            "clocks": clk.summary(),
            "records": recs,
        }
        print(json.dumps(out), flush=True)
        if args.out_json:
            with open(args.out_json, "w") as f:
                json.dump(out, f)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_config5(args):
    """Config-5 roofline sweep: one JSON line per (w, m), each parity-checked."""
    import torch

    peak, kind = hbm_peak()
    for w in [int(x) for x in args.c5_ws.split(",")]:
        for m in [int(x) for x in args.c5_ms.split(",")]:
            r = config5_bucket(torch, w=w, m=m, reps=args.steps)
            r.update({"workload": "config5", "frac": r["gbs"] / peak, "peak_gbs": peak,
                      "peak_source": kind})
            print(json.dumps(r), flush=True)
    return 0


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="config2", choices=sorted(WORKLOADS) + ["config5"])
    ap.add_argument("--angle-sets", type=int, default=0,
                    help="angle sets per step per GPU (weak) or in all (strong); "
                         "0: the workload's default (1024 for config 2)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="multi-GPU: weak = batch of angle sets x N, jobs sharded; "
                         "strong = fixed batch, jobs sharded")
    ap.add_argument("--dtype", default=None)
    ap.add_argument("--slices", type=int, default=0,
                    help="split every edge network into 2^k slices (config 4)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-step-seconds", type=float, default=1.0,
                    help="reference arm: CPU seconds per step of the bounded sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-records", action="store_true")
    ap.add_argument("--edge-ids", default=None,
                    help="comma list overriding the workload's edges (e.g. config 4 edge 16)")
    ap.add_argument("--out-json", default=None, help="rank 0 also writes its line here")
    ap.add_argument("--c5-w", type=int, default=30)
    ap.add_argument("--c5-m", type=int, default=16)
    ap.add_argument("--c5-ws", default="20,22,24,26,28,30,31,32")
    ap.add_argument("--c5-ms", default="4,8,16")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    apply_edge_override(args)
    return args


def apply_edge_override(args):
    if args.edge_ids and args.workload in WORKLOADS:
        WORKLOADS[args.workload] = dict(WORKLOADS[args.workload],
                                        edges=[int(x) for x in args.edge_ids.split(",")])


def rank_main(args):
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "config5":
        return run_config5(args)
    return run_gpu(args)


def main_with(args, target):
    """`--gpus N` outside torchrun: spawn the N ranks here (one per GPU)."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        return spawn_ranks(args, target, args.gpus)
    return target(args)


def main(argv=None):
    return main_with(parse_args(argv), rank_main)


if __name__ == "__main__":
    sys.exit(main())
