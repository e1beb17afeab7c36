"""GPU parity at the configs' full sizes.

* Config 3 default (N=244, p=3, H/CNOT form, widths 13-24): the energy over
  all 366 edge networks against the reference (tests/golden/config3.json,
  every edge contracted by the real qtnsim), complex64 at 1e-5 and
  complex128 at 1e-10 relative, plus every per-edge value.
* Config 5 (synthetic bucket, w = 20..32): `qtn_bucket_contract` against the
  float64 restatement of contraction.py:82-96 (oracle.bucket_sampled) on
  4096 random outputs plus the first and last 4096-output tile, complex128
  and complex64 at w in {20, 24, 28, 30}, complex64 at w = 32, m in {4, 16}.
"""

import ctypes as C

import numpy as np
import pytest

import paper_2106_15740_b200 as Q
import qtn_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,tol,edge_tol", [("complex64", 1e-5, 1e-5),
                                                ("complex128", 1e-10, 1e-10)])
def test_config3_default_all_366_edges(golden, dtype, tol, edge_tol):
    G = golden("config3.json")
    recs = G["modes"]["default"]
    assert len(recs) == 366
    graph = Q.random_regular_graph(G["n"], 3, 0)
    params = Q.QaoaParams(G["gammas"], G["betas"])
    plan = Q.EnergyPlan(graph, G["p"], "default", dtype=dtype)
    assert len(plan.jobs) == 366 and plan.hbm_jobs
    want = sum((1 - r["value"][0]) / 2 for r in recs)
    e = plan.energies(params)[0]
    assert abs(e - want) / abs(want) < tol, (e, want)
    zz = plan.zz_values(params)
    for r in recs:
        w = complex(*r["value"])
        assert abs(zz[r["edge_index"]] - w) <= edge_tol * max(abs(w), 1e-3), r["edge_index"]


def _bucket(torch, w, m, c64, seed):
    """The config-5 bucket of bench.config5_bucket (same seeding)."""
    rng = np.random.default_rng(seed)
    perm = [int(x) for x in rng.permutation(w + 1)]
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    fdt = torch.float32 if c64 else torch.float64
    cdt = torch.complex64 if c64 else torch.complex128
    ops_vars = [perm]
    datas = [torch.randn(4 << w, dtype=fdt, device=dev, generator=g).view(cdt)]
    for _ in range(m):
        ops_vars.append([0] if rng.random() < 0.5 else [0, int(rng.integers(1, w + 1))])
        datas.append(torch.randn(2 << len(ops_vars[-1]), dtype=fdt, device=dev,
                                 generator=g).view(cdt))
    return ops_vars, datas


@pytest.mark.parametrize("w,c64", [(20, False), (20, True), (24, False), (24, True),
                                   (28, False), (28, True), (30, False), (30, True),
                                   (32, True)])
@pytest.mark.parametrize("m", [4, 16])
def test_config5_bucket_sampled(w, c64, m):
    import torch

    from paper_2106_15740_b200 import _native as N

    free, _ = torch.cuda.mem_get_info()
    need = (3 << w) * (8 if c64 else 16) + (1 << 30)
    if need > free:
        pytest.skip(f"needs {need >> 30} GiB, {free >> 30} GiB free")
    seed = 100 * w + m
    ops_vars, datas = _bucket(torch, w, m, c64, seed)
    ranks = np.asarray([len(v) for v in ops_vars], dtype=np.int32)
    offs = np.zeros(len(ranks) + 1, dtype=np.int32)
    offs[1:] = np.cumsum(ranks)
    flat = np.asarray([x for v in ops_vars for x in v], dtype=np.int32)
    ov = np.zeros(w, dtype=np.int32)
    r = C.c_int32()
    N.check(N.lib.qtn_bucket_layout(len(ranks), N.i32(ranks), N.i32(offs), N.i32(flat), 0,
                                    C.byref(r), N.i32(ov)))
    assert r.value == w and sorted(ov.tolist()) == list(range(1, w + 1))
    cdt = torch.complex64 if c64 else torch.complex128
    out = torch.empty(1 << w, dtype=cdt, device="cuda")
    ptrs = (C.c_void_p * len(datas))(*[d.data_ptr() for d in datas])
    flags = np.full(len(datas), 1 if c64 else 0, dtype=np.uint8)
    N.check(N.lib.qtn_bucket_contract(len(ranks), N.i32(ranks), N.i32(offs), N.i32(flat), ptrs,
                                      N.u8(flags), 0, w, N.i32(ov), 1 if c64 else 0,
                                      out.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    rng = np.random.default_rng(seed + 1)
    outs = np.unique(np.concatenate([rng.integers(0, 1 << w, 4096, dtype=np.int64),
                                     np.arange(4096, dtype=np.int64),
                                     (1 << w) - 1 - np.arange(4096, dtype=np.int64)]))

    def fetch(t, idx):
        return datas[t][torch.from_numpy(idx).cuda()].cpu().numpy()

    want = O.bucket_sampled(outs, ov.tolist(), ops_vars, fetch)
    got = out[torch.from_numpy(outs).cuda()].cpu().numpy().astype(np.complex128)
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err < (1e-5 if c64 else 1e-12), (w, m, c64, err)
    del datas, out
    torch.cuda.empty_cache()
