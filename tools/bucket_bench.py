"""Time one synthetic bucket through qtn_bucket_contract (dev tool).

usage: python tools/bucket_bench.py SPEC [SPEC ...]
SPEC = "P=22;G=21:5:6;T=1"  primary rank 22 (v + 21 vars), a gathered operand
of rank 21 with 5 new variables and 6 of the primary's 11 lowest vars, one
rank-1 table operand on v.  Output rank = 21 + new.
"""
import ctypes as C
import json
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2106_15740_b200 import _native as N  # noqa: E402


def run(spec, reps=5, seed=0):
    kv = dict(x.split("=") for x in spec.split(";"))
    rp = int(kv["P"])
    g = [int(x) for x in kv.get("G", "0:0:0").split(":")]
    rg, gnew, glow = g
    nt = int(kv.get("T", "1"))
    rng = np.random.default_rng(seed)
    v = 0
    pvars = list(range(0, rp))  # v first (MSB); layout decides
    pvars = [v] + list(range(1, rp))
    ops = [pvars]
    newv = list(range(rp, rp + gnew))
    if rg:
        low = pvars[-11:]  # the primary's lowest vars
        shared_low = list(rng.choice(low, size=glow, replace=False))
        rest = [x for x in pvars[1:] if x not in low]
        shared_hi = list(rng.choice(rest, size=rg - 1 - gnew - glow, replace=False))
        gv = [v] + newv + [int(x) for x in shared_hi + shared_low]
        ops.append(gv)
    for _ in range(nt):
        ops.append([v])
    dev = torch.device("cuda")
    datas = [torch.randn(2 << len(o), dtype=torch.float32, device=dev).view(torch.complex64)
             for o in ops]
    ranks = np.asarray([len(o) for o in ops], dtype=np.int32)
    offs = np.zeros(len(ops) + 1, dtype=np.int32)
    offs[1:] = np.cumsum(ranks)
    flat = np.asarray([x for o in ops for x in o], dtype=np.int32)
    ov = np.zeros(64, dtype=np.int32)
    r = C.c_int32()
    N.check(N.lib.qtn_bucket_layout(len(ops), N.i32(ranks), N.i32(offs), N.i32(flat), v,
                                    C.byref(r), N.i32(ov)))
    R = r.value
    out = torch.empty(1 << R, dtype=torch.complex64, device=dev)
    ptrs = (C.c_void_p * len(ops))(*[d.data_ptr() for d in datas])
    flags = np.ones(len(ops), dtype=np.uint8)
    st = torch.cuda.current_stream()

    def go():
        N.check(N.lib.qtn_bucket_contract(len(ops), N.i32(ranks), N.i32(offs), N.i32(flat), ptrs,
                                          N.u8(flags), v, R, N.i32(ov[:R].copy()), 1,
                                          out.data_ptr(), st.cuda_stream))
    for _ in range(2):
        go()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        go()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    alg = 8.0 * (sum(2 << len(o) for o in ops) / 2 + (1 << R))
    t = statistics.median(ts)
    return {"spec": spec, "R": R, "seconds": t, "gbs": alg / t / 1e9}


if __name__ == "__main__":
    for sp in sys.argv[1:]:
        print(json.dumps(run(sp)), flush=True)
