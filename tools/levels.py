"""Per-level bucket statistics of an HBM-executor network (dev tool)."""
import sys
from collections import defaultdict
sys.path.insert(0, ".")
import paper_2106_15740_b200 as Q


def levels(tpl, order, mixed=12):
    live = {k: (tuple(s), 0) for k, s in enumerate(tpl.structure)}
    nid = len(live)
    out = defaultdict(list)
    for v in order.sequence:
        ids = sorted(k for k, (vs, _) in live.items() if v in vs)
        if not ids:
            continue
        uni, lv, ops = [], 0, []
        for k in ids:
            vs, l = live.pop(k)
            ops.append(len(vs))
            lv = max(lv, l)
            for u in vs:
                if u not in uni:
                    uni.append(u)
        uni.remove(v)
        R = len(uni)
        e = lambda r, inp: 16 if (inp or r < mixed) else 8
        alg = sum((16 if k < len(tpl.structure) or r < mixed else 8) << r for k, r in zip(ids, ops)) + (e(R, False) << R)
        out[lv].append((R, ops, alg))
        live[nid] = (tuple(uni), lv + 1)
        nid += 1
    return out


if __name__ == "__main__":
    g = Q.random_regular_graph(1000, 3, 0)
    tpl = Q.energy_template(g, g.edges[int(sys.argv[1]) if len(sys.argv) > 1 else 1058], 5, "zz+diagonal")
    order, rep = Q.rgreedy_order(tpl.line_graph())
    L = levels(tpl, order)
    tot = 0
    for lv in sorted(L):
        b = L[lv]
        alg = sum(x[2] for x in b)
        tot += alg
        big = sorted(b, key=lambda x: -x[2])[:3]
        print(lv, len(b), f"{alg/1e6:.1f}MB", [(x[0], x[1]) for x in big])
    print("total", tot / 1e9, "GB")


def bucket_layouts(tpl, order, min_rank=20):
    """(level, R, op ranks, staging k of the widest non-primary op) for big buckets."""
    live = {k: (tuple(s), 0) for k, s in enumerate(tpl.structure)}
    nid = len(live)
    res = []
    for v in order.sequence:
        ids = sorted(k for k, (vs, _) in live.items() if v in vs)
        if not ids:
            continue
        opv = [live[k][0] for k in ids]
        lv = max(live[k][1] for k in ids)
        for k in ids:
            live.pop(k)
        p = max(range(len(opv)), key=lambda i: (len(opv[i]), -i))
        uni = []
        for vs in opv:
            for u in vs:
                if u not in uni:
                    uni.append(u)
        out = [u for u in uni if u != v and u not in opv[p]] + [u for u in opv[p] if u != v]
        R = len(out)
        if R >= min_rank:
            ks = []
            for i, vs in enumerate(opv):
                if i == p or len(vs) - 1 <= 8:
                    continue
                bits = [R - 1 - out.index(u) for u in vs if u != v]
                ks.append((len(vs), sum(b < 11 for b in bits)))
            res.append((lv, R, [len(x) for x in opv], ks))
        live[nid] = (tuple(out), lv + 1)
        nid += 1
    return res
