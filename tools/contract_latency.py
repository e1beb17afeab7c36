"""Latency of the drop-in contract() call (plan + batch + execute) on one network."""
import sys
import time

sys.path.insert(0, ".")
import paper_2106_15740_b200 as Q  # noqa: E402

for n, p, mode in ((100, 2, "zz+diagonal"), (244, 3, "default")):
    g = Q.random_regular_graph(n, 3, 0)
    net = Q.build_energy_network(g, g.edges[0], Q.seeded_angles(p, 0), mode)
    order, _ = Q.rgreedy_order(Q.line_graph(net))
    Q.contract(net, order)
    ts = []
    for _ in range(20):
        t = time.perf_counter()
        v = Q.contract(net, order)
        ts.append(time.perf_counter() - t)
    ts.sort()
    print(n, p, mode, "median ms", round(ts[len(ts) // 2] * 1e3, 3), "min ms", round(ts[0] * 1e3, 3), v)
