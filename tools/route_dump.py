import sys; sys.path.insert(0,'.')
import paper_2106_15740_b200 as Q
from paper_2106_15740_b200.contraction import PlanBatch
g=Q.random_regular_graph(244,3,0)
jobs=Q.plan_edges(g,3,'default',list(range(366)),dtype='complex64')
try:
    b=PlanBatch([j.plan for j in jobs])
except Exception as e:
    print("ERR", e)
