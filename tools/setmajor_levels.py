import sys; sys.path.insert(0,'.')
import numpy as np, paper_2106_15740_b200 as Q
g=Q.random_regular_graph(100,3,0)
plan=Q.EnergyPlan(g,2,"zz+diagonal",dtype="complex64")
plan.energies(np.random.default_rng(0).uniform(0,3,(1024,4)))
