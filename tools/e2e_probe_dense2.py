import sys, time, cProfile, pstats, numpy as np
sys.path.insert(0, '.')
import torch
from paper_2505_22631_b200 import dynamics as dyn, workloads
from paper_2505_22631_b200.model import SolverParams
n = 16384
R = int(sys.argv[1]) if len(sys.argv) > 1 else 28
J8 = workloads.sk_dense(n)
g = dyn.DeviceGraph.from_dense(0, J8.astype(np.float64))
params = SolverParams.tuned_for(n, 2, seed=0)
seeds = list(range(R))
phi0 = dyn._initial_phases_host(0, seeds, n)
for _ in range(2): dyn.run_batch(None, params, "maxcut", seeds, steps=1024, graph=g, phi0=phi0)
pr = cProfile.Profile(); pr.enable()
for _ in range(3): dyn.run_batch(None, params, "maxcut", seeds, steps=1024, graph=g, phi0=phi0)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
