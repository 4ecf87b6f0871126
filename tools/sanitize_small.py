"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2505_22631_b200 as pkg
from paper_2505_22631_b200 import dynamics, workloads

which = sys.argv[1:] or ["resident", "cluster", "stream", "dense-tc"]
u, v, w = workloads.random_gnm(128, 700, seed=1, weights=(1.0,))
J = pkg.CouplingMatrix.from_edges(128, (u, v, w))
p = pkg.SolverParams.tuned_for(128, 2, seed=0, t_stop=0.6)
if "resident" in which:
    b = pkg.run_batch(J, p, "maxcut", list(range(20)), kernel="resident")
    print("resident", b.best_objective.max())
    c3 = pkg.run_batch(J, pkg.SolverParams.tuned_for(128, 3, seed=0, t_stop=0.6), "coloring", list(range(20)), kernel="resident")
    print("resident N=3", c3.best_objective.min())
if "cluster" in which:
    b = pkg.run_batch(J, p, "maxcut", [0, 1], kernel="cluster")
    print("cluster", b.best_objective.max())
if "stream" in which:
    b = pkg.run_batch(J, p, "maxcut", [0, 1, 2], kernel="stream", precision="f64")
    print("stream", b.best_objective.max())
if "dense-tc" in which:
    rng = np.random.default_rng(3)
    U = np.triu(rng.choice(np.array([-1.0, 1.0]), size=(300, 300)), 1)
    g = dynamics.DeviceGraph.from_dense(0, U + U.T)
    b = pkg.run_batch(None, pkg.SolverParams(K=0.02, ks_max=1.0, ks_period=0.5, kn=0.1, h=0.01, t_stop=0.3, seed=0), "maxcut", [0, 1, 2], graph=g)
    print("dense-tc", b.kernel, b.best_objective.max())
    g.close()
