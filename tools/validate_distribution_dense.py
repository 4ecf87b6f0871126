"""Noise-on parity of the tensor-core dense kernel: best cuts on a dense +-1 SK graph (n = 1024, 4000 Euler
steps) from `k_dense_umma` (float32 epilogue, device noise) against the CPU oracle (numpy's noise stream)."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
from scipy import stats

import paper_2505_22631_b200 as pkg
from oracle import oracle as O
from paper_2505_22631_b200 import dynamics as dyn, workloads

n, R = 1024, int(sys.argv[1]) if len(sys.argv) > 1 else 84
J8 = workloads.sk_dense(n)
Jf = J8.astype(np.float64)
params = pkg.SolverParams(K=0.05, ks_max=1.0, ks_period=4.0, kn=0.15, h=0.01, t_stop=40.0, seed=0)
g = dyn.DeviceGraph.from_dense(0, Jf)
t0 = time.perf_counter()
b = dyn.run_batch(None, params, "maxcut", list(range(R)), graph=g, want_phases=False)
t_gpu = time.perf_counter() - t0
mask = ~np.eye(n, dtype=bool)
indices = np.broadcast_to(np.arange(n, dtype=np.int64), (n, n))[mask]
data = Jf[mask]
indptr = np.arange(n + 1, dtype=np.int64) * (n - 1)
O.build()
t0 = time.perf_counter()
c = O.simulate(indptr, indices, data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period, kn=params.kn, h=params.h,
               t_stop=params.t_stop, n_states=2, seeds=list(range(50_000, 50_000 + R)), objective="maxcut", threads=O.max_threads())
t_cpu = time.perf_counter() - t0
ks = stats.ks_2samp(b.best_objective, c.best_objective)
print(json.dumps({
    "graph": f"dense +-1 SK n={n}", "steps": b.steps, "kernel": b.kernel,
    "gpu": {"replicas": R, "mean": float(b.best_objective.mean()), "std": float(b.best_objective.std()), "wall_s": t_gpu},
    "cpu_oracle": {"replicas": R, "mean": float(c.best_objective.mean()), "std": float(c.best_objective.std()), "wall_s": t_cpu},
    "ks_2samp": {"statistic": float(ks.statistic), "pvalue": float(ks.pvalue)},
    "mean_difference_in_cpu_std": float((b.best_objective.mean() - c.best_objective.mean()) / c.best_objective.std())}))
