"""Noise-on parity at full size: best cuts of the GPU solver (float32 persistent kernel, device Philox
noise) against the CPU oracle (the reference algorithm with numpy's own noise stream) on the G22-shape
graph, whole default schedule.  Two-sample Kolmogorov-Smirnov + Mann-Whitney on best_objective.

    python tools/validate_distribution.py [gpu_replicas] [cpu_replicas] [workload] > report.json
"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
from scipy import stats

import bench
from oracle import oracle as O
from paper_2505_22631_b200 import dynamics as dyn

R_gpu = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
R_cpu = int(sys.argv[2]) if len(sys.argv) > 2 else 64
workload = sys.argv[3] if len(sys.argv) > 3 else "G22x1024"
shape, J, params, kind, _ = bench.load_workload(workload)
t0 = time.perf_counter()
g = dyn.run_batch(J, params, kind, list(range(R_gpu)), want_phases=False, want_states=False)
t_gpu = time.perf_counter() - t0
O.build()
t0 = time.perf_counter()
c = O.simulate(J.indptr, J.indices, J.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period, kn=params.kn,
               h=params.h, t_stop=params.t_stop, n_states=params.n_states, seeds=list(range(10_000, 10_000 + R_cpu)), objective=kind,
               threads=O.max_threads())
t_cpu = time.perf_counter() - t0
ks = stats.ks_2samp(g.best_objective, c.best_objective)
mw = stats.mannwhitneyu(g.best_objective, c.best_objective, alternative="two-sided")
print(json.dumps({
    "graph": f"{shape}-shape n={J.n} nnz={J.nnz} N={params.n_states} objective={kind} (synthetic)", "params": {"K": params.K, "ks_max": params.ks_max, "kn": params.kn,
                                                                          "h": params.h, "t_stop": params.t_stop},
    "steps": g.steps,
    "gpu": {"replicas": R_gpu, "kernel": g.kernel, "mean": float(g.best_objective.mean()), "std": float(g.best_objective.std()),
            "min": float(g.best_objective.min()), "max": float(g.best_objective.max()), "wall_s": t_gpu},
    "cpu_oracle": {"replicas": R_cpu, "mean": float(c.best_objective.mean()), "std": float(c.best_objective.std()),
                   "min": float(c.best_objective.min()), "max": float(c.best_objective.max()), "wall_s": t_cpu,
                   "threads": O.max_threads()},
    "ks_2samp": {"statistic": float(ks.statistic), "pvalue": float(ks.pvalue)},
    "mannwhitneyu": {"statistic": float(mw.statistic), "pvalue": float(mw.pvalue)},
    "mean_difference_in_cpu_std": float((g.best_objective.mean() - c.best_objective.mean()) / c.best_objective.std()),
}))
