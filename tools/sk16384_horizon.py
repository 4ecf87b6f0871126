"""Error of the tensor-core dense kernel against the oracle fixture, per horizon (calibrates tests/test_fullsize_parity.py)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2505_22631_b200 as pkg
from paper_2505_22631_b200 import dynamics as dyn, workloads

fix = np.load("tests/golden/fullsize_fixtures.npz")
n = 16384
g = dyn.DeviceGraph.from_dense(0, workloads.sk_dense(n).astype(np.float64))
for tag, K, Ns in (("tuned", float(fix["sk16384_tuned_K"]), (1, 2, 3, 5, 10)), ("mild", 0.02, (10,))):
    for N in Ns:
        for prec in ("f64", "f32"):
            p = pkg.SolverParams.tuned_for(n, 2, seed=0, K=K)
            b = dyn.run_batch(None, p, "maxcut", [0], steps=N, graph=g, noise_off=True, precision=prec)
            d = np.abs(b.final_phases[0] - fix[f"sk16384_{tag}_phi_N{N}"])
            d = 2 * np.pi * np.minimum(d, 1 - d)
            print(tag, K, N, prec, b.kernel, "max err rad %.3e" % d.max(), "best", b.best_objective, fix[f"sk16384_{tag}_best_N{N}"])
