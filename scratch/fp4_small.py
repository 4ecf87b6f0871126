import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
os.environ["OSCB_UMMA_FP4"] = sys.argv[1] if len(sys.argv) > 1 else "1"
import paper_2505_22631_b200 as pkg
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
rng = np.random.default_rng(5)
J = rng.choice([-1.0, 1.0], size=(n, n)); J = np.triu(J, 1); J = J + J.T
Jd = pkg.CouplingMatrix.from_dense(J, storage="dense")
params = pkg.SolverParams(K=0.01, ks_max=1.0, ks_period=0.5, kn=0.2, h=0.01, t_stop=0.05, seed=70)
r = pkg.run_batch(Jd, params, "maxcut", [70], precision="f32", kernel="dense-tc")
print(r.final_phases[0, :8], r.best_objective)
