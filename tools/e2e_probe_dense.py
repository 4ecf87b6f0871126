"""Where the wall time of a dense tensor-core call goes beyond the kernel (SK 16384)."""
import sys, time, numpy as np
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
def t(label, **kw):
    for _ in range(2): dyn.run_batch(None, params, "maxcut", seeds, steps=1024, graph=g, **kw)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(3): b = dyn.run_batch(None, params, "maxcut", seeds, steps=1024, graph=g, **kw)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 3
    print("%-12s wall %.2f ms  device %.2f ms  launches %d" % (label, dt * 1e3, b.device_ms, b.kernel_launches))
t("no io", want_phases=False, want_states=False, want_traces=False)
t("phi0 in", phi0=phi0, want_phases=False, want_states=False, want_traces=False)
t("phases out", want_phases=True, want_states=False, want_traces=False)
t("states out", want_phases=False, want_states=True, want_traces=False)
t("traces out", want_phases=False, want_states=False, want_traces=True)
t("all", phi0=phi0)
