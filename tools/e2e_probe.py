import sys, time, numpy as np
sys.path.insert(0, '.')
import torch
import bench
from paper_2505_22631_b200 import dynamics as dyn
shape, J, params, kind, R = bench.load_workload("G22x1024")
seeds = list(range(R))
g = dyn.device_graph(J, 0)
phi0 = dyn._initial_phases_host(0, seeds, J.n)
def t(label, **kw):
    for _ in range(2): dyn.run_batch(J, params, kind, seeds, steps=2048, **kw)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(4): b = dyn.run_batch(J, params, kind, seeds, steps=2048, **kw)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 4
    print(label, "wall %.2f ms  device %.2f ms" % (dt * 1e3, b.device_ms))
t("no io", want_phases=False, want_states=False, want_traces=False)
t("phi0 in", phi0=phi0, want_phases=False, want_states=False, want_traces=False)
t("phases out", want_phases=True, want_states=False, want_traces=False)
t("states out", want_phases=False, want_states=True, want_traces=False)
t("traces out", want_phases=False, want_states=False, want_traces=True)
t("all", phi0=phi0)
