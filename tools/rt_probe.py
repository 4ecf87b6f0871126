"""Time one workload of bench.py for several replicas-per-CTA choices of the resident kernel."""
import sys
sys.path.insert(0, '.')
import bench
from paper_2505_22631_b200 import dynamics as dyn
name = sys.argv[1]
shape, J, params, kind, R = bench.load_workload(name)
seeds = list(range(R))
for rt in [int(x) for x in sys.argv[2].split(",")]:
    try:
        for _ in range(2):
            b = dyn.run_batch(J, params, kind, seeds, steps=2048, replicas_per_cta=rt, want_phases=False, want_states=False, want_traces=False)
        print(name, "rt", rt, "-> used", b.replicas_per_cta, "smem", b.smem_bytes, "ms %.2f" % b.device_ms, "upd/s %.3e" % (R * J.nnz * 2048 / (b.device_ms * 1e-3)))
    except Exception as e:
        print(name, "rt", rt, "ERR", str(e)[:100])
