"""The fused row-sharded dense run across PROCESSES: two ranks, one process each, both on cuda:0,
their exchange blocks mapped into each other with CUDA IPC (the path a torchrun job takes on an
8-GPU node, minus NVLink).  Two processes time-slice one GPU, so the kernels advance a step per
context switch -- the run is kept short and the whole thing sits under a hard timeout."""
import os
import pickle
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = Path(__file__).resolve().parent


def test_two_processes_one_gpu_match_single_handle(tmp_path):
    import paper_2505_22631_b200 as pkg
    from paper_2505_22631_b200 import _native, dynamics
    assert _native.device_count() > 0, "no CUDA device: " + _native.last_error()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    steps = 24
    env = dict(os.environ, FUSED_IPC_STEPS=str(steps))
    procs = [subprocess.Popen([sys.executable, str(HERE / "fused_ipc_worker.py"), str(r), "2", str(port), str(tmp_path)], env=env)
             for r in range(2)]
    try:
        for p in procs:
            assert p.wait(timeout=240) == 0
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    got = [pickle.load(open(tmp_path / f"rank{r}.pkl", "rb")) for r in range(2)]
    sys.path.insert(0, str(HERE))
    from fused_ipc_worker import sk_graph
    n = 512
    J = sk_graph(n, 5)
    old = dynamics.DENSE_DEVICE_MIN_N
    dynamics.DENSE_DEVICE_MIN_N = 0
    try:
        Jd = pkg.CouplingMatrix.from_dense(J, storage="dense")
        params = pkg.SolverParams(K=0.02, ks_max=1.0, ks_period=0.5, kn=0.2, h=0.01, t_stop=1.2, seed=40)
        want = pkg.run_batch(Jd, params, "maxcut", [40, 41], precision="f32", kernel="dense-tc", steps=steps)
    finally:
        dynamics.DENSE_DEVICE_MIN_N = old
    for b in got:
        assert np.array_equal(b.final_phases, want.final_phases)
        assert np.array_equal(b.best_states, want.best_states)
        assert np.array_equal(b.best_objective, want.best_objective)
        assert np.array_equal(b.best_trace, want.best_trace)
        assert np.array_equal(b.energy, want.energy)
