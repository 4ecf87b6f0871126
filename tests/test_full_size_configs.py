"""BASELINE.json configs[2], [3], [4] at their full sizes, checked through size-independent
properties (the oracle cannot run these sizes in seconds): phase containment, best objective ==
objective recomputed on the host from the best states (the reference recomputes it the same way,
dynamics.py:416-421), monotone best trace, kernels agreeing with each other.  configs[1] at full
size is in test_gpu_parity.py::test_full_size_g22_properties."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2505_22631_b200 as p
    from paper_2505_22631_b200 import _native
    assert _native.device_count() > 0, "no CUDA device: " + _native.last_error()
    return p


def circ(a, b):
    d = np.abs(a - b)
    return 2 * np.pi * np.minimum(d, 1 - d)


def test_flat200_coloring_4096_replicas(pkg):
    """configs[2]: SATLIB flat200-479 shape, N = 3 OPM, 4096 replicas."""
    from paper_2505_22631_b200 import workloads
    n, (u, v, w), N, kind = workloads.shape_graph("flat200")
    assert (n, N, kind) == (200, 3, "coloring")
    J = pkg.CouplingMatrix.from_edges(n, (u, v, w))
    params = pkg.SolverParams.tuned_for(n, 3, seed=0)
    b = pkg.run_batch(J, params, kind, list(range(4096)), steps=600)
    assert b.kernel == "lowdeg"
    assert b.final_phases.min() >= 0.0 and b.final_phases.max() < 1.0
    piu, pjv, _ = J.pairs()
    s = b.best_states.astype(np.int64)
    assert s.max() <= 2
    conflicts = (s[:, piu] == s[:, pjv]).sum(axis=1).astype(np.float64)
    assert np.array_equal(conflicts, b.best_objective)
    assert np.all(np.diff(b.best_trace, axis=1) <= 0)                 # conflicts only ever improve downwards
    assert b.best_objective.min() <= 0.05 * len(piu)                 # annealing is doing its job after 600 steps
    # the thresholds of the final phases agree with the reference rule (model.py:411-416)
    st, obj = pkg.score_phases(J, b.final_phases[:64], 3, "coloring")
    k = np.rint(b.final_phases[:64] * 3).astype(np.int64) % 3
    near_tie = np.abs(b.final_phases[:64] * 3 - np.rint(b.final_phases[:64] * 3)) > 0.499
    assert np.array_equal(st[~near_tie], k[~near_tie])


def test_g81_shape_20000_nodes(pkg):
    """configs[3]: 100 x 200 torus with +-1 weights (20000 oscillators); the persistent kernel and the
    streaming kernel integrate the same replicas to the same phases over a short horizon."""
    from paper_2505_22631_b200 import workloads
    n, (u, v, w), N, kind = workloads.shape_graph("G81")
    assert n == 20000 and len(u) == 40000
    J = pkg.CouplingMatrix.from_edges(n, (u, v, w))
    params = pkg.SolverParams.tuned_for(n, 2, seed=0)
    seeds = list(range(8))
    a = pkg.run_batch(J, params, kind, seeds, steps=20, kernel="resident", noise_off=True)
    b = pkg.run_batch(J, params, kind, seeds, steps=20, kernel="stream", noise_off=True)
    assert a.kernel == "resident" and b.kernel == "stream"
    assert circ(a.final_phases, b.final_phases).max() <= 1e-4       # N = 20 steps, float32
    full = pkg.run_batch(J, params, kind, seeds, steps=400)
    piu, pjv, pw = J.pairs()
    s = full.best_states.astype(np.int64)
    recomputed = (pw[None, :] * (s[:, piu] != s[:, pjv])).sum(axis=1)
    assert np.array_equal(recomputed, full.best_objective)
    assert np.all(np.diff(full.best_trace, axis=1) >= 0)
    assert full.final_phases.min() >= 0.0 and full.final_phases.max() < 1.0


def test_sk_16384_dense_tensor_core(pkg):
    """configs[4]: dense +-1 SK graph, 16384 oscillators, on the tensor-core kernel: the cut of the
    best states recomputed on the host from J equals the in-kernel objective; 10 noise-free steps
    agree with the SIMT dense path within 1e-4 rad."""
    from paper_2505_22631_b200 import dynamics as dyn, workloads
    n = 16384
    J8 = workloads.sk_dense(n)
    g = dyn.DeviceGraph.from_dense(0, J8.astype(np.float64))
    try:
        params = pkg.SolverParams.tuned_for(n, 2, seed=0)
        seeds = [0, 1]
        b = dyn.run_batch(None, params, "maxcut", seeds, steps=60, graph=g)
        assert b.kernel == "dense-tc"
        assert b.final_phases.min() >= 0.0 and b.final_phases.max() < 1.0
        Jf = J8.astype(np.float32)
        for r in range(2):
            sgn = 1.0 - 2.0 * b.best_states[r].astype(np.float32)       # spins +-1
            # cut = sum_{i<j} J_ij [s_i != s_j] = (sum_{i<j} J_ij - sum_{i<j} J_ij s_i s_j) / 2
            quad = float(sgn @ (Jf @ sgn)) / 2.0                         # exact: integers below 2^24 per row
            total = float(J8.sum(dtype=np.int64)) / 2.0
            assert (total - quad) / 2.0 == b.best_objective[r]
        assert np.all(np.diff(b.best_trace, axis=1) >= 0)
        # the call above streamed J as packed e2m1 tiles (<= 12 replicas); the int8 stream must give the same bits
        os.environ["OSCB_UMMA_FP4"] = "0"
        try:
            b8 = dyn.run_batch(None, params, "maxcut", seeds, steps=60, graph=g)
        finally:
            os.environ.pop("OSCB_UMMA_FP4", None)
        assert g.tc_stream(2, len(seeds)) == (4, 12)
        assert np.array_equal(b8.final_phases, b.final_phases) and np.array_equal(b8.best_states, b.best_states)
        assert np.array_equal(b8.best_objective, b.best_objective) and np.array_equal(b8.energy, b.energy)
        # (K = 1 on 16384 all-to-all couplings moves a phase by ~1 turn per step -- any two float32
        # evaluations decorrelate within a few steps; the comparison runs in the contractive regime)
        mild = pkg.SolverParams.tuned_for(n, 2, seed=0, K=0.02)
        tc = dyn.run_batch(None, mild, "maxcut", seeds, steps=10, graph=g, noise_off=True)
        simt = dyn.run_batch(None, mild, "maxcut", seeds, steps=10, graph=g, noise_off=True, kernel="stream")
        assert tc.kernel == "dense-tc" and simt.kernel == "stream"
        assert circ(tc.final_phases, simt.final_phases).max() <= 1e-4   # N = 10 steps, float32 epilogue
        assert np.array_equal(tc.best_objective, simt.best_objective)
    finally:
        g.close()
