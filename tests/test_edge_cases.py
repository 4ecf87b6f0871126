"""Edge cases of the solver path on the GPU: empty and tiny graphs, isolated oscillators, a star
whose hub exceeds the persistent kernel's row limit, more oscillators than the persistent kernel
holds, ragged replica counts -- each checked against the oracle (noise-free float64) or through the
result contract.  The reference's behaviour for these inputs: dynamics.py:333-431 (n >= 1, any CSR)."""
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


def check_vs_oracle(pkg, oracle, J, params, kind, seeds, kernels=("stream", "resident"), tol=1e-9):
    want = oracle.simulate(J.indptr, J.indices, J.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period,
                           kn=0.0, h=params.h, t_stop=params.t_stop, n_states=params.n_states, seeds=seeds, objective=kind)
    for kernel in kernels:
        got = pkg.run_batch(J, params, kind, seeds, precision="f64", kernel=kernel, noise_off=True)
        assert got.kernel == kernel
        assert circ(got.final_phases, want.final_phases).max() <= tol, kernel
        assert np.array_equal(got.best_objective, want.best_objective), kernel
        assert np.array_equal(got.best_states.astype(np.int64), want.best_states), kernel
        assert np.array_equal(got.best_trace, want.best_trace), kernel


def test_single_oscillator_and_empty_graph(pkg, oracle):
    params = pkg.SolverParams(K=1.0, ks_max=1.0, ks_period=1.0, kn=0.0, h=0.01, t_stop=1.0, seed=1)
    one = pkg.CouplingMatrix.from_edges(1, [])
    check_vs_oracle(pkg, oracle, one, params, "maxcut", [1, 2, 3])
    empty = pkg.CouplingMatrix.from_edges(37, [])
    check_vs_oracle(pkg, oracle, empty, params, "maxcut", [5])
    r = pkg.run(empty, pkg.SolverParams.tuned_for(37, 2, seed=0, t_stop=2.0))
    assert r.best_objective == 0.0 and r.steps_executed == 200 and len(r.energy_trace) >= 2
    col = pkg.run(empty, pkg.SolverParams.tuned_for(37, 3, seed=0, t_stop=2.0), "coloring")
    assert col.best_objective == 0.0


def test_isolated_oscillators_and_ragged_replicas(pkg, oracle):
    # 3 components + isolated nodes; replica counts that do not fill a tile
    edges = [(0, 1, 1.0), (1, 2, -2.0), (4, 5, 1.0), (7, 8, 3.0), (8, 9, 1.0), (7, 9, 1.0)]
    J = pkg.CouplingMatrix.from_edges(13, edges)
    params = pkg.SolverParams(K=0.5, ks_max=1.5, ks_period=0.8, kn=0.0, h=0.01, t_stop=2.0, seed=3)
    for R in (1, 3, 9, 33):
        check_vs_oracle(pkg, oracle, J, params, "maxcut", list(range(100, 100 + R)))
    check_vs_oracle(pkg, oracle, J, pkg.SolverParams(K=0.5, ks_max=1.5, ks_period=0.8, kn=0.0, h=0.01, t_stop=2.0, n_states=4, seed=3),
                    "coloring", [1, 2, 3, 4, 5])


def test_star_hub_beyond_the_resident_row_limit(pkg, oracle):
    """A hub of degree 1499 (> 1020 neighbours per row): the persistent kernel declines; auto takes the
    cluster kernel (a row is split over 8 lanes there, any degree) or the streaming kernel; the float64
    streaming run still matches the oracle."""
    n = 1500
    J = pkg.CouplingMatrix.from_edges(n, [(0, j, 1.0) for j in range(1, n)])
    params = pkg.SolverParams(K=0.001, ks_max=1.0, ks_period=1.0, kn=0.0, h=0.01, t_stop=0.5, seed=2)
    check_vs_oracle(pkg, oracle, J, params, "maxcut", [2, 3], kernels=("stream",))
    auto = pkg.run_batch(J, params, "maxcut", [2, 3], precision="f32")
    assert auto.kernel in ("cluster", "stream")
    assert circ(auto.final_phases, pkg.run_batch(J, params, "maxcut", [2, 3], precision="f64", kernel="stream").final_phases).max() <= 1e-4
    with pytest.raises(ValueError):
        pkg.run_batch(J, params, "maxcut", [2, 3], kernel="resident")


def test_more_oscillators_than_the_resident_kernel_holds(pkg):
    """n = 70000 ring (> 60000): auto uses the streaming kernel; the result contract holds and a
    noise-free float32 run agrees with the float64 run over a short horizon."""
    n = 70000
    u = np.arange(n)
    J = pkg.CouplingMatrix.from_edges(n, (u, (u + 1) % n, np.ones(n)))
    params = pkg.SolverParams.tuned_for(n, 2, seed=0)
    a = pkg.run_batch(J, params, "maxcut", [0, 1], precision="f32", steps=20, noise_off=True)
    b = pkg.run_batch(J, params, "maxcut", [0, 1], precision="f64", steps=20, noise_off=True)
    assert a.kernel == "stream" and b.kernel == "stream"
    assert circ(a.final_phases, b.final_phases).max() <= 1e-4
    full = pkg.run_batch(J, params, "maxcut", [0, 1], steps=300)
    piu, pjv, pw = J.pairs()
    s = full.best_states.astype(np.int64)
    assert np.array_equal((pw[None, :] * (s[:, piu] != s[:, pjv])).sum(axis=1), full.best_objective)
    assert full.final_phases.min() >= 0.0 and full.final_phases.max() < 1.0


def test_many_replicas_one_call(pkg):
    """4100 replicas of a small graph in one call (more tiles than SMs, last tile ragged): replica r
    equals the solo run with its seed."""
    rng = np.random.default_rng(0)
    iu, jv = np.triu_indices(24, 1)
    keep = rng.random(len(iu)) < 0.3
    J = pkg.CouplingMatrix.from_edges(24, (iu[keep], jv[keep], np.ones(keep.sum())))
    params = pkg.SolverParams.tuned_for(24, 2, seed=7, t_stop=3.0)
    R = 4100
    seeds = [(7 + r) % 2**64 for r in range(R)]
    # float64 parity mode keeps the reference's CSR summation order whatever the tile shape, so the
    # reference's contract "batched == solo" (test_dynamics.py:257-267) holds bit for bit ...
    allr = pkg.run_batch(J, params, "maxcut", seeds, precision="f64")
    for r in (0, 1, 2047, 4096, 4099):
        solo = pkg.run_batch(J, params, "maxcut", [seeds[r]], precision="f64")
        assert np.array_equal(solo.final_phases[0], allr.final_phases[r])
        assert solo.best_objective[0] == allr.best_objective[r]
        assert np.array_equal(solo.best_states[0], allr.best_states[r])
    # ... and in float32 throughput mode for equal tile shapes (the neighbour order inside a row follows
    # the tile shape, so different shapes differ in the last bits)
    all32 = pkg.run_batch(J, params, "maxcut", seeds, precision="f32")
    part = pkg.run_batch(J, params, "maxcut", seeds[4096:], precision="f32", replicas_per_cta=all32.replicas_per_cta)
    assert np.array_equal(part.final_phases, all32.final_phases[4096:])
    assert np.array_equal(part.best_objective, all32.best_objective[4096:])
