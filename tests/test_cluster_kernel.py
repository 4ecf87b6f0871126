"""Latency mode (csrc/oscb_cluster.cuh, kernel "cluster"): one replica integrated by a cluster of 8
CTAs exchanging the (cos, sin) pairs through distributed shared memory.  Checked against the float64
streaming kernel / the oracle over a short noise-free horizon, through the result contract, and
against the persistent kernel statistically (the summation order inside a row differs, so noisy
float32 trajectories agree in distribution, not bit for bit)."""
import math

import numpy as np
import pytest

from conftest import circ_dist_rad, random_graph_arrays

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2505_22631_b200 as p
    from paper_2505_22631_b200 import _native
    assert _native.device_count() > 0, "no CUDA device: " + _native.last_error()
    return p


def g1(pkg):
    from paper_2505_22631_b200 import workloads
    n, (u, v, w), N, kind = workloads.shape_graph("G1")
    return pkg.CouplingMatrix.from_edges(n, (u, v, w)), pkg.SolverParams.tuned_for(n, 2, seed=0, K=0.2, ks_max=1.0, kn=0.15)


def test_noise_free_short_horizon_vs_float64_and_oracle(pkg, oracle):
    J, params = g1(pkg)
    seeds = [0, 1, 2]
    a = pkg.run_batch(J, params, "maxcut", seeds, kernel="cluster", steps=20, noise_off=True)
    ref = pkg.run_batch(J, params, "maxcut", seeds, kernel="stream", precision="f64", steps=20, noise_off=True)
    assert a.kernel == "cluster"
    assert circ_dist_rad(a.final_phases, ref.final_phases).max() <= 1e-4            # N = 20 steps, float32
    want = oracle.simulate(J.indptr, J.indices, J.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period, kn=0.0,
                           h=params.h, t_stop=20 * params.h, n_states=2, seeds=seeds, objective="maxcut")
    assert circ_dist_rad(a.final_phases, want.final_phases).max() <= 1e-4
    assert np.abs(a.energy - want.energy).max() <= 1e-3 * J.nnz
    assert np.array_equal(a.trace_t, want.trace_t)
    # scored states of identical phases: the initial sample is bit-exact (same Philox phases, same threshold rule)
    assert np.array_equal(a.best_trace[:, 0], want.best_trace[:, 0])


@pytest.mark.parametrize("weights", [(1.0,), (1.0, -1.0), (3.0, -2.0, 1.0)])
def test_result_contract_and_scoring(pkg, weights):
    n = 200
    iu, iv, w = random_graph_arrays(n, 0.1, seed=5, weights=weights)
    J = pkg.CouplingMatrix.from_edges(n, (iu, iv, w))
    params = pkg.SolverParams.tuned_for(n, 2, seed=4, t_stop=8.0)
    res = pkg.run(J, params, "maxcut", kernel="cluster")
    assert res.steps_executed == math.ceil(params.t_stop / params.h)
    p = res.final_phases.phases
    assert p.min() >= 0.0 and p.max() < 1.0
    piu, pjv, pw = J.pairs()
    s = res.best_assignment.states
    assert res.best_objective == float((pw * (s[piu] != s[pjv])).sum())
    ts = [t for t, _, _ in res.energy_trace]
    assert ts[0] == 0.0 and all(b > a for a, b in zip(ts, ts[1:]))
    sched = pkg.KsSchedule(params.ks_max, params.ks_period)
    assert all(ks == sched.value(t) for t, _, ks in res.energy_trace)
    assert all(b >= a for a, b in zip(res.best_trace, res.best_trace[1:])) and res.best_trace[-1] == res.best_objective
    # every scored sample really is a cut of the graph: the trace energy of the final sample equals the host formula
    final_energy = float((pw * np.cos(2 * np.pi * (p[piu] - p[pjv]))).sum())
    assert abs(res.energy_trace[-1][1] - final_energy) <= 1e-4 * max(1.0, np.abs(pw).sum())
    # batch == solo, run == rerun (each replica has its own cluster)
    b3 = pkg.run_batch(J, params, "maxcut", [4, 5, 6], kernel="cluster")
    b1 = pkg.run_batch(J, params, "maxcut", [5], kernel="cluster")
    assert np.array_equal(b3.final_phases[1], b1.final_phases[0]) and b3.best_objective[1] == b1.best_objective[0]
    assert np.array_equal(pkg.run_batch(J, params, "maxcut", [4, 5, 6], kernel="cluster").final_phases, b3.final_phases)
    assert np.array_equal(b3.final_phases[0], res.final_phases.phases)


def test_statistics_match_the_persistent_kernel(pkg):
    """Noise on: best cuts of 16 seeds from the cluster kernel and from the persistent kernel (same noise
    source, different summation order) have the same mean within 1 %; a target is hit at the same time scale."""
    J, params = g1(pkg)
    seeds = list(range(16))
    c = pkg.run_batch(J, params, "maxcut", seeds, kernel="cluster", steps=3000, target=11000.0)
    r = pkg.run_batch(J, params, "maxcut", seeds, kernel="resident", steps=3000, target=11000.0)
    assert c.kernel == "cluster" and r.kernel == "resident"
    piu, pjv, pw = J.pairs()
    s = c.best_states.astype(np.int64)
    assert np.array_equal((pw[None, :] * (s[:, piu] != s[:, pjv])).sum(axis=1), c.best_objective)
    assert abs(c.best_objective.mean() - r.best_objective.mean()) <= 0.01 * r.best_objective.mean()
    assert (c.first_hit_step >= 0).all() and abs(np.median(c.first_hit_step) - np.median(r.first_hit_step)) <= 0.5 * np.median(r.first_hit_step) + 50


def test_auto_selection_and_limits(pkg):
    J, params = g1(pkg)
    assert pkg.run_batch(J, params, "maxcut", [0], steps=50).kernel == "cluster"           # few replicas: latency mode
    assert pkg.run_batch(J, params, "maxcut", list(range(64)), steps=50).kernel == "resident"  # many: throughput mode
    assert pkg.run_batch(J, params, "maxcut", [0], steps=50, precision="f64").kernel != "cluster"
    iu, iv, w = random_graph_arrays(100, 0.2, seed=1, weights=(0.37, -1.2))
    Jw = pkg.CouplingMatrix.from_edges(100, (iu, iv, w))
    pw = pkg.SolverParams.tuned_for(100, 2, seed=0, t_stop=1.0)
    assert pkg.run_batch(Jw, pw, "maxcut", [0]).kernel == "resident"                       # non-integer couplings
    with pytest.raises(ValueError):
        pkg.run_batch(Jw, pw, "maxcut", [0], kernel="cluster")
    with pytest.raises(ValueError):
        pkg.run_batch(J, pkg.SolverParams.tuned_for(800, 3, seed=0, t_stop=1.0), "coloring", [0], kernel="cluster")


def test_numerical_error(pkg):
    J, _ = g1(pkg)
    bad = pkg.SolverParams(K=1e38, ks_max=0.0, ks_period=10.0, kn=0.0, h=1.0, t_stop=3.0)
    with pytest.raises(pkg.NumericalError) as err:
        pkg.run(J, bad, "maxcut", kernel="cluster")
    assert "oscillator" in str(err.value) and "step" in str(err.value)


def test_best_cut_distribution_matches_reference_oracle(pkg, oracle):
    """Noise ON, the cluster kernel's device Philox stream vs the reference's numpy stream (replayed by the
    oracle): best cuts and final-state cuts over 96 seeds agree in distribution (two-sample KS)."""
    from scipy import stats
    n = 96
    iu, iv, w = random_graph_arrays(n, 0.12, seed=77, weights=(1.0,))
    J = pkg.CouplingMatrix.from_edges(n, (iu, iv, w))
    params = pkg.SolverParams(K=0.2, ks_max=1.0, ks_period=3.0, kn=0.15, h=0.01, t_stop=9.0, seed=1000)
    seeds = [params.seed + r for r in range(96)]
    want = oracle.simulate(J.indptr, J.indices, J.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period, kn=params.kn,
                           h=params.h, t_stop=params.t_stop, n_states=2, seeds=seeds, objective="maxcut", threads=oracle.max_threads())
    got = pkg.run_batch(J, params, "maxcut", seeds, kernel="cluster")
    assert got.kernel == "cluster"
    assert stats.ks_2samp(got.best_objective, want.best_objective).pvalue > 0.01
    assert abs(got.best_objective.mean() - want.best_objective.mean()) < 0.6 * (want.best_objective.std() + 0.5)
    iu_, jv_, w_ = J.pairs()
    _, cut_got = oracle.score(got.final_phases, 2, iu_, jv_, w_, True)
    _, cut_want = oracle.score(want.final_phases, 2, iu_, jv_, w_, True)
    assert stats.ks_2samp(cut_got, cut_want).pvalue > 0.01
