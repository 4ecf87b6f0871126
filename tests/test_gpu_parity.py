"""GPU parity tests: the CUDA path, called through the C ABI (liboscb.so via the package's
ctypes layer), against the CPU oracle and the committed golden vectors of the reference.

Bars (north_star): integer/index work bit-exact (initial phases, thresholds, cut/conflict
counts); noise-free trajectories within 1e-4 rad after the stated N steps; noise-on results
agree in distribution over >= 64 seeds."""
import math

import numpy as np
import pytest

from conftest import circ_dist_rad, coupling_from_golden, graph_from_golden, params_from_row, random_graph_arrays

pytestmark = pytest.mark.gpu

KERNELS = ["stream", "resident", "resident-generic"]


@pytest.fixture(scope="module")
def pkg():
    import paper_2505_22631_b200 as p
    from paper_2505_22631_b200 import _native
    assert _native.device_count() > 0, "no CUDA device: " + _native.last_error()
    return p


def make_coupling(pkg, n, iu, iv, w):
    return pkg.CouplingMatrix.from_edges(n, (np.asarray(iu), np.asarray(iv), np.asarray(w, dtype=float)))


# ------------------------------------------------------------------------------------------
def test_initial_phases_bit_exact(pkg, oracle, golden):
    for s, want in zip(golden["init_seeds"], golden["init_phases"]):
        got = pkg.NoiseSource(int(s)).initial_phases(want.shape[0])
        assert np.array_equal(got, want)
    for n in (1, 2, 3, 4, 5, 800, 2001):
        assert np.array_equal(pkg.NoiseSource(42).initial_phases(n), oracle.initial_phases(42, n))


def test_step_known_answers(pkg, golden):
    from paper_2505_22631_b200.dynamics import _step_raw
    J = coupling_from_golden(golden, "pair2")
    out = _step_raw(J, np.array([[0.0, 0.25]]), None, 1.0, 0.0, 0.1, 0.0, 2, "f64", None)[0]
    assert out == pytest.approx([0.9, 0.35], abs=1e-12)          # reference test_dynamics.py:143-154
    J = coupling_from_golden(golden, "ring5")
    out = _step_raw(J, golden["ring5_phi"][None], None, 1.3, 0.935, 0.01, 0.0, 3, "f64", None)[0]
    assert np.abs(out - golden["ring5_out"]).max() <= 1e-14
    out32 = _step_raw(J, golden["ring5_phi"][None], None, 1.3, 0.935, 0.01, 0.0, 3, "f32", None)[0]
    assert circ_dist_rad(out32, golden["ring5_out"]).max() <= 2e-6
    # identity step: K acc = 0 and ks = 0 leaves phases unchanged
    out = _step_raw(J, golden["ring5_phi"][None], None, 1e-300, 0.0, 0.01, 0.0, 3, "f64", None)[0]
    assert np.array_equal(out, golden["ring5_phi"])


def test_step_with_injected_noise_matches_reference(pkg, golden):
    """euler_step of the reference with its own numpy normals handed to the device (parity hook)."""
    from paper_2505_22631_b200.dynamics import _step_raw
    J = coupling_from_golden(golden, "g9")
    K, ks_max, ks_period, kn, h, _, N, _ = golden["g9_params"]
    ks = pkg.KsSchedule(ks_max, ks_period).value(float(golden["g9_t"][0]))
    out = _step_raw(J, golden["g9_phi"][None], golden["g9_noise"][None], K, ks, h, kn * math.sqrt(h), int(N), "f64", None)[0]
    assert np.abs(out - golden["g9_out"]).max() <= 1e-12
    out32 = _step_raw(J, golden["g9_phi"][None], golden["g9_noise"][None], K, ks, h, kn * math.sqrt(h), int(N), "f32", None)[0]
    assert circ_dist_rad(out32, golden["g9_out"]).max() <= 2e-6


def test_phase_drift_matches_formula(pkg, golden):
    J = coupling_from_golden(golden, "g9")
    K, ks_max, ks_period, *_ = golden["g9_params"]
    ks = pkg.KsSchedule(ks_max, ks_period).value(float(golden["g9_t"][0]))
    phi = pkg.PhaseState(golden["g9_phi"])
    got = [pkg.phase_drift(J, phi, i, K, ks, 3) for i in range(9)]
    assert np.abs(np.array(got) - golden["g9_drift"]).max() <= 1e-12
    assert pkg.phase_drift(pkg.CouplingMatrix.from_edges(1, []), pkg.PhaseState(np.array([0.125])), 0, 1.0, 1.0, 2) == pytest.approx(-1.0, abs=1e-14)  # test_dynamics.py:122-127
    with pytest.raises(IndexError):
        pkg.phase_drift(J, phi, 9, K, ks, 3)


@pytest.mark.parametrize("precision,tol", [("f64", 1e-12), ("f32", 3e-6)])
@pytest.mark.parametrize("R", [1, 5, 64])
def test_step_batched_vs_oracle(pkg, oracle, precision, tol, R):
    """Random signed graph, ragged degrees (incl. isolated nodes), all replicas in one call."""
    from paper_2505_22631_b200.dynamics import _step_raw
    n = 203
    iu, iv, w = random_graph_arrays(n, 0.05, seed=R, weights=(-1.0, 1.0, 0.5, 2.0))
    keep = (iu != 7) & (iv != 7)          # node 7 isolated
    J = make_coupling(pkg, n, iu[keep], iv[keep], w[keep])
    rng = np.random.default_rng(100 + R)
    phi = rng.random((R, n))
    noise = rng.standard_normal((R, n))
    for N in (2, 3):
        want = oracle.step(J.indptr, J.indices, J.data, phi, noise, 0.7, 0.9, 0.01, 0.03, N)
        got = _step_raw(J, phi, noise, 0.7, 0.9, 0.01, 0.03, N, precision, None)
        assert got.shape == want.shape
        assert circ_dist_rad(got, want).max() <= tol
        assert got.min() >= 0.0 and got.max() < 1.0


@pytest.mark.parametrize("N", [2, 3, 5])
def test_score_bit_exact_golden(pkg, golden, N):
    J = coupling_from_golden(golden, "g40")
    phi = golden[f"score_N{N}_phi"]
    for kind, maximize in (("maxcut", 1), ("coloring", 0)):
        states, obj = pkg.score_phases(J, phi, N, kind)
        assert np.array_equal(states, golden[f"score_N{N}_max{maximize}_states"])
        assert np.array_equal(obj, golden[f"score_N{N}_max{maximize}_obj"])


@pytest.mark.parametrize("R,n,weights", [(1, 50, (1.0,)), (33, 300, (1.0, -1.0)), (128, 120, (0.3, -1.7, 2.25))])
def test_score_and_energy_vs_oracle(pkg, oracle, R, n, weights):
    iu, iv, w = random_graph_arrays(n, 0.08, seed=n, weights=weights)
    J = make_coupling(pkg, n, iu, iv, w)
    rng = np.random.default_rng(n + R)
    phi = rng.random((R, n))
    phi[0, :6] = [0.25, 0.75, 0.5, 0.0, 1 / 3, 2 / 3]
    phi32 = phi.astype(np.float32).astype(np.float64)     # values the f32 kernels can hold
    piu, pjv, pw = J.pairs()
    for N, kind in ((2, "maxcut"), (3, "coloring"), (4, "coloring")):
        for p in (phi, phi32):
            ws, wo = oracle.score(p, N, piu, pjv, pw, kind == "maxcut")
            gs, go = pkg.score_phases(J, p, N, kind)
            assert np.array_equal(gs, ws)
            assert np.array_equal(go, wo)        # incl. non-integer weights: same summation order
    want = np.array([oracle.continuous_energy(phi[r], piu, pjv, pw) for r in range(R)])
    got = pkg.sample_energy(J, phi)
    assert np.abs(got - want).max() <= 1e-9 * max(1.0, np.abs(pw).sum())


def test_score_empty_graph(pkg):
    J = pkg.CouplingMatrix.from_edges(4, [])
    states, obj = pkg.score_phases(J, np.array([[0.1, 0.3, 0.6, 0.9]]), 2, "maxcut")
    assert states.tolist() == [[0, 1, 1, 0]] and obj.tolist() == [0.0]


# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("kernel", KERNELS)
def test_run_noise_free_matches_reference_golden(pkg, golden, kernel):
    """400 noise-free steps, float64 parity mode: trajectory, traces and best states vs the
    reference itself (golden)."""
    J = coupling_from_golden(golden, "g30")
    params = params_from_row(golden["run30_quiet_params"])
    res = pkg.run_replica_set(J, params, "maxcut", replicas=3, precision="f64", kernel=kernel)
    assert res[0].steps_executed == int(golden["run30_quiet_steps"][0]) == 400
    for r, one in enumerate(res):
        assert circ_dist_rad(one.final_phases.phases, golden["run30_quiet_final"][r]).max() <= 1e-9   # N = 400 steps
        assert np.array_equal(one.best_assignment.states, golden["run30_quiet_best_states"][r])
        assert one.best_objective == golden["run30_quiet_best_obj"][r]
        t, e, ks = map(np.array, zip(*one.energy_trace))
        assert np.array_equal(t, golden["run30_quiet_trace_t"])
        assert np.array_equal(ks, golden["run30_quiet_trace_ks"])
        assert np.abs(e - golden["run30_quiet_energy"][r]).max() <= 1e-8
        assert np.array_equal(np.array(one.best_trace), golden["run30_quiet_best_trace"][r])
        assert one.replica_index == r and one.objective_kind == "maxcut"


@pytest.mark.parametrize("kernel", KERNELS)
def test_run_noise_free_f32_short_horizon(pkg, golden, kernel):
    """fp32 throughput mode: 1e-4 rad holds over a short horizon (N = 40 steps here)."""
    J = coupling_from_golden(golden, "g30")
    params = params_from_row(golden["run30_quiet_params"], t_stop=0.4)
    ref = pkg.run_batch(J, params, "maxcut", [7, 8, 9], precision="f64", kernel="stream")
    got = pkg.run_batch(J, params, "maxcut", [7, 8, 9], precision="f32", kernel=kernel)
    assert got.steps == 40
    assert circ_dist_rad(got.final_phases, ref.final_phases).max() <= 1e-4


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("graph,tag,kind,replicas,stride", [
    ("g30", "run30_noisy", "maxcut", 3, None),
    ("col24", "run_col24", "coloring", 2, 0.37),
])
def test_run_with_reference_noise_injected(pkg, oracle, golden, kernel, graph, tag, kind, replicas, stride):
    """Noisy trajectories: the reference's own numpy normals are injected through the parity
    hook (OSCB_NOISE_HOST), so the whole noisy run must follow the reference's."""
    J = coupling_from_golden(golden, graph)
    params = params_from_row(golden[f"{tag}_params"])
    steps = int(golden[f"{tag}_steps"][0])
    seeds = [(params.seed + r) % 2**64 for r in range(replicas)]
    n = J.n
    noise = np.empty((steps, replicas, n))
    for r, s in enumerate(seeds):
        for c in range((steps + 255) // 256):
            chunk = oracle.normal_chunk(s, c, n)
            lo, hi = c * 256, min(steps, (c + 1) * 256)
            noise[lo:hi, r] = chunk[: hi - lo]
    b = pkg.run_batch(J, params, kind, seeds, trace_stride=stride, precision="f64", kernel=kernel, noise=noise)
    assert b.steps == steps
    assert np.array_equal(b.trace_t, golden[f"{tag}_trace_t"])
    assert np.array_equal(b.trace_ks, golden[f"{tag}_trace_ks"])
    assert circ_dist_rad(b.final_phases, golden[f"{tag}_final"]).max() <= 1e-8
    assert np.array_equal(b.best_states.astype(np.int64), golden[f"{tag}_best_states"])
    assert np.array_equal(b.best_objective, golden[f"{tag}_best_obj"])
    assert np.array_equal(b.best_trace, golden[f"{tag}_best_trace"])
    assert np.abs(b.energy - golden[f"{tag}_energy"]).max() <= 1e-7


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("shape,steps32", [("G1", 20), ("G22", 20), ("flat200", 100), ("G81", 20)])
def test_config_shapes_noise_free_vs_oracle(pkg, oracle, kernel, shape, steps32):
    """BASELINE.json config shapes, noise off: f64 parity over N = 200 steps, f32 over the short
    horizon SURVEY 7-A measured (N = 20; 100 for flat200)."""
    from paper_2505_22631_b200 import workloads
    n, (u, v, w), N, kind = workloads.shape_graph(shape)
    J = pkg.CouplingMatrix.from_edges(n, (u, v, w))
    tune = dict(K=0.2, ks_max=1.0, kn=0.0) if N == 2 else dict(kn=0.0)
    params = pkg.SolverParams.tuned_for(n, N, seed=5, **tune)
    R = 2 if shape == "G81" else 4
    seeds = [params.seed + r for r in range(R)]
    kw = dict(K=params.K, ks_max=params.ks_max, ks_period=params.ks_period, kn=0.0, h=params.h, n_states=N,
              seeds=seeds, objective=kind, threads=oracle.max_threads())
    for precision, steps, tol in (("f64", 200, 1e-9), ("f32", steps32, 1e-4)):
        want = oracle.simulate(J.indptr, J.indices, J.data, t_stop=steps * params.h, **kw)
        use = "auto" if (shape == "G81" and precision == "f64" and kernel.startswith("resident")) else kernel   # 16-byte pairs of 20000 oscillators exceed one SM
        got = pkg.run_batch(J, params, kind, seeds, precision=precision, kernel=use, steps=steps)
        assert got.steps == want.steps == steps
        assert circ_dist_rad(got.final_phases, want.final_phases).max() <= tol, (shape, precision)
        if precision == "f64":
            assert np.array_equal(got.best_states.astype(np.int64), want.best_states)
            assert np.array_equal(got.best_objective, want.best_objective)


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_run_equals_chain_of_euler_steps(pkg, golden, precision):
    """reference test_dynamics.py:270-281 (bit-identical) on the streaming kernels, device noise on."""
    J = coupling_from_golden(golden, "g30")
    params = params_from_row(golden["run30_noisy_params"], t_stop=0.25)
    full = pkg.run(J, params, "maxcut", precision=precision, kernel="stream")
    src = pkg.NoiseSource(params.seed)
    phi = pkg.PhaseState(src.initial_phases(J.n))
    for k in range(25):
        phi = pkg.euler_step(phi, J, params, k * params.h, src, k, precision=precision)
    assert np.array_equal(phi.phases, full.final_phases.phases)


@pytest.mark.parametrize("kernel", KERNELS)
def test_determinism_and_replica_independence(pkg, golden, kernel):
    """reference test_dynamics.py:257-267, :311-341: same call twice is bit-identical; a replica
    inside a batch equals the solo run with replica_seed."""
    J = coupling_from_golden(golden, "g30")
    params = params_from_row(golden["run30_noisy_params"], t_stop=1.0)
    a = pkg.run_replica_set(J, params, "maxcut", replicas=5, kernel=kernel)
    b = pkg.run_replica_set(J, params, "maxcut", replicas=5, kernel=kernel)
    for x, y in zip(a, b):
        assert np.array_equal(x.final_phases.phases, y.final_phases.phases)
        assert x.energy_trace == y.energy_trace and x.best_objective == y.best_objective
    import dataclasses
    solo = pkg.run(J, dataclasses.replace(params, seed=params.seed + 3), "maxcut", kernel=kernel)
    assert np.array_equal(solo.final_phases.phases, a[3].final_phases.phases)
    assert solo.best_objective == a[3].best_objective


def test_sign_of_cosine_is_the_binary_threshold(pkg):
    """The float32 kernel scores N = 2 states as the sign bit of cospi(2 phi): exhaustive check over
    every float32 in [0, 1) against the reference threshold rule (dynamics.py:203-213)."""
    import ctypes as C
    from paper_2505_22631_b200 import _native as nat
    bad = C.c_uint64(123)
    assert nat.lib().oscb_selftest_sign_state(0, C.byref(bad)) == 0, nat.last_error()
    assert bad.value == 0


@pytest.mark.parametrize("shape,R", [("G22", 24), ("G1", 3), ("flat200", 70), ("G81", 2)])
def test_resident_kernels_agree_on_scoring(pkg, shape, R):
    """Noise ON, float32: the specialised kernel (scoring fused into the gather for N = 2) and the
    streaming kernel follow different code paths but the same arithmetic contract; over a short
    noisy window their best cuts must be statistically indistinguishable and each must equal the
    cut recomputed from its own best states."""
    from paper_2505_22631_b200 import workloads
    n, (u, v, w), N, kind = workloads.shape_graph(shape)
    J = pkg.CouplingMatrix.from_edges(n, (u, v, w))
    tune = dict(K=0.2, ks_max=1.0, kn=0.15) if N == 2 else {}
    params = pkg.SolverParams.tuned_for(n, N, seed=3, **tune)
    piu, pjv, pw = J.pairs()
    res = {}
    for kernel in ("resident", "resident-generic", "stream"):
        b = pkg.run_batch(J, params, kind, list(range(R)), kernel=kernel, steps=400)
        s = b.best_states.astype(np.int64)
        if kind == "maxcut":
            recomputed = (pw[None, :] * (s[:, piu] != s[:, pjv])).sum(axis=1)
        else:
            recomputed = (s[:, piu] == s[:, pjv]).sum(axis=1).astype(float)
        assert np.array_equal(recomputed, b.best_objective), kernel
        assert np.all(np.diff(b.best_trace, axis=1) >= 0) if kind == "maxcut" else np.all(np.diff(b.best_trace, axis=1) <= 0)
        res[kernel] = b
    scale = max(1.0, abs(res["stream"].best_objective.mean()))
    for kernel in ("resident", "resident-generic"):
        assert abs(res[kernel].best_objective.mean() - res["stream"].best_objective.mean()) < 0.02 * scale


def test_device_normals_statistics(pkg):
    """reference test_dynamics.py:76-105: repeatable, stream-separated, unit moments."""
    src = pkg.NoiseSource(11)
    a = src.step_normals(5, 250_000)
    assert np.array_equal(a, src.step_normals(5, 250_000))
    assert np.array_equal(a[:1000], src.step_normals(5, 1000))           # independent of n
    assert not np.array_equal(a, src.step_normals(6, 250_000))
    assert not np.array_equal(a, pkg.NoiseSource(12).step_normals(5, 250_000))
    big = np.concatenate([src.step_normals(s, 250_000) for s in range(4)])
    assert abs(big.mean()) < 0.01 and abs(big.var() - 1.0) < 0.01
    assert abs((big ** 3).mean()) < 0.02 and abs((big ** 4).mean() - 3.0) < 0.05
    d = pkg.NoiseSource(11, precision="f64").step_normals(5, 4096)
    assert np.abs(d - a[:4096]).max() < 1e-5                              # same draws, two arithmetics


@pytest.mark.parametrize("kernel", KERNELS)
def test_noise_increment_std(pkg, kernel):
    """reference test_dynamics.py:386-399: with K ~ 0 and ks = 0 the per-step increment has
    std kn*sqrt(h)."""
    J = pkg.CouplingMatrix.from_edges(4000, [(0, 1, 1.0)])
    params = pkg.SolverParams(K=1e-12, ks_max=0.0, kn=0.5, h=0.01, t_stop=1.0, seed=3)
    b = pkg.run_batch(J, params, "maxcut", [3, 4, 5, 6], kernel=kernel, steps=1)
    start = np.stack([pkg.NoiseSource(s).initial_phases(4000) for s in (3, 4, 5, 6)])
    d = b.final_phases - start
    d -= np.round(d)
    assert abs(d.std() / (0.5 * 0.1) - 1.0) < 0.03


@pytest.mark.parametrize("kernel", KERNELS)
def test_best_cut_distribution_matches_reference_oracle(pkg, oracle, kernel):
    """Noise ON, device Philox stream vs the reference's numpy stream (replayed by the oracle):
    the distribution of best cuts over 96 seeds must agree (two-sample KS), and so must the
    mean."""
    from scipy import stats
    n = 60
    iu, iv, w = random_graph_arrays(n, 0.15, seed=77, weights=(1.0,))
    J = make_coupling(pkg, n, iu, iv, w)
    params = pkg.SolverParams(K=0.2, ks_max=1.0, ks_period=3.0, kn=0.15, h=0.01, t_stop=9.0, seed=1000)
    seeds = [params.seed + r for r in range(96)]
    want = oracle.simulate(J.indptr, J.indices, J.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period,
                           kn=params.kn, h=params.h, t_stop=params.t_stop, n_states=2, seeds=seeds,
                           objective="maxcut", threads=oracle.max_threads())
    for precision in ("f32", "f64"):
        got = pkg.run_batch(J, params, "maxcut", seeds, precision=precision, kernel=kernel)
        ks = stats.ks_2samp(got.best_objective, want.best_objective)
        assert ks.pvalue > 0.01, (precision, ks)
        assert abs(got.best_objective.mean() - want.best_objective.mean()) < 0.6 * (want.best_objective.std() + 0.5)
        # final-state cuts too (not only the best-so-far)
        iu_, jv_, w_ = J.pairs()
        _, cut_got = oracle.score(got.final_phases, 2, iu_, jv_, w_, True)
        _, cut_want = oracle.score(want.final_phases, 2, iu_, jv_, w_, True)
        assert stats.ks_2samp(cut_got, cut_want).pvalue > 0.01


@pytest.mark.parametrize("kernel", KERNELS)
def test_result_contract(pkg, oracle, kernel):
    """SURVEY 8b result contract (test_dynamics.py:196-202, :284-299)."""
    n = 64
    iu, iv, w = random_graph_arrays(n, 0.2, seed=9, weights=(1.0, -1.0))
    J = make_coupling(pkg, n, iu, iv, w)
    params = pkg.SolverParams.tuned_for(n, 2, seed=4, t_stop=6.0)
    res = pkg.run(J, params, "maxcut", kernel=kernel)
    assert res.steps_executed == math.ceil(params.t_stop / params.h)
    p = res.final_phases.phases
    assert p.min() >= 0.0 and p.max() < 1.0
    piu, pjv, pw = J.pairs()
    _, obj = oracle.score(np.zeros((1, n)), 2, piu, pjv, pw, True)   # exercise the checker, all-zero state cut = 0
    assert obj[0] == 0.0
    s = res.best_assignment.states
    assert res.best_objective == float((pw * (s[piu] != s[pjv])).sum())
    ts = [t for t, _, _ in res.energy_trace]
    assert ts[0] == 0.0 and all(b > a for a, b in zip(ts, ts[1:]))
    sched = pkg.KsSchedule(params.ks_max, params.ks_period)
    assert all(ks == sched.value(t) for t, _, ks in res.energy_trace)
    assert all(b >= a for a, b in zip(res.best_trace, res.best_trace[1:]))
    assert res.best_trace[-1] == res.best_objective
    best = pkg.run_replicas(J, params, "maxcut", replicas=6, kernel=kernel)
    allr = pkg.run_replica_set(J, params, "maxcut", replicas=6, kernel=kernel)
    assert best.best_objective == max(r.best_objective for r in allr)
    assert best.replica_index == min(r.replica_index for r in allr if r.best_objective == best.best_objective)


@pytest.mark.parametrize("kernel", KERNELS)
def test_numerical_error_reports_oscillator_and_step(pkg, kernel):
    """reference test_dynamics.py:186-192: overflow -> NumericalError naming oscillator & step."""
    J = pkg.CouplingMatrix.from_edges(3, [(0, 1, 1e308), (1, 2, 1e308)])
    params = pkg.SolverParams(K=1e308, ks_max=0.0, kn=0.0, h=0.5, t_stop=2.0, seed=1)
    with pytest.raises(pkg.NumericalError) as ei:
        pkg.run(J, params, "maxcut", precision="f64", kernel=kernel)
    assert "oscillator" in str(ei.value) and "step" in str(ei.value)
    with pytest.raises(pkg.NumericalError):
        pkg.euler_step(pkg.PhaseState(np.array([0.1, 0.2, 0.3])), J, params, 0.0, pkg.NoiseSource(1), 0, precision="f64")


def test_argument_errors(pkg):
    J = pkg.CouplingMatrix.from_edges(3, [(0, 1, 1.0)])
    with pytest.raises(ValueError):
        pkg.run(J, pkg.SolverParams(t_stop=1.0), "tsp")
    with pytest.raises(ValueError):
        pkg.run(J, pkg.SolverParams(t_stop=1.0, n_states=3), "maxcut")
    with pytest.raises(ValueError):
        pkg.run_replica_set(J, pkg.SolverParams(t_stop=1.0), "maxcut", replicas=0)
    with pytest.raises(ValueError):
        pkg.euler_step(pkg.PhaseState(np.array([0.1, 0.2])), J, pkg.SolverParams(), 0.0, pkg.NoiseSource(0), 0)
    with pytest.raises(ValueError):
        pkg.run(J, pkg.SolverParams(t_stop=1.0), "maxcut", trace_stride=0.0)


@pytest.mark.parametrize("kernel", KERNELS)
def test_solution_quality_small_instances(pkg, kernel):
    """reference test_dynamics.py:216-236 bars: single edge -> cut 1, triangle -> cut 2."""
    edge = pkg.CouplingMatrix.from_edges(2, [(0, 1, 1.0)])
    tri = pkg.CouplingMatrix.from_edges(3, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0)])
    pe = pkg.SolverParams.tuned_for(2, 2, seed=0)
    pt = pkg.SolverParams.tuned_for(3, 2, seed=0)
    e = pkg.run_replica_set(edge, pe, "maxcut", replicas=100, kernel=kernel)
    t = pkg.run_replica_set(tri, pt, "maxcut", replicas=100, kernel=kernel)
    assert sum(r.best_objective == 1.0 for r in e) >= 99
    assert sum(r.best_objective == 2.0 for r in t) >= 95


@pytest.mark.parametrize("kernel", KERNELS)
def test_full_size_g22_properties(pkg, kernel):
    """BASELINE configs[1] at full size (G22 shape, 1024 replicas), a 300-step window: size-
    independent properties -- phase containment, best = recomputed cut of the best states,
    monotone best trace, sane cut range."""
    from paper_2505_22631_b200 import workloads
    n, (u, v, w), N, kind = workloads.shape_graph("G22")
    J = pkg.CouplingMatrix.from_edges(n, (u, v, w))
    params = pkg.SolverParams.tuned_for(n, 2, seed=0, K=0.2, ks_max=1.0, kn=0.15)
    b = pkg.run_batch(J, params, kind, list(range(1024)), kernel=kernel, steps=300)
    assert b.final_phases.min() >= 0.0 and b.final_phases.max() < 1.0
    piu, pjv, pw = J.pairs()
    s = b.best_states.astype(np.int64)
    recomputed = (pw[None, :] * (s[:, piu] != s[:, pjv])).sum(axis=1)
    assert np.array_equal(recomputed, b.best_objective)
    assert np.all(np.diff(b.best_trace, axis=1) >= 0)
    assert 0.5 * len(pw) < b.best_objective.min() and b.best_objective.max() <= len(pw)
    assert len(np.unique(b.best_objective)) > 3          # replicas are really different
