"""Tensor-core dense integrator (csrc/oscb_umma.cuh, kernel "dense-tc") against the float64 SIMT
dense path and the CPU oracle on the same couplings and seeds.

The coupling sums of the tensor-core kernel are exact integer dot products of J with the 2^-30
fixed-point digits of (cos, sin), so with a float64 epilogue the trajectory differs from the
reference only by that quantisation: the noise-free bar is 1e-6 rad after N = 200 steps (the
north-star tolerance is 1e-4 rad); cut values, best states and traces are bit-exact."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def sk_graph(n, seed, weights=(-1.0, 1.0)):
    rng = np.random.default_rng(seed)
    U = np.triu(rng.choice(np.asarray(weights, dtype=np.float64), size=(n, n)), 1)
    return U + U.T


@pytest.fixture(scope="module")
def pkg():
    import paper_2505_22631_b200 as p
    from paper_2505_22631_b200 import _native, dynamics
    assert _native.device_count() > 0, "no CUDA device: " + _native.last_error()
    old = dynamics.DENSE_DEVICE_MIN_N
    dynamics.DENSE_DEVICE_MIN_N = 0
    yield p
    dynamics.DENSE_DEVICE_MIN_N = old


def circ(a, b):
    d = np.abs(a - b)
    return 2 * np.pi * np.minimum(d, 1 - d)


@pytest.mark.parametrize("n,R,weights,grid_cap", [
    (256, 3, (-1.0, 1.0), None),
    (300, 5, (-1.0, 1.0), None),                     # ragged last tile
    (200, 2, (-3.0, -1.0, 0.0, 0.0, 1.0, 2.0), None),  # general small integers, zeros
    (640, 4, (-1.0, 1.0), "2"),                      # 5 row tiles on 2 CTAs: several tiles per CTA
])
def test_noise_free_run_matches_float64_stream_and_oracle(pkg, oracle, n, R, weights, grid_cap):
    J = sk_graph(n, 100 + n, weights)
    Jd = pkg.CouplingMatrix.from_dense(J, storage="dense")
    Js = pkg.CouplingMatrix.from_dense(J, storage="sparse")
    params = pkg.SolverParams(K=0.02, ks_max=1.0, ks_period=1.0, kn=0.0, h=0.01, t_stop=2.0, seed=4)
    seeds = list(range(4, 4 + R))
    if grid_cap:
        os.environ["OSCB_UMMA_MAX_GRID"] = grid_cap
    try:
        got = pkg.run_batch(Jd, params, "maxcut", seeds, precision="f64", kernel="dense-tc")
    finally:
        os.environ.pop("OSCB_UMMA_MAX_GRID", None)
    assert got.kernel == "dense-tc" and got.steps == 200
    want = pkg.run_batch(Jd, params, "maxcut", seeds, precision="f64", kernel="stream")
    ref = oracle.simulate(Js.indptr, Js.indices, Js.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period,
                          kn=0.0, h=params.h, t_stop=params.t_stop, n_states=2, seeds=seeds, objective="maxcut")
    assert circ(got.final_phases, want.final_phases).max() <= 1e-6          # N = 200 steps
    assert circ(got.final_phases, ref.final_phases).max() <= 1e-6
    assert np.array_equal(got.best_objective, ref.best_objective)
    assert np.array_equal(got.best_states.astype(np.int64), ref.best_states)
    assert np.array_equal(got.trace_t, ref.trace_t) and np.array_equal(got.trace_ks, ref.trace_ks)
    assert np.array_equal(got.best_trace, ref.best_trace)
    assert np.abs(got.energy - ref.energy).max() <= 1e-6 * n


def test_noisy_f32_run_is_consistent(pkg):
    """Noise on, float32 epilogue: same (seed, step, oscillator) noise as the SIMT path, so 30 steps
    agree within 1e-4 rad; the result contract holds; best objective == cut of best states."""
    n, R = 384, 6
    J = sk_graph(n, 7)
    Jd = pkg.CouplingMatrix.from_dense(J, storage="dense")
    params = pkg.SolverParams(K=0.02, ks_max=1.0, ks_period=1.0, kn=0.2, h=0.01, t_stop=3.0, seed=11)
    seeds = list(range(11, 11 + R))
    a = pkg.run_batch(Jd, params, "maxcut", seeds, precision="f32", kernel="dense-tc", steps=30)
    b = pkg.run_batch(Jd, params, "maxcut", seeds, precision="f32", kernel="stream", steps=30)
    assert circ(a.final_phases, b.final_phases).max() <= 1e-4                # N = 30 steps
    full = pkg.run_batch(Jd, params, "maxcut", seeds, precision="f32")        # auto -> dense-tc
    assert full.kernel == "dense-tc" and full.steps == 300
    assert (full.final_phases >= 0).all() and (full.final_phases < 1).all()
    iu, jv = np.triu_indices(n, 1)
    for r in range(R):
        s = full.best_states[r].astype(np.int64)
        assert full.best_objective[r] == float((J[iu, jv] * (s[iu] != s[jv])).sum())
        assert (np.diff(full.best_trace[r]) >= 0).all()
    again = pkg.run_batch(Jd, params, "maxcut", seeds, precision="f32")
    assert np.array_equal(again.final_phases, full.final_phases)              # deterministic
    assert np.array_equal(again.energy, full.energy)


def test_replica_chunks_equal_single_runs(pkg):
    """More replicas than one launch takes (28): the chunks reproduce the solo runs bit for bit."""
    n, R = 256, 31
    J = sk_graph(n, 3)
    Jd = pkg.CouplingMatrix.from_dense(J, storage="dense")
    params = pkg.SolverParams(K=0.02, ks_max=1.0, ks_period=0.5, kn=0.1, h=0.01, t_stop=0.6, seed=0)
    seeds = list(range(R))
    allr = pkg.run_batch(Jd, params, "maxcut", seeds, precision="f32", target=0.0)
    for r in (0, 27, 28, 30):
        solo = pkg.run_batch(Jd, params, "maxcut", [seeds[r]], precision="f32", target=0.0)
        assert np.array_equal(solo.final_phases[0], allr.final_phases[r])
        assert np.array_equal(solo.best_states[0], allr.best_states[r])
        assert solo.best_objective[0] == allr.best_objective[r]
        assert np.array_equal(solo.energy[0], allr.energy[r])
        assert solo.first_hit_step[0] == allr.first_hit_step[r]


@pytest.mark.parametrize("n,cuts,precision", [
    (512, (0, 256, 512), "f32"),
    (600, (0, 256, 600), "f64"),          # ragged last shard
    (600, (0, 128, 384, 600), "f32"),     # three ranks
])
def test_fused_virtual_ranks_equal_single_handle(pkg, n, cuts, precision):
    """The multi-GPU protocol of the fused kernel (peer-pointer push of the digit planes, cut atomics
    and step-counter arrivals into every rank's exchange block) with the ranks as concurrent kernels
    on ONE GPU: row shards of J, one persistent kernel each, must reproduce the single-handle run bit
    for bit (noise on; the integer sums are exact, so sharding cannot change a bit)."""
    from paper_2505_22631_b200 import dense_fused
    R = 3
    J = sk_graph(n, 5)
    Jd = pkg.CouplingMatrix.from_dense(J, storage="dense")
    params = pkg.SolverParams(K=0.02, ks_max=1.0, ks_period=0.5, kn=0.2, h=0.01, t_stop=1.2, seed=40)
    seeds = [40, 41, 42]
    want = pkg.run_batch(Jd, params, "maxcut", seeds, precision=precision, kernel="dense-tc", target=0.0)
    shards = [(J[a:b], a, b, 0) for a, b in zip(cuts[:-1], cuts[1:])]
    got = dense_fused.run_fused_in_process(shards, n, params, seeds, pair_count=n * (n - 1) // 2, precision=precision)
    assert got.steps == want.steps == 120
    assert np.array_equal(got.final_phases, want.final_phases)
    assert np.array_equal(got.best_states, want.best_states)
    assert np.array_equal(got.best_objective, want.best_objective)
    assert np.array_equal(got.trace_t, want.trace_t) and np.array_equal(got.trace_ks, want.trace_ks)
    assert np.array_equal(got.best_trace, want.best_trace)
    assert np.array_equal(got.energy, want.energy)


@pytest.mark.parametrize("n,N,R", [(256, 3, 4), (300, 4, 3), (200, 7, 2)])
def test_potts_colouring_on_the_tensor_cores(pkg, oracle, n, N, R):
    """OPM on a dense unit-coupled graph: N one-hot state planes in B give sum_j J_ij [s_j == s_i] exactly;
    the N-th harmonic SHIL and the N-state threshold run in the epilogue.  Noise-free float64 epilogue vs
    the oracle (1e-6 rad after 150 steps, conflicts / states / traces equal), then a noisy float32 run
    through the result contract."""
    rng = np.random.default_rng(N)
    U = np.triu((rng.random((n, n)) < 0.4).astype(np.float64), 1)
    A = U + U.T
    Jd = pkg.CouplingMatrix.from_dense(A, storage="dense")
    Js = pkg.CouplingMatrix.from_dense(A, storage="sparse")
    params = pkg.SolverParams(K=0.01, ks_max=0.5, ks_period=0.5, kn=0.0, h=0.01, t_stop=1.5, n_states=N, seed=8)
    seeds = list(range(8, 8 + R))
    got = pkg.run_batch(Jd, params, "coloring", seeds, precision="f64", kernel="dense-tc")
    assert got.kernel == "dense-tc" and got.steps == 150
    ref = oracle.simulate(Js.indptr, Js.indices, Js.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period,
                          kn=0.0, h=params.h, t_stop=params.t_stop, n_states=N, seeds=seeds, objective="coloring")
    assert circ(got.final_phases, ref.final_phases).max() <= 1e-6          # N = 150 steps
    assert np.array_equal(got.best_objective, ref.best_objective)
    assert np.array_equal(got.best_states.astype(np.int64), ref.best_states)
    assert np.array_equal(got.best_trace, ref.best_trace)
    assert np.abs(got.energy - ref.energy).max() <= 1e-6 * n * n
    noisy = pkg.run_batch(Jd, pkg.SolverParams.tuned_for(n, N, seed=1, t_stop=4.0), "coloring", seeds, precision="f32")
    assert noisy.kernel == "dense-tc"
    iu, jv = np.nonzero(np.triu(A, 1))
    s = noisy.best_states.astype(np.int64)
    assert s.max() < N
    assert np.array_equal((s[:, iu] == s[:, jv]).sum(axis=1).astype(np.float64), noisy.best_objective)
    assert np.all(np.diff(noisy.best_trace, axis=1) <= 0)
    # weighted couplings with the colouring objective are not a tensor-core case: the SIMT path takes them
    W = A * 2.0
    Jw = pkg.CouplingMatrix.from_dense(W, storage="dense")
    assert pkg.run_batch(Jw, params, "coloring", seeds[:1], precision="f32", steps=5).kernel == "stream"


@pytest.mark.parametrize("kind,N", [("maxcut", 2), ("coloring", 3)])
def test_best_objective_distribution_matches_reference_oracle(pkg, oracle, kind, N):
    """Noise ON, the tensor-core kernel (float32 epilogue, device Philox noise) vs the oracle with the
    reference's numpy stream: best objectives over 96 seeds agree in distribution (two-sample KS)."""
    from scipy import stats
    n = 256
    rng = np.random.default_rng(31)
    if kind == "maxcut":
        A = sk_graph(n, 31)
        params = pkg.SolverParams(K=0.05, ks_max=1.0, ks_period=2.0, kn=0.15, h=0.01, t_stop=6.0, seed=500)
    else:
        U = np.triu((rng.random((n, n)) < 0.3).astype(np.float64), 1)
        A = U + U.T
        params = pkg.SolverParams(K=0.02, ks_max=0.5, ks_period=2.0, kn=0.1, h=0.01, t_stop=6.0, n_states=3, seed=500)
    Jd = pkg.CouplingMatrix.from_dense(A, storage="dense")
    Js = pkg.CouplingMatrix.from_dense(A, storage="sparse")
    seeds = [params.seed + r for r in range(96)]
    want = oracle.simulate(Js.indptr, Js.indices, Js.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period, kn=params.kn,
                           h=params.h, t_stop=params.t_stop, n_states=N, seeds=seeds, objective=kind, threads=oracle.max_threads())
    got = pkg.run_batch(Jd, params, kind, seeds, precision="f32")
    assert got.kernel == "dense-tc"
    assert stats.ks_2samp(got.best_objective, want.best_objective).pvalue > 0.01
    assert abs(got.best_objective.mean() - want.best_objective.mean()) < 0.6 * (want.best_objective.std() + 0.5)


def test_fp4_stream_equals_int8_stream(pkg):
    """Couplings in {0, +-1, +-2, +-3, +-4, +-6} can stream as packed e2m1 codes (half the bytes) and be multiplied on the
    block-scaled 4-bit tensor path (kind::mxf4, all scales 1.0) against e2m1 balanced base-9 digit planes, float32
    accumulators holding exact integers (the default for up to 12 replicas per call).  The
    reassembled sums are the same integers as on the int8 path, so the two modes must agree bit for bit (noise on,
    ragged n, several tiles per CTA, zeros and weights up to 6 included)."""
    for n, cap, weights in ((256, None, (-1.0, 1.0)), (300, None, (-6.0, -3.0, -1.0, 0.0, 0.0, 1.0, 2.0, 4.0)), (640, "2", (-1.0, 1.0))):
        J = sk_graph(n, 900 + n, weights)
        Jd = pkg.CouplingMatrix.from_dense(J, storage="dense")
        params = pkg.SolverParams(K=0.01, ks_max=1.0, ks_period=0.5, kn=0.2, h=0.01, t_stop=1.0, seed=70)
        seeds = [70, 71, 72]
        if cap:
            os.environ["OSCB_UMMA_MAX_GRID"] = cap
        try:
            runs = {}
            for mode in ("0", "1"):                    # 0: int8 stream, 1: packed e2m1 stream
                os.environ["OSCB_UMMA_FP4"] = mode
                try:
                    runs[mode] = pkg.run_batch(Jd, params, "maxcut", seeds, precision="f32", kernel="dense-tc")
                finally:
                    os.environ.pop("OSCB_UMMA_FP4", None)
            int8, fp4 = runs["0"], runs["1"]
        finally:
            os.environ.pop("OSCB_UMMA_MAX_GRID", None)
        assert np.array_equal(fp4.final_phases, int8.final_phases)
        assert np.array_equal(fp4.best_states, int8.best_states)
        assert np.array_equal(fp4.best_objective, int8.best_objective)
        assert np.array_equal(fp4.energy, int8.energy)


def test_stream_choice_reported_by_the_abi(pkg):
    """oscb_dense_tc_stream: packed e2m1 tiles when every coupling is an e2m1 value and the call fits one launch of that
    stream (21 B columns per replica at N = 2 -> 12 replicas; 20 + N columns at N states), int8 tiles otherwise."""
    from paper_2505_22631_b200 import dynamics
    g = dynamics.DeviceGraph.from_dense(0, sk_graph(256, 1))
    try:
        assert g.tc_stream(2, 1) == (4, 12) and g.tc_stream(2, 12) == (4, 12)
        assert g.tc_stream(2, 13) == (8, 28) and g.tc_stream(2, 1000) == (8, 28)
        assert g.tc_stream(3, 11) == (4, 11) and g.tc_stream(3, 12) == (8, 23)
    finally:
        g.close()
    g5 = dynamics.DeviceGraph.from_dense(0, sk_graph(256, 2, (-5.0, 1.0)))       # 5 is not an e2m1 value
    try:
        assert g5.tc_stream(2, 1) == (8, 28)
    finally:
        g5.close()
    sparse = pkg.CouplingMatrix.from_dense(sk_graph(64, 3), storage="sparse")
    gs = dynamics.device_graph(sparse, 0)
    with pytest.raises(ValueError):
        gs.tc_stream(2, 1)


def test_fused_ranks_agree_on_one_stream(pkg):
    """A coupling outside {0, +-1, +-2, +-3, +-4, +-6} in ONE rank's rows only (its diagonal block) makes that shard an
    int8 shard while its peer could stream packed e2m1.  At R = 1 both exchange blocks have the same size, so the ranks
    used to connect and corrupt each other's B images silently.  Now (a) the driver agrees on one stream before create
    and the run equals the single-handle run bit for bit, and (b) ranks created with different streams refuse to connect."""
    from paper_2505_22631_b200 import dense_fused
    n = 512
    J = sk_graph(n, 9)
    J[300, 301] = J[301, 300] = 5.0            # only in rank 1's diagonal block
    Jd = pkg.CouplingMatrix.from_dense(J, storage="dense")
    params = pkg.SolverParams(K=0.02, ks_max=1.0, ks_period=0.5, kn=0.2, h=0.01, t_stop=0.6, seed=7)
    want = pkg.run_batch(Jd, params, "maxcut", [7], kernel="dense-tc")
    shards = [(J[0:256], 0, 256, 0), (J[256:512], 256, 512, 0)]
    got = dense_fused.run_fused_in_process(shards, n, params, [7], pair_count=n * (n - 1) // 2)
    assert np.array_equal(got.final_phases, want.final_phases) and np.array_equal(got.best_objective, want.best_objective)
    assert np.array_equal(got.best_states, want.best_states) and np.array_equal(got.energy, want.energy)
    # (b) the shards' own choices differ ...
    ranks = [dense_fused.FusedDenseRank(Jr, n, a, b, 0, params, 1, n * (n - 1) // 2, 2, r) for r, (Jr, a, b, _) in enumerate(shards)]
    try:
        assert dense_fused.shard_stream_bits(ranks[0].graph, 2, 1) == 4 and dense_fused.shard_stream_bits(ranks[1].graph, 2, 1) == 8
        assert dense_fused.agree_stream([4, 8]) == 8 and dense_fused.agree_stream([4, 4]) == 4
        blobs = [rk.export() for rk in ranks]
        assert len(blobs[0]) == len(blobs[1])
        with pytest.raises(ValueError, match="same stream"):          # ... and connect says so instead of corrupting
            ranks[0].connect(blobs)
    finally:
        for rk in ranks:
            rk.close()


def test_watchdog_abandons_a_run_whose_peer_never_arrives(pkg, monkeypatch):
    """The producers spin on the step barrier of ALL ranks.  A peer that never launches used to hang the GPU; now the
    wait has a deadline (OSCB_UMMA_WATCHDOG_MS, default 20 s): the kernel free-runs to its end and finish() fails."""
    from paper_2505_22631_b200 import dense_fused
    monkeypatch.setenv("OSCB_UMMA_WATCHDOG_MS", "200")
    n = 512
    J = sk_graph(n, 3)
    params = pkg.SolverParams(K=0.02, ks_max=1.0, ks_period=0.5, kn=0.2, h=0.01, t_stop=0.3, seed=1)
    ranks = [dense_fused.FusedDenseRank(J[a:b], n, a, b, 0, params, 2, n * (n - 1) // 2, 2, r) for r, (a, b) in enumerate(((0, 256), (256, 512)))]
    try:
        blobs = [rk.export() for rk in ranks]
        for rk in ranks:
            rk.connect(blobs)
        for rk in ranks:
            rk.prepare([1, 2])
        ranks[0].launch()                      # rank 1 never launches
        with pytest.raises(RuntimeError, match="abandoned"):
            ranks[0].finish()
    finally:
        for rk in ranks:
            rk.close()
    # the device is fine afterwards: the same ranks run to completion when both launch
    shards = [(J[0:256], 0, 256, 0), (J[256:512], 256, 512, 0)]
    ok = dense_fused.run_fused_in_process(shards, n, params, [1, 2], pair_count=n * (n - 1) // 2)
    assert ok.steps == 30 and ok.final_phases.shape == (2, n)


@pytest.mark.parametrize("splitk", ["2", "4"])
@pytest.mark.parametrize("precision,fp4", [("f32", "1"), ("f64", "0")])
def test_split_k_is_bit_identical(pkg, monkeypatch, splitk, precision, fp4):
    """Split-K (S CTAs share a row tile; partial sums meet in a global int32 accumulator): integer sums do not depend
    on S, so single-handle runs and 2- / 4-virtual-rank row-sharded runs with split-K on equal the unsplit single-handle
    run bit for bit -- phases, states, objectives, traces, energies (noise on, both J streams)."""
    from paper_2505_22631_b200 import dense_fused
    n, R = 1024, 3
    J = sk_graph(n, 12)
    Jd = pkg.CouplingMatrix.from_dense(J, storage="dense")
    params = pkg.SolverParams(K=0.02, ks_max=1.0, ks_period=0.5, kn=0.2, h=0.01, t_stop=0.8, seed=60)
    seeds = [60, 61, 62]
    monkeypatch.setenv("OSCB_UMMA_FP4", fp4)
    monkeypatch.setenv("OSCB_UMMA_SPLITK", "1")
    want = pkg.run_batch(Jd, params, "maxcut", seeds, precision=precision, kernel="dense-tc")
    monkeypatch.setenv("OSCB_UMMA_SPLITK", splitk)
    got = [pkg.run_batch(Jd, params, "maxcut", seeds, precision=precision, kernel="dense-tc")]
    for cuts in ((0, 512, 1024), (0, 256, 512, 768, 1024)):
        shards = [(J[a:b], a, b, 0) for a, b in zip(cuts[:-1], cuts[1:])]
        got.append(dense_fused.run_fused_in_process(shards, n, params, seeds, pair_count=n * (n - 1) // 2, precision=precision))
    for g in got:
        assert g.steps == want.steps == 80
        for f in ("final_phases", "best_states", "best_objective", "best_trace", "energy"):
            assert np.array_equal(getattr(g, f), getattr(want, f)), f


def test_split_k_fills_the_rank_of_an_8_gpu_run(pkg, monkeypatch):
    """configs[4] at 8 GPUs: a rank owns 16 of the 128 row tiles of SK 16384.  One CTA per tile would leave 132 SMs idle;
    the plan splits every tile's K range so that >= 128 CTAs are busy (asserted from the plan, as the 8-GPU node is
    not available: `gpurun` has one GPU)."""
    from paper_2505_22631_b200 import dense_fused, workloads
    monkeypatch.delenv("OSCB_UMMA_SPLITK", raising=False)
    n, world = 16384, 8
    rows = n // world
    J8 = workloads.sk_dense(n)[:rows].astype(np.float64)
    params = pkg.SolverParams.tuned_for(n, 2, seed=0)
    rk = dense_fused.FusedDenseRank(J8, n, 0, rows, 0, params, 1, n * (n - 1) // 2, world, 0, steps=4)
    try:
        assert rk.rows == rows and rk.splits >= 8 and rk.ctas == 16 * rk.splits >= 128
    finally:
        rk.close()
