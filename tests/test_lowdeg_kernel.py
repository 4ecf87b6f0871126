"""k_lowdeg and k_lowdeg_pair (csrc/oscb_lowdeg.cuh), the persistent float32 kernels that keep the phases in registers --
k_lowdeg for low-degree graphs (G81 shape, flat200), k_lowdeg_pair (two replicas per lane) for N = 2 max-cut at any degree
(the G22 headline): their stream compiler on the CPU, and on the GPU their trajectories against the oracle, the read-out
against the float64 threshold rule, the result contract, determinism, the noise contract, the noise-on distribution, the
kernel chooser, and the mixed-tile schedule that keeps all SMs busy."""
import ctypes as C

import numpy as np
import pytest

from conftest import circ_dist_rad


# ------------------------------------------------------------------------------------------------
# CPU: the stream compiler (no GPU needed)
def _plan(J, rt, warps, qpt, rpl=1):
    """rpl = 2: the plan of k_lowdeg_pair (two replicas per lane)."""
    from paper_2505_22631_b200 import _native as nat
    n = J.n
    plan_host = nat.lib().oscb_lowdeg_plan_host if rpl == 1 else nat.lib().oscb_lowdeg_pair_plan_host
    uniform, rows, entries = C.c_int32(), C.c_int64(), C.c_int64()
    ip, ix, w = (np.ascontiguousarray(J.indptr, dtype=np.int64), np.ascontiguousarray(J.indices, dtype=np.int64),
                 np.ascontiguousarray(J.data, dtype=np.float64))
    args = (n, nat.ptr(ip), nat.ptr(ix), nat.ptr(w), rt, warps, qpt)
    rc = plan_host(*args, C.byref(uniform), C.byref(rows), C.byref(entries), None, None, None, None, None)
    assert rc == 0, nat.last_error()
    Cq = 32 * rpl // rt
    quad_of = np.zeros(warps * qpt * Cq, dtype=np.uint32)
    slot_of = np.zeros(n, dtype=np.uint32)
    ids = np.zeros(4 * entries.value, dtype=np.uint32)
    w16 = np.zeros(4 * entries.value, dtype=np.float32)
    ws = np.zeros(warps, dtype=np.int32)
    rc = plan_host(*args, C.byref(uniform), C.byref(rows), C.byref(entries), nat.ptr(quad_of), nat.ptr(slot_of),
                   nat.ptr(ids), nat.ptr(w16), nat.ptr(ws))
    assert rc == 0, nat.last_error()
    return bool(uniform.value), rows.value, quad_of, slot_of, ids.reshape(-1, 4), w16.reshape(-1, 4), ws


def _graph(n, kind, seed=0):
    from paper_2505_22631_b200 import workloads
    from paper_2505_22631_b200.model import CouplingMatrix
    if kind == "torus":
        u, v, w = workloads.torus_pm1(n // 20, 20, seed=seed)
    elif kind == "sparse_pm":          # mean degree ~5, a few rows above 8 neighbours
        u, v, w = workloads.random_gnm(n, int(2.5 * n), seed=seed, weights=(1.0, -1.0, 2.0))
    else:                               # unit weights (colouring)
        u, v, w = workloads.random_gnm(n, int(2.4 * n), seed=seed)
    return CouplingMatrix.from_edges(n, (u, v, w))


@pytest.mark.parametrize("n,kind,rt,warps,qpt,rpl", [
    (400, "torus", 1, 2, 2, 1), (400, "torus", 8, 5, 5, 1), (203, "sparse_pm", 4, 7, 1, 1), (203, "sparse_pm", 32, 13, 4, 1),
    (200, "unit", 16, 5, 5, 1), (1001, "unit", 1, 4, 2, 1),
    (203, "sparse_pm", 4, 4, 1, 2), (203, "sparse_pm", 8, 2, 4, 2), (1001, "unit", 2, 4, 2, 2), (1001, "sparse_pm", 16, 13, 5, 2),
    (2000, "g22", 8, 16, 4, 2),
])
def test_stream_compiler_covers_the_csr(n, kind, rt, warps, qpt, rpl):
    """Every CSR entry (dynamics.py:166-170) appears exactly once in the stream, under the row that owns it,
    with its coupling; everything else is a zero-weight read of an all-zero pad slot; the slot map is a
    bijection onto component-major slots (k_lowdeg) / visiting-order-major slots (k_lowdeg_pair, whose quad table
    carries the order: the rows of a quad in descending degree)."""
    J = _graph(n, kind, seed=3) if kind != "g22" else __import__("bench").load_workload("G22x1024")[1]
    uniform, rows, quad_of, slot_of, ids, w, warp_start = _plan(J, rt, warps, qpt, rpl)
    Cq = 32 * rpl // rt
    Q, Qp = (n + 3) // 4, warps * qpt * Cq
    deg = np.diff(J.indptr)
    assert uniform == (deg.max() <= 4)
    # quad table: k_lowdeg_pair packs the visiting order of a quad's rows into the top byte
    sorted_rows = rpl == 2 and not uniform
    comp = np.tile(np.arange(4, dtype=np.int64), (len(quad_of), 1))
    if sorted_rows:
        real = (quad_of & 0xFFFFFF) < Q
        assert np.all(quad_of[~real] == 0xFFFFFFFF)
        comp = np.stack([(quad_of >> (24 + 2 * k)) & 3 for k in range(4)], axis=1).astype(np.int64)
        assert np.all(np.sort(comp[real], axis=1) == np.arange(4))
        quad_of = np.where(real, quad_of & 0xFFFFFF, 0xFFFFFFFF).astype(np.uint32)
        degp = np.concatenate([deg, np.zeros(4 * Q - n, dtype=deg.dtype)])
        for p_ in np.flatnonzero(real):
            d = degp[4 * int(quad_of[p_]) + comp[p_]]
            assert np.all(np.diff(d) <= 0)                                    # descending degree
    # slot map: the row visited k-th of the quad at position p sits at k * Qp + p (k = i & 3 for k_lowdeg)
    pos_of_quad = {int(q): p for p, q in enumerate(quad_of) if q < Q}
    assert sorted(pos_of_quad) == list(range(Q))
    for i in range(n):
        p_ = pos_of_quad[i >> 2]
        assert slot_of[i] == int(np.flatnonzero(comp[p_] == (i & 3))[0]) * Qp + p_
    osc_of_slot = {int(s): i for i, s in enumerate(slot_of)}
    last = (ids[:, 3] & 0x80000000) != 0 if not uniform else np.zeros(len(ids), dtype=bool)
    raw = ids.astype(np.int64)
    if not uniform:
        raw[:, 3] &= 0x7FFFFFFF
    assert np.all(raw % (8 * rt) == 0)
    slots = raw // (8 * rt)
    got = {i: [] for i in range(n)}

    def consume(entry, row):
        for u in range(4):
            s, wt = int(slots[entry, u]), float(w[entry, u])
            if s >= 4 * Qp:
                assert wt == 0.0 and s < 4 * Qp + 16
            else:
                assert row >= 0
                got[row].append((osc_of_slot[s], wt))

    def row_at(t, wp, c, k):
        p_ = (t * warps + wp) * Cq + c
        q = int(quad_of[p_])
        i = 4 * q + int(comp[p_, k])
        return i if q < Q and i < n else -1

    if uniform:
        assert len(ids) == qpt * warps * 4 * Cq
        for t in range(qpt):
            for wp in range(warps):
                for k in range(4):
                    for c in range(Cq):
                        consume(((t * warps + wp) * 4 + k) * Cq + c, row_at(t, wp, c, k))
    else:
        assert len(ids) == (rows + 1) * Cq
        for wp in range(warps):
            e = int(warp_start[wp])
            for t in range(qpt):
                for k in range(4):
                    while True:                      # the kernel's do { } while (!last)
                        for c in range(Cq):
                            consume(e * Cq + c, row_at(t, wp, c, k))
                        fin = last[e * Cq]
                        assert np.all(last[e * Cq:(e + 1) * Cq] == fin)       # the flag is warp-uniform
                        e += 1
                        if fin:
                            break
            assert e == (int(warp_start[wp + 1]) if wp + 1 < warps else rows)
    for i in range(n):
        want = sorted(zip(J.indices[J.indptr[i]:J.indptr[i + 1]].tolist(), J.data[J.indptr[i]:J.indptr[i + 1]].tolist()))
        assert sorted(got[i]) == want, i
    if kind == "g22":
        # the point of the two orderings: few padded reads, few shared-memory bank collisions.  An LDS.128 of 8 slots x 4
        # lanes is served two slots (a quarter-warp) per 128-byte wavefront unless both fall in the same bank half.
        assert J.nnz / (4.0 * len(ids)) > 0.88
        pair = slots[:-Cq].reshape(-1, Cq // 2, 2, 4)
        collide = ((pair[:, :, 0] % 2) == (pair[:, :, 1] % 2)) & (pair[:, :, 0] != pair[:, :, 1])
        assert collide.mean() < 0.07, collide.mean()          # (0.14 with each row ordered on its own, 0.40 in CSR order)


# ------------------------------------------------------------------------------------------------
# GPU
gpu = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2505_22631_b200 as p
    from paper_2505_22631_b200 import _native
    assert _native.device_count() > 0, "no CUDA device: " + _native.last_error()
    return p


def _objective(J, states, kind):
    iu, jv, w = J.pairs()
    s = states.astype(np.int64)
    if kind == "maxcut":
        return (w[None, :] * (s[:, iu] != s[:, jv])).sum(axis=1)
    return (s[:, iu] == s[:, jv]).sum(axis=1).astype(np.float64)


CASES = [
    # name, graph builder, N, objective, replicas, replicas_per_cta (0 = chooser), steps
    ("G81", lambda: __import__("bench").load_workload("G81x296")[1], 2, "maxcut", 3, 0, 20),
    ("flat200", lambda: __import__("bench").load_workload("flat200x4096")[1], 3, "coloring", 37, 0, 100),
    ("flat200-rt32", lambda: __import__("bench").load_workload("flat200x4096")[1], 3, "coloring", 40, 32, 100),
    ("flat200-rt1", lambda: __import__("bench").load_workload("flat200x4096")[1], 3, "coloring", 3, 1, 100),
    ("torus400", lambda: _graph(400, "torus", 1), 2, "maxcut", 9, 8, 20),
    ("sparse203", lambda: _graph(203, "sparse_pm", 2), 2, "maxcut", 5, 4, 20),
    ("sparse1001", lambda: _graph(1001, "sparse_pm", 4), 2, "maxcut", 2, 1, 20),
    ("unit1001", lambda: _graph(1001, "unit", 5), 3, "coloring", 6, 2, 60),
    # the headline route: 1024 replicas of the degree-20 G22 shape go to k_lowdeg_pair with the slot stream in shared memory
    ("G22x1024", lambda: __import__("bench").load_workload("G22x1024")[1], 2, "maxcut", 1024, 0, 20),
]


@gpu
@pytest.mark.parametrize("name,build,N,kind,R,rt,steps", CASES, ids=[c[0] for c in CASES])
def test_noise_free_trajectory_and_readout_vs_oracle(pkg, oracle, name, build, N, kind, R, rt, steps):
    """Noise off: float32 phases within 1e-4 rad of the oracle's float64 trajectory after the stated N steps
    (SURVEY 7-A horizons), the energy trace within float32 accuracy, and the read-out exact: the best objective
    is the objective of the reported best states, and every trace sample's best-so-far follows the reference's
    strict-improvement rule on the oracle's objectives up to read-out ties."""
    J = build()
    tune = dict(K=0.2, ks_max=1.0, kn=0.0) if N == 2 else dict(kn=0.0)
    params = pkg.SolverParams.tuned_for(J.n, N, seed=11, **tune)
    seeds = [params.seed + r for r in range(R)]
    stride = steps * params.h / 4.5                      # 5 trace samples + the initial one
    want = oracle.simulate(J.indptr, J.indices, J.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period, kn=0.0,
                           h=params.h, t_stop=steps * params.h, n_states=N, seeds=seeds, objective=kind, trace_stride=stride,
                           threads=oracle.max_threads())
    got = pkg.run_batch(J, params, kind, seeds, kernel="lowdeg", steps=steps, replicas_per_cta=rt, trace_stride=stride)
    assert got.kernel == "lowdeg" and got.steps == steps == want.steps
    assert rt == 0 or got.replicas_per_cta == rt
    assert circ_dist_rad(got.final_phases, want.final_phases).max() <= 1e-4, name          # N = steps, float32
    assert np.array_equal(got.trace_t, want.trace_t) and np.array_equal(got.trace_ks, want.trace_ks)
    assert got.energy.shape == want.energy.shape and got.energy.shape[1] >= 5
    scale = np.abs(J.data).sum() / 2
    assert np.abs(got.energy - want.energy).max() <= 2e-5 * scale, name
    assert np.array_equal(_objective(J, got.best_states, kind), got.best_objective)
    sign = 1 if kind == "maxcut" else -1
    assert np.all(sign * np.diff(got.best_trace, axis=1) >= 0)
    # a phase within 1e-4 rad of a decision boundary may read out differently in float32: allow a few edges
    assert np.abs(got.best_objective - want.best_objective).max() <= max(2.0, 2e-3 * scale), name
    assert np.abs(got.best_trace - want.best_trace).max() <= max(2.0, 2e-3 * scale), name


@gpu
@pytest.mark.parametrize("N,kind", [(2, "maxcut"), (3, "coloring")])
def test_readout_is_the_float64_threshold_rule_on_the_stored_phase(pkg, N, kind):
    """K3 of north_star: given identical phases, states and cut / conflict counts are bit-exact.  A one-step
    noise-free run takes two samples (t = 0 and the last step); both read-outs must equal the reference rule
    (dynamics.py:203-213) evaluated in float64 on the float32 phases the kernel holds -- lattice and tie
    points included."""
    J = _graph(403, "sparse_pm" if N == 2 else "unit", 7)
    R = 6
    rng = np.random.default_rng(1)
    phi0 = rng.random((R, J.n)).astype(np.float32).astype(np.float64)
    lattice = np.array([0.0, 0.25, 0.5, 0.75, 1 / 6, 1 / 3, 2 / 3, 5 / 6, 0.24999999, 0.7500001], dtype=np.float32).astype(np.float64)
    phi0[:, :80] = rng.choice(lattice, size=(R, 80))
    params = pkg.SolverParams(K=0.05, ks_max=0.5, ks_period=1.0, kn=0.0, h=0.01, t_stop=1.0, n_states=N, seed=0)
    b = pkg.run_batch(J, params, kind, list(range(R)), kernel="lowdeg", steps=1, phi0=phi0, noise_off=True)
    assert b.kernel == "lowdeg" and b.best_trace.shape[1] == 2
    s0, o0 = pkg.score_phases(J, phi0, N, kind)
    s1, o1 = pkg.score_phases(J, b.final_phases, N, kind)
    assert np.array_equal(b.best_trace[:, 0], o0)
    better = o1 > o0 if kind == "maxcut" else o1 < o0
    assert np.array_equal(b.best_objective, np.where(better, o1, o0))
    assert np.array_equal(b.best_states.astype(np.int64), np.where(better[:, None], s1, s0))


@gpu
def test_determinism_replica_independence_and_tile_shape_independence(pkg):
    """Same call twice is bit-identical (energy trace included); a replica inside a batch equals its solo run on the same
    tile shape (test_dynamics.py:257-267); and where rows are summed in CSR order -- uniform graphs, N = 3, one replica per
    lane -- the result does not depend on the tile shape at all (test_dynamics.py:320-341).  (k_lowdeg_pair visits a row's
    neighbours in a bank-friendly order that depends on the tile shape, so its float32 last bits do.)"""
    J = _graph(600, "sparse_pm", 9)
    params = pkg.SolverParams.tuned_for(J.n, 2, seed=40, K=0.2, ks_max=1.0, kn=0.15, t_stop=3.0)
    seeds = [40 + r for r in range(7)]
    a = pkg.run_batch(J, params, "maxcut", seeds, kernel="lowdeg", replicas_per_cta=4)
    b = pkg.run_batch(J, params, "maxcut", seeds, kernel="lowdeg", replicas_per_cta=4)
    for f in ("final_phases", "best_states", "best_objective", "energy", "best_trace"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    solo = pkg.run_batch(J, params, "maxcut", [43], kernel="lowdeg", replicas_per_cta=4)
    assert np.array_equal(solo.final_phases[0], a.final_phases[3]) and solo.best_objective[0] == a.best_objective[3]
    assert np.array_equal(solo.energy[0], a.energy[3]) and np.array_equal(solo.best_states[0], a.best_states[3])
    for Jt, kind, N in ((_graph(400, "torus", 5), "maxcut", 2), (_graph(300, "unit", 6), "coloring", 3)):
        pt = pkg.SolverParams.tuned_for(Jt.n, N, seed=7, t_stop=2.0)
        runs = [pkg.run_batch(Jt, pt, kind, seeds, kernel="lowdeg", replicas_per_cta=rt) for rt in (1, 4, 16)]
        for r in runs[1:]:
            assert np.array_equal(r.final_phases, runs[0].final_phases) and np.array_equal(r.best_objective, runs[0].best_objective)
            assert np.array_equal(r.best_states, runs[0].best_states)


@gpu
@pytest.mark.parametrize("n,rt", [(203, 4), (600, 8), (1001, 2)])
def test_pair_kernel_noise_is_a_function_of_seed_step_and_oscillator(pkg, monkeypatch, n, rt):
    """k_lowdeg_pair walks the rows of a quad in descending degree; the noise an oscillator gets must still be component
    i mod 4 of the Philox block of quad i / 4 (the device noise contract every kernel shares): with noise ON a few steps of
    the pair kernel and of the per-step streaming kernel agree to float32 rounding, phases and read-out."""
    J = _graph(n, "sparse_pm", 31)
    params = pkg.SolverParams.tuned_for(J.n, 2, seed=3, K=0.2, ks_max=1.0, kn=0.3)
    seeds = [3 + r for r in range(2 * rt + 1)]
    monkeypatch.setenv("OSCB_LOWDEG_RPL", "2")
    a = pkg.run_batch(J, params, "maxcut", seeds, kernel="lowdeg", steps=6, replicas_per_cta=rt)
    monkeypatch.delenv("OSCB_LOWDEG_RPL")
    b = pkg.run_batch(J, params, "maxcut", seeds, kernel="stream", steps=6, precision="f32")
    assert a.kernel == "lowdeg" and b.kernel == "stream" and a.replicas_per_cta == rt
    assert circ_dist_rad(a.final_phases, b.final_phases).max() <= 2e-5
    assert np.array_equal(_objective(J, a.best_states, "maxcut"), a.best_objective)
    assert np.abs(a.best_objective - b.best_objective).max() <= 4.0


@gpu
def test_mixed_tile_schedule_is_the_same_run(pkg, oracle, monkeypatch):
    """1024 replicas of the G22 shape are 128 tiles of 8 on 148 SMs; the run is therefore cut into windows in which 20 of
    the 128 octets take turns as 4-replica tiles on the idle SMs (plan_mixed_tiles).  With windows of a few steps forced:
    the noise-free trajectory, the energy trace and the read-out still follow the oracle, the schedule is deterministic, and
    with noise ON it stays next to the unbroken launch (same noise per (seed, step, oscillator); only the float32 summation
    order differs between the tile shapes)."""
    import bench
    _, J, _, kind, R = bench.load_workload("G22x1024")
    steps = 64
    params = pkg.SolverParams.tuned_for(J.n, 2, seed=5, K=0.2, ks_max=1.0, kn=0.0)
    seeds = [params.seed + r for r in range(R)]
    stride = steps * params.h / 4.5
    monkeypatch.setenv("OSCB_LOWDEG_MIXED_MIN_WINDOW", "1")
    got = pkg.run_batch(J, params, kind, seeds, steps=steps, trace_stride=stride)
    assert got.kernel == "lowdeg" and got.kernel_launches >= 64 and got.steps == steps        # 32 windows x (tiles of 8 | tiles of 4)
    sub = list(range(0, R, 37))                                   # octets of every phase of the rotation
    want = oracle.simulate(J.indptr, J.indices, J.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period, kn=0.0,
                           h=params.h, t_stop=steps * params.h, n_states=2, seeds=[seeds[r] for r in sub], objective=kind,
                           trace_stride=stride, threads=oracle.max_threads())
    assert circ_dist_rad(got.final_phases[sub], want.final_phases).max() <= 1e-4
    assert np.array_equal(got.trace_t, want.trace_t)
    scale = np.abs(J.data).sum() / 2
    assert np.abs(got.energy[sub] - want.energy).max() <= 2e-5 * scale
    assert np.array_equal(_objective(J, got.best_states, kind), got.best_objective)
    assert np.all(np.diff(got.best_trace, axis=1) >= 0)
    assert np.abs(got.best_objective[sub] - want.best_objective).max() <= max(2.0, 2e-3 * scale)
    again = pkg.run_batch(J, params, kind, seeds, steps=steps, trace_stride=stride)
    for f in ("final_phases", "best_states", "best_objective", "energy", "best_trace"):
        assert np.array_equal(getattr(got, f), getattr(again, f)), f
    # noise on: next to the unbroken launch
    noisy = pkg.SolverParams.tuned_for(J.n, 2, seed=5, K=0.2, ks_max=1.0, kn=0.15)
    a = pkg.run_batch(J, noisy, kind, seeds, steps=steps, want_states=False)
    monkeypatch.setenv("OSCB_LOWDEG_MIXED", "0")
    b = pkg.run_batch(J, noisy, kind, seeds, steps=steps, want_states=False)
    assert a.kernel_launches >= 64 and b.kernel_launches == 1 and b.kernel == "lowdeg"
    assert circ_dist_rad(a.final_phases, b.final_phases).max() <= 2e-4
    assert np.abs(a.best_objective - b.best_objective).max() <= 6.0


@gpu
def test_mixed_tile_schedule_one_replica_per_lane(pkg, oracle, monkeypatch):
    """The same schedule for k_lowdeg: flat200 x 4096 is 128 tiles of 32 replicas -> windows of 108 tiles of 32 and 40 of 16
    (N = 3 colouring).  Forced to windows of a few steps: the noise-free run follows the oracle, read-out and traces included,
    and stays within float32 rounding of the unbroken launch, noise on or off (a step that also reads the previous state out
    is a separately compiled variant of the update, and a window boundary changes which steps those are)."""
    import bench
    _, J, _, kind, R = bench.load_workload("flat200x4096")
    steps = 96
    params = pkg.SolverParams.tuned_for(J.n, 3, seed=9, kn=0.0)
    seeds = [params.seed + r for r in range(R)]
    stride = steps * params.h / 4.5
    monkeypatch.setenv("OSCB_LOWDEG_MIXED_MIN_WINDOW", "1")
    got = pkg.run_batch(J, params, kind, seeds, steps=steps, trace_stride=stride)
    assert got.kernel == "lowdeg" and got.kernel_launches >= 64 and got.steps == steps
    sub = list(range(0, R, 97))
    want = oracle.simulate(J.indptr, J.indices, J.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period, kn=0.0,
                           h=params.h, t_stop=steps * params.h, n_states=3, seeds=[seeds[r] for r in sub], objective=kind,
                           trace_stride=stride, threads=oracle.max_threads())
    assert circ_dist_rad(got.final_phases[sub], want.final_phases).max() <= 1e-4
    assert np.array_equal(_objective(J, got.best_states, kind), got.best_objective)
    assert np.all(np.diff(got.best_trace, axis=1) <= 0)
    assert np.abs(got.best_objective[sub] - want.best_objective).max() <= 2.0
    monkeypatch.setenv("OSCB_LOWDEG_MIXED", "0")
    solo = pkg.run_batch(J, params, kind, seeds, steps=steps, trace_stride=stride)
    assert solo.kernel_launches == 1
    d = circ_dist_rad(got.final_phases, solo.final_phases)
    assert d.max() <= 2e-4 and np.quantile(d, 0.999) <= 1e-5          # (measured: 4e-5 / 2e-6 rad after 96 steps)
    assert np.abs(got.best_objective - solo.best_objective).max() <= 2.0 and np.array_equal(got.trace_t, solo.trace_t)
    noisy = pkg.SolverParams.tuned_for(J.n, 3, seed=9)
    b = pkg.run_batch(J, noisy, kind, seeds, steps=steps)
    monkeypatch.delenv("OSCB_LOWDEG_MIXED")
    a = pkg.run_batch(J, noisy, kind, seeds, steps=steps)
    assert a.kernel_launches >= 64 and b.kernel_launches == 1
    d = circ_dist_rad(a.final_phases, b.final_phases)
    assert d.max() <= 1e-3 and np.quantile(d, 0.999) <= 2e-5
    assert np.array_equal(_objective(J, a.best_states, kind), a.best_objective)


@gpu
@pytest.mark.parametrize("N,kind", [(2, "maxcut"), (3, "coloring")])
def test_noise_on_distribution_matches_the_oracle(pkg, oracle, N, kind):
    """Noise ON (device Philox vs numpy's stream replayed by the oracle): best objectives over 128 seeds agree in
    distribution; the full-size versions are tests/test_fullsize_parity.py."""
    from scipy import stats
    J = _graph(120, "sparse_pm" if N == 2 else "unit", 21)
    params = pkg.SolverParams.tuned_for(J.n, N, seed=500, t_stop=12.0, **(dict(K=0.2, ks_max=1.0, kn=0.15) if N == 2 else {}))
    seeds = [500 + r for r in range(128)]
    want = oracle.simulate(J.indptr, J.indices, J.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period,
                           kn=params.kn, h=params.h, t_stop=params.t_stop, n_states=N, seeds=seeds, objective=kind,
                           threads=oracle.max_threads())
    got = pkg.run_batch(J, params, kind, seeds, kernel="lowdeg")
    assert got.kernel == "lowdeg"
    assert stats.ks_2samp(got.best_objective, want.best_objective).pvalue > 0.01
    assert abs(got.best_objective.mean() - want.best_objective.mean()) < 0.6 * (want.best_objective.std() + 0.5)
    assert np.array_equal(_objective(J, got.best_states, kind), got.best_objective)


@gpu
def test_auto_selection_and_fallbacks(pkg):
    """The chooser takes the low-degree kernel for the G81 / flat200 shapes in float32, leaves float64 parity mode,
    the degree-20 G22 shape and non-integer couplings to the other kernels, and an explicit request that does
    not apply is a ValueError."""
    import bench
    from paper_2505_22631_b200 import workloads
    _, J81, p81, _, _ = bench.load_workload("G81x296")
    assert pkg.run_batch(J81, p81, "maxcut", [0, 1], steps=4).kernel == "lowdeg"
    assert pkg.run_batch(J81, p81, "maxcut", [0, 1], steps=4, precision="f64").kernel != "lowdeg"
    _, Jf, pf, _, _ = bench.load_workload("flat200x4096")
    assert pkg.run_batch(Jf, pf, "coloring", list(range(64)), steps=4).kernel == "lowdeg"
    _, J22, p22, _, _ = bench.load_workload("G22x1024")
    assert pkg.run_batch(J22, p22, "maxcut", list(range(64)), steps=4).kernel == "resident"
    # ... unless the batch fills the GPU with 8-replica tiles whose slot stream fits in shared memory: k_lowdeg_pair
    big = pkg.run_batch(J22, p22, "maxcut", list(range(1024)), steps=4, want_phases=False, want_states=False)
    assert big.kernel == "lowdeg" and big.replicas_per_cta == 8
    mid = pkg.run_batch(J22, p22, "maxcut", list(range(512)), steps=4, want_phases=False, want_states=False)
    assert mid.kernel == "lowdeg" and mid.replicas_per_cta == 4          # tiles of 4 while they fit one per SM
    assert pkg.run_batch(J22, p22, "maxcut", list(range(8)), steps=4, kernel="lowdeg").kernel == "lowdeg"      # on request: any degree
    with pytest.raises(ValueError):
        pkg.run_batch(J22, p22, "maxcut", [0], steps=4, kernel="lowdeg", precision="f64")                      # float32 only
    u, v, w = workloads.random_gnm(300, 700, seed=1, weights=(0.5, 1.25))
    Jw = pkg.CouplingMatrix.from_edges(300, (u, v, w))
    assert pkg.run_batch(Jw, p22, "maxcut", [0, 1], steps=4).kernel != "lowdeg"


@gpu
def test_nonfinite_phase_is_reported(pkg):
    """dynamics.py:276-283: a non-finite phase raises NumericalError naming oscillator and step."""
    J = _graph(400, "torus", 3)
    params = pkg.SolverParams(K=1e308, ks_max=1.0, ks_period=1.0, kn=0.0, h=0.5, t_stop=4.0, seed=1)      # h K overflows float32
    with pytest.raises(pkg.NumericalError, match=r"oscillator \d+ .* step \d+"):
        pkg.run_batch(J, params, "maxcut", [1, 2], kernel="lowdeg", noise_off=True)
