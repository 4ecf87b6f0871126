"""Pins the CPU oracle (oracle/oscim_oracle.c) against golden vectors generated from the
unmodified reference (tests/golden/make_golden.py) and the reference's own known-answer tests.
CPU only.  The oracle is what the GPU parity tests compare the CUDA path with."""
import math

import numpy as np
import pytest

from conftest import graph_from_golden, circ_dist_rad


def test_philox_block_kat(oracle):
    # raw Philox4x64-10 words at counter (1<<192)+1, key [3, 0]
    words = oracle.philox4x64_10((1 << 192) + 1, 3)
    assert [hex(int(w)) for w in words] == ["0xe1633a65f2ad86f5", "0x3a933285b9f5adb8",
                                            "0xc970c00d25c690ac", "0x46d9331aeecaac8"]


def test_initial_phases_bit_exact(oracle, golden):
    for s, want in zip(golden["init_seeds"], golden["init_phases"]):
        got = oracle.initial_phases(int(s), want.shape[0])
        assert np.array_equal(got, want)
    assert oracle.initial_phases(3, 4).tolist() == [0.8804203509231936, 0.22880855336003114,
                                                    0.786876681527952, 0.01729698145838887]


def test_normal_chunks_bit_exact(oracle, golden):
    assert np.array_equal(oracle.normal_chunk(99, 1, 3), golden["normal_chunk_seed99_c1_n3"])
    assert np.array_equal(oracle.normal_chunk(5, 0, 4), golden["normal_chunk_seed5_c0_n4"])
    assert np.array_equal(oracle.normal_chunk(2**64 - 1, 7, 17), golden["normal_chunk_seedmax_c7_n17"])
    # layout depends on n (SURVEY divergence 2)
    assert np.array_equal(oracle.step_normals(99, 300, 3), golden["step_normals_seed99_s300_n3"])
    assert np.array_equal(oracle.step_normals(99, 300, 4), golden["step_normals_seed99_s300_n4"])
    assert oracle.step_normals(99, 300, 3).tolist() == [0.4828444880671921, 0.433666223898129, -0.2630520333695628]


def test_schedule(oracle, golden):
    for t, a, b in zip(golden["ks_t"], golden["ks_val_2_10"], golden["ks_val_17_4"]):
        assert oracle.ks_value(2.0, 10.0, float(t)) == a
        assert oracle.ks_value(1.7, 4.0, float(t)) == b
    # reference test_dynamics.py:52-58
    assert oracle.ks_value(2.0, 10.0, 0.0) == 0.0
    assert oracle.ks_value(2.0, 10.0, 5.0) == 2.0
    assert oracle.ks_value(2.0, 10.0, 2.5) == pytest.approx(1.0)
    assert oracle.ks_value(2.0, 10.0, 7.5) == pytest.approx(1.0)
    assert oracle.ks_value(2.0, 10.0, 10.0) == 0.0


def test_cadence(oracle, golden):
    for (n, m), want in zip(golden["cadence_cases"], golden["cadence_values"]):
        assert oracle.objective_cadence(int(n), int(m)) == want


def test_step_kats(oracle, golden):
    # reference test_dynamics.py:143-154: (0.0, 0.25) -> (0.9, 0.35)
    ip, ix, d = graph_from_golden(golden, "pair2")
    out = oracle.step(ip, ix, d, np.array([[0.0, 0.25]]), None, 1.0, 0.0, 0.1, 0.0, 2)[0]
    assert out == pytest.approx([0.9, 0.35], abs=1e-12)
    assert np.abs(out - golden["pair2_out"]).max() <= 1e-15
    # SURVEY 8c KAT3
    ip, ix, d = graph_from_golden(golden, "ring5")
    out = oracle.step(ip, ix, d, golden["ring5_phi"][None], None, 1.3, 0.935, 0.01, 0.0, 3)[0]
    assert np.abs(out - golden["ring5_out"]).max() <= 1e-15
    assert out == pytest.approx([0.037076899382396396, 0.3314957921089346, 0.5315643088974058,
                                 0.7864697660373168, 0.9709575424713522], abs=1e-15)


def test_step_noisy_n3(oracle, golden):
    # reference test_dynamics.py:157-173 case: euler_step output and the formula-level drift
    ip, ix, d = graph_from_golden(golden, "g9")
    K, ks_max, ks_period, kn, h, _, N, seed = golden["g9_params"]
    t, idx = float(golden["g9_t"][0]), int(golden["g9_step_index"][0])
    noise = oracle.step_normals(int(seed), idx, 9)
    assert np.array_equal(noise, golden["g9_noise"])
    ks = oracle.ks_value(ks_max, ks_period, t)
    out = oracle.step(ip, ix, d, golden["g9_phi"][None], noise[None], K, ks, h, kn * math.sqrt(h), int(N))[0]
    assert np.abs(out - golden["g9_out"]).max() <= 1e-15
    want = golden["g9_phi"] + h * golden["g9_drift"] + kn * math.sqrt(h) * noise
    want -= np.floor(want)
    assert np.abs(out - want).max() <= 1e-12


@pytest.mark.parametrize("N", [2, 3, 5])
def test_score_kernel(oracle, golden, N):
    ip, ix, d = graph_from_golden(golden, "g40")
    iu, jv, w = oracle.pairs_from_csr(ip, ix, d)
    phi = golden[f"score_N{N}_phi"]
    for maximize in (1, 0):
        states, obj = oracle.score(phi, N, iu, jv, w, maximize)
        assert np.array_equal(states, golden[f"score_N{N}_max{maximize}_states"])
        assert np.array_equal(obj, golden[f"score_N{N}_max{maximize}_obj"])
    assert np.array_equal(states, golden[f"score_N{N}_threshold"])


def _run_case(oracle, golden, graph, tag, kind, replicas, stride=None):
    ip, ix, d = graph_from_golden(golden, graph)
    K, ks_max, ks_period, kn, h, t_stop, N, seed = golden[f"{tag}_params"]
    seeds = [(int(seed) + r) % 2**64 for r in range(replicas)]
    return oracle.simulate(ip, ix, d, K=K, ks_max=ks_max, ks_period=ks_period, kn=kn, h=h, t_stop=t_stop,
                           n_states=int(N), seeds=seeds, objective=kind, trace_stride=stride)


@pytest.mark.parametrize("graph,tag,kind,replicas,stride", [
    ("g30", "run30_quiet", "maxcut", 3, None),
    ("g30", "run30_noisy", "maxcut", 3, None),
    ("col24", "run_col24", "coloring", 2, 0.37),
])
def test_whole_runs(oracle, golden, graph, tag, kind, replicas, stride):
    res = _run_case(oracle, golden, graph, tag, kind, replicas, stride)
    assert res.steps == int(golden[f"{tag}_steps"][0])
    assert np.array_equal(res.trace_t, golden[f"{tag}_trace_t"])
    assert np.array_equal(res.trace_ks, golden[f"{tag}_trace_ks"])
    # libm vs numpy sin/cos differ by <= 1 ulp per call; a few hundred steps stay far below 1e-9 rad
    assert circ_dist_rad(res.final_phases, golden[f"{tag}_final"]).max() < 1e-9
    assert np.array_equal(res.best_states, golden[f"{tag}_best_states"])
    assert np.array_equal(res.best_objective, golden[f"{tag}_best_obj"])
    assert np.array_equal(res.best_trace, golden[f"{tag}_best_trace"])
    assert np.abs(res.energy - golden[f"{tag}_energy"]).max() < 1e-8


def test_golden_provenance(golden):
    assert str(golden["meta_oscim"]) == "0.1.0"


def test_fullsize_fixture_reproduces(oracle):
    """tests/golden/fullsize_fixtures.npz (the oracle's results at the benchmarked sizes) is what the oracle
    built here produces: the first replicas of the flat200 whole-schedule fixture, bit for bit."""
    from pathlib import Path
    import bench
    fix = np.load(Path(__file__).resolve().parent / "golden" / "fullsize_fixtures.npz")
    _, J, params, kind, _ = bench.load_workload("flat200x4096")
    seeds = [int(s) for s in fix["flat200_seeds"][:6]]
    r = oracle.simulate(J.indptr, J.indices, J.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period,
                        kn=params.kn, h=params.h, t_stop=params.t_stop, n_states=3, seeds=seeds, objective=kind,
                        threads=oracle.max_threads())
    assert np.array_equal(r.best_objective, fix["flat200_best"][:6])
    assert float(fix["g22_target_best"]) == fix["g22_best"].max() and len(fix["g22_best"]) >= 64
