"""Generate tests/golden/reference_vectors.npz from the UNMODIFIED reference package.

Run in the build container only (the reference is mounted read-only at /root/reference and
does not exist on the GPU box):

    python tests/golden/make_golden.py

Every array is produced by importing `oscim` from /root/reference/pkg/src and calling its
public API / private kernels; nothing here comes from this repo's own code.  The vectors pin
the CPU oracle (oracle/oscim_oracle.c), which in turn checks the CUDA path.
Reference versions at generation time are recorded in the file (`meta_*`).
"""
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import numba  # noqa: E402
import numpy as np  # noqa: E402
import oscim  # noqa: E402
from oscim import dynamics as dyn  # noqa: E402
from oscim.model import CouplingMatrix, PhaseState, SolverParams, _threshold  # noqa: E402

OUT = Path(__file__).resolve().parent / "reference_vectors.npz"
G = {}


def random_graph_arrays(n, density, seed, weights=(-1.0, 1.0)):
    rng = np.random.default_rng(seed)
    iu, iv = np.triu_indices(n, 1)
    keep = rng.random(len(iu)) < density
    iu, iv = iu[keep], iv[keep]
    w = rng.choice(weights, size=len(iu))
    return iu.astype(np.int64), iv.astype(np.int64), w


def coupling(n, iu, iv, w):
    return CouplingMatrix.from_edges(n, list(zip(iu.tolist(), iv.tolist(), w.tolist())))


def put_graph(tag, J):
    G[f"{tag}_indptr"] = np.array(J.indptr)
    G[f"{tag}_indices"] = np.array(J.indices)
    G[f"{tag}_data"] = np.array(J.data)


# --- 1. initial phases (dynamics.py:127-129) ------------------------------------------------
init_seeds = np.array([0, 3, 12345678901234567, 2**64 - 1], dtype=np.uint64)
G["init_seeds"] = init_seeds
G["init_phases"] = np.stack([dyn.NoiseSource(int(s)).initial_phases(11) for s in init_seeds])

# --- 2. normal chunks (dynamics.py:116-125) -------------------------------------------------
G["normal_chunk_seed99_c1_n3"] = dyn.NoiseSource(99).normal_chunk(1, 3)
G["normal_chunk_seed5_c0_n4"] = dyn.NoiseSource(5).normal_chunk(0, 4)
G["normal_chunk_seedmax_c7_n17"] = dyn.NoiseSource(2**64 - 1).normal_chunk(7, 17)
G["step_normals_seed99_s300_n3"] = dyn.NoiseSource(99).step_normals(300, 3)
G["step_normals_seed99_s300_n4"] = dyn.NoiseSource(99).step_normals(300, 4)

# --- 3. schedule (dynamics.py:83-88) --------------------------------------------------------
ts = np.array([0.0, 0.3, 2.5, 5.0, 7.5, 9.99, 10.0, 12.5, 1234.567, 0.01 * 66874])
G["ks_t"] = ts
G["ks_val_2_10"] = np.array([dyn.KsSchedule(2.0, 10.0).value(float(t)) for t in ts])
G["ks_val_17_4"] = np.array([dyn.KsSchedule(1.7, 4.0).value(float(t)) for t in ts])

# --- 4. single steps (dynamics.py:286-314) --------------------------------------------------
# 4a: the reference's own kernel-vs-formula case (test_dynamics.py:157-173): 9 nodes, signed, N=3
iu, iv, w = random_graph_arrays(9, 0.6, seed=5)
J9 = coupling(9, iu, iv, w)
put_graph("g9", J9)
p9 = SolverParams(K=0.8, ks_max=1.2, ks_period=6.0, kn=0.4, h=0.02, t_stop=1.0, n_states=3, seed=21)
phi9 = PhaseState(np.random.default_rng(8).random(9))
G["g9_phi"] = np.array(phi9.phases)
G["g9_params"] = np.array([p9.K, p9.ks_max, p9.ks_period, p9.kn, p9.h, p9.t_stop, p9.n_states, p9.seed])
G["g9_t"] = np.array([1.7])
G["g9_step_index"] = np.array([170])
G["g9_noise"] = dyn.NoiseSource(p9.seed).step_normals(170, 9)
G["g9_out"] = np.array(dyn.euler_step(phi9, J9, p9, 1.7, dyn.NoiseSource(p9.seed), 170).phases)
G["g9_drift"] = np.array([dyn.phase_drift(J9, phi9, i, p9.K, dyn.KsSchedule(p9.ks_max, p9.ks_period).value(1.7), 3)
                          for i in range(9)])

# 4b: KAT3 of SURVEY 8c: weighted 5-ring, N=3, noise off
ring = [(0, 1, 1.0), (1, 2, -1.0), (2, 3, 1.0), (3, 4, 2.0), (0, 4, 1.0)]
J5 = CouplingMatrix.from_edges(5, ring)
put_graph("ring5", J5)
p5 = SolverParams(K=1.3, ks_max=1.7, ks_period=4.0, kn=0.0, h=0.01, t_stop=2.0, n_states=3, seed=0)
phi5 = PhaseState(np.array([0.05, 0.30, 0.55, 0.80, 0.95]))
G["ring5_phi"] = np.array(phi5.phases)
G["ring5_out"] = np.array(dyn.euler_step(phi5, J5, p5, 1.1, dyn.NoiseSource(0), 110).phases)
G["ring5_thresholds"] = _threshold(G["ring5_out"], 3)

# 4c: the reference's hand-computed pair (test_dynamics.py:143-154): (0.0, 0.25) -> (0.9, 0.35)
J2 = CouplingMatrix.from_edges(2, [(0, 1, 1.0)])
put_graph("pair2", J2)
p2 = SolverParams(K=1.0, ks_max=0.0, ks_period=10.0, kn=0.0, h=0.1, t_stop=1.0, n_states=2, seed=0)
G["pair2_out"] = np.array(dyn.euler_step(PhaseState(np.array([0.0, 0.25])), J2, p2, 0.0, dyn.NoiseSource(0), 0).phases)

# --- 5. score kernel (dynamics.py:193-223, test_dynamics.py:402-418) -------------------------
iu, iv, w = random_graph_arrays(40, 0.2, seed=11, weights=(1.0, 2.0, -1.0))
J40 = coupling(40, iu, iv, w)
put_graph("g40", J40)
rng = np.random.default_rng(3)
for N in (2, 3, 5):
    phi = rng.random((6, 40))
    lattice = np.arange(N) / N
    phi[0, :N] = lattice                              # exact lattice points
    phi[1, :N] = (lattice + 0.5 / N) % 1.0            # exact tie points
    phi[2, :4] = [0.25, 0.75, 0.5, 0.0]
    phi[3, :4] = np.nextafter([0.25, 0.75, 0.25, 0.75], [0, 0, 1, 1])
    piu, pjv, pw = J40.pairs()
    for maximize in (True, False):
        states = np.zeros((6, 40), dtype=np.int64)
        obj = np.zeros(6)
        dyn._score_kernel(phi, N, piu, pjv, pw, maximize, states, obj)
        G[f"score_N{N}_max{int(maximize)}_states"] = states
        G[f"score_N{N}_max{int(maximize)}_obj"] = obj
    G[f"score_N{N}_phi"] = phi
    G[f"score_N{N}_threshold"] = _threshold(phi, N)

# --- 6. whole runs (dynamics.py:333-431) -----------------------------------------------------
def put_run(tag, J, params, kind, replicas, stride=None):
    res = dyn.run_replica_set(J, params, kind, replicas=replicas, workers=1, trace_stride=stride)
    G[f"{tag}_params"] = np.array([params.K, params.ks_max, params.ks_period, params.kn, params.h,
                                   params.t_stop, params.n_states, params.seed])
    G[f"{tag}_final"] = np.stack([np.array(r.final_phases.phases) for r in res])
    G[f"{tag}_best_states"] = np.stack([np.array(r.best_assignment.states) for r in res])
    G[f"{tag}_best_obj"] = np.array([r.best_objective for r in res])
    G[f"{tag}_trace_t"] = np.array([t for t, _, _ in res[0].energy_trace])
    G[f"{tag}_trace_ks"] = np.array([k for _, _, k in res[0].energy_trace])
    G[f"{tag}_energy"] = np.stack([np.array([e for _, e, _ in r.energy_trace]) for r in res])
    G[f"{tag}_best_trace"] = np.stack([np.array(r.best_trace) for r in res])
    G[f"{tag}_steps"] = np.array([res[0].steps_executed])


# 6a: noise OFF, signed 30-node graph, max-cut, 3 replicas, 400 steps (trajectory parity target)
iu, iv, w = random_graph_arrays(30, 0.3, seed=2)
J30 = coupling(30, iu, iv, w)
put_graph("g30", J30)
put_run("run30_quiet", J30, SolverParams(K=0.5, ks_max=1.0, ks_period=2.0, kn=0.0, h=0.01, t_stop=4.0, seed=7), "maxcut", 3)
# 6b: noise ON (numpy Ziggurat stream), same graph: 300 steps crosses a 256-step chunk boundary
put_run("run30_noisy", J30, SolverParams(K=0.5, ks_max=1.0, ks_period=2.0, kn=0.3, h=0.01, t_stop=3.0, seed=7), "maxcut", 3)
# 6c: 3-colouring, planted graph, noise on, odd trace stride
gcol = oscim.generate_colorable_graph(24, 50, 3, seed=4)
Jc = oscim.build_coloring_coupling(gcol, 3)
put_graph("col24", Jc)
put_run("run_col24", Jc, SolverParams.tuned_for(24, 3, seed=11, t_stop=5.0, ks_period=1.0), "coloring", 2, stride=0.37)
# 6d: cadence / group helpers
G["cadence_cases"] = np.array([[800, 19176], [2000, 19990], [200, 479], [20000, 40000], [16384, 134209536],
                               [10, 5], [10, 15], [10, 25], [7, 0], [3, 1000]])
G["cadence_values"] = np.array([dyn._objective_cadence(int(n), int(m)) for n, m in G["cadence_cases"]])

G["meta_numpy"] = np.array(np.__version__)
G["meta_numba"] = np.array(numba.__version__)
G["meta_oscim"] = np.array(oscim.__version__)
np.savez_compressed(OUT, **G)
print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(G)} arrays)")
