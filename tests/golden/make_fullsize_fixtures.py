"""Generate tests/golden/fullsize_fixtures.npz: CPU-oracle results at the BENCHMARKED sizes.

    python tests/golden/make_fullsize_fixtures.py            (build container; ~10 min on 8 cores)

The arrays come from oracle/ (the C restatement of the reference algorithm, itself pinned bit for
bit against the unmodified reference by tests/golden/reference_vectors.npz) on the synthetic graphs
of bench.py's workloads.  They gate the GPU kernels at the sizes that are timed
(tests/test_fullsize_parity.py, `-m gpu`):

  g22_best / flat200_best / sk1024_best
        best_objective of independent noisy replicas over the WHOLE default schedule (numpy's own
        Philox + Ziggurat stream, dynamics.py:116-125) -- the samples of the two-sample tests;
  g22_target_best
        max of g22_best: the reference-anchored target of bench.py's time-to-99 %-best-cut;
  sk16384_*
        noise-free float64 phases of the dense +-1 SK graph (n = 16384, seed 0) after N Euler
        steps at the tuned K (chaotic: ~1 turn per step) and at K = 0.02 (contractive);
  flat200_u / flat200_v
        the edge list of the reference's own generate_colorable_graph(200, 479, 3, seed=0)
        (problems.py:255-276), imported unmodified, when /root/reference is present.
"""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2505_22631_b200 import workloads  # noqa: E402
from paper_2505_22631_b200.model import SolverParams  # noqa: E402

OUT = Path(__file__).resolve().parent / "fullsize_fixtures.npz"
G = {}
O.build()
T = O.max_threads()


def noisy_best(workload, seeds):
    shape, J, params, kind, _ = bench.load_workload(workload)
    t0 = time.perf_counter()
    r = O.simulate(J.indptr, J.indices, J.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period, kn=params.kn,
                   h=params.h, t_stop=params.t_stop, n_states=params.n_states, seeds=seeds, objective=kind, threads=T)
    print(f"{workload}: {len(seeds)} replicas x {r.steps} steps in {time.perf_counter() - t0:.1f} s, "
          f"best {r.best_objective.min()}..{r.best_objective.max()} mean {r.best_objective.mean():.2f}", flush=True)
    return r.best_objective, np.asarray(seeds, dtype=np.int64)


G["g22_best"], G["g22_seeds"] = noisy_best("G22x1024", list(range(10_000, 10_096)))
G["g22_target_best"] = np.array(G["g22_best"].max())
G["flat200_best"], G["flat200_seeds"] = noisy_best("flat200x4096", list(range(20_000, 20_256)))

# dense +-1 SK n = 1024, 4000 steps (tools/validate_distribution_dense.py's setting)
n = 1024
J8 = workloads.sk_dense(n)
indptr, indices, data = bench.dense_csr(J8)
p = SolverParams(K=0.05, ks_max=1.0, ks_period=4.0, kn=0.15, h=0.01, t_stop=40.0, seed=0)
seeds = list(range(50_000, 50_128))
t0 = time.perf_counter()
r = O.simulate(indptr, indices, data, K=p.K, ks_max=p.ks_max, ks_period=p.ks_period, kn=p.kn, h=p.h, t_stop=p.t_stop,
               n_states=2, seeds=seeds, objective="maxcut", threads=T)
print(f"SK1024: {len(seeds)} replicas x {r.steps} steps in {time.perf_counter() - t0:.1f} s", flush=True)
G["sk1024_best"], G["sk1024_seeds"] = r.best_objective, np.asarray(seeds, dtype=np.int64)

# dense +-1 SK n = 16384 (configs[4]), one replica (seed 0), noise-free
n = 16384
J8 = workloads.sk_dense(n)
indptr, indices, data = bench.dense_csr(J8)
tuned = SolverParams.tuned_for(n, 2, seed=0)
G["sk16384_tuned_K"] = np.array(tuned.K)
for tag, K, horizons in (("tuned", tuned.K, (1, 2, 3, 5, 10)), ("mild", 0.02, (10,))):
    for N in horizons:
        t0 = time.perf_counter()
        r = O.simulate(indptr, indices, data, K=K, ks_max=tuned.ks_max, ks_period=tuned.ks_period, kn=0.0, h=tuned.h,
                       t_stop=N * tuned.h, n_states=2, seeds=[0], objective="maxcut", threads=T)
        assert r.steps == N
        G[f"sk16384_{tag}_phi_N{N}"] = r.final_phases[0]
        G[f"sk16384_{tag}_best_N{N}"] = r.best_objective
        print(f"SK16384 {tag} K={K}: {N} steps in {time.perf_counter() - t0:.1f} s", flush=True)
del indptr, indices, data

ref_src = Path("/root/reference/pkg/src")
if ref_src.exists():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, str(ref_src))
    import oscim  # noqa: E402
    g = oscim.generate_colorable_graph(200, 479, 3, seed=0)
    G["flat200_u"], G["flat200_v"] = np.asarray(g.u, dtype=np.int64), np.asarray(g.v, dtype=np.int64)

G["meta_threads"] = np.array(T)
G["meta_numpy"] = np.array(np.__version__)
np.savez_compressed(OUT, **G)
print(f"wrote {OUT} ({OUT.stat().st_size / 1e3:.0f} kB, {len(G)} arrays)")
