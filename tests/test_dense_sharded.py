"""Row-sharded dense driver (dense_sharded.py).

CPU part (not gpu): the orchestration -- row partition, per-step all-gather, all-reduced scoring,
cadence, sample schedule, best tracking -- runs on a world_size-2 gloo group with a float64
torch-CPU stand-in for the CUDA shard (test infrastructure only) and must reproduce the CPU
oracle's noise-free run.  GPU part: the CUDA shard kernels against the single-handle dense path."""
import math
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def sk_graph(n, seed, weights=(-1.0, 1.0)):
    rng = np.random.default_rng(seed)
    J = np.triu(rng.choice(np.array(weights), size=(n, n)), 1)
    return J + J.T


class CpuDenseShard:
    """float64 torch-CPU restatement of the shard step / objective / energy (tests only)."""

    def __init__(self, J_rows, n, row_begin, row_end):
        import torch
        self.torch = torch
        self.n, self.row_begin, self.row_end = n, row_begin, row_end
        self.J = torch.as_tensor(np.ascontiguousarray(J_rows, dtype=np.float64))
        self.device = 0

    def tensor(self, shape, dtype=None):
        return self.torch.zeros(shape, dtype=dtype or self.torch.float64)

    def from_host(self, a, dtype=None):
        return self.torch.as_tensor(np.array(a, dtype=np.float64))

    def seeds(self, seeds):
        return self.torch.zeros(len(seeds), dtype=self.torch.int64)

    def step(self, phi, out, seeds_dev, K, ks, h, kn_sqrt_h, n_states, noise_on, step):
        t = self.torch
        assert not noise_on
        c, s = t.cos(2 * math.pi * phi), t.sin(2 * math.pi * phi)
        ci, si = c[self.row_begin:self.row_end], s[self.row_begin:self.row_end]
        acc = si * (self.J @ c) - ci * (self.J @ s)
        p = phi[self.row_begin:self.row_end]
        x = p + h * (K * acc - ks * t.sin((2 * math.pi * n_states) * p))
        out.copy_(x - t.floor(x))

    def _states(self, phi, n_states):
        from paper_2505_22631_b200.model import _threshold
        return self.torch.as_tensor(_threshold(phi.numpy().T, n_states).T.copy())

    def objective(self, phi, n_states, maximize, out):
        t = self.torch
        st = self._states(phi, n_states)
        rows = t.arange(self.row_begin, self.row_end)
        upper = (t.arange(self.n)[None, :] > rows[:, None]).to(t.float64)
        for r in range(phi.shape[1]):
            same = (st[rows, r][:, None] == st[:, r][None, :]).to(t.float64)
            if maximize:
                out[r] = (self.J * upper * (1 - same)).sum()
            else:
                out[r] = ((self.J != 0).to(t.float64) * upper * same).sum()

    def energy(self, phi, out):
        t = self.torch
        rows = t.arange(self.row_begin, self.row_end)
        upper = (t.arange(self.n)[None, :] > rows[:, None]).to(t.float64)
        for r in range(phi.shape[1]):
            d = phi[rows, r][:, None] - phi[:, r][None, :]
            out[r] = (self.J * upper * t.cos(2 * math.pi * d)).sum()

    def nonfinite(self):
        return [-1, -1, -1]


def _case():
    import paper_2505_22631_b200 as pkg
    n = 32
    J = sk_graph(n, 3)
    params = pkg.SolverParams(K=0.05, ks_max=1.0, ks_period=1.0, kn=0.0, h=0.01, t_stop=2.5, seed=11)
    return n, J, params, [11, 12, 13]


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import pickle
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2505_22631_b200 import dense_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, J, params, seeds = _case()
    rows = n // world
    shard = CpuDenseShard(J[rank * rows:(rank + 1) * rows], n, rank * rows, (rank + 1) * rows)
    phi0 = np.stack([O.initial_phases(s, n) for s in seeds])
    res = dense_sharded.run_dense_sharded(shard, params, "maxcut", seeds, pair_count=n * (n - 1) // 2, phi0=phi0)
    with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump(res, f)
    dist.destroy_process_group()


def test_two_rank_gloo_orchestration_matches_oracle(tmp_path, oracle):
    import pickle
    import torch.multiprocessing as mp
    import paper_2505_22631_b200 as pkg
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    got = [pickle.load(open(tmp_path / f"rank{r}.pkl", "rb")) for r in range(2)]
    n, J, params, seeds = _case()
    Jc = pkg.CouplingMatrix.from_dense(J, storage="sparse")
    want = oracle.simulate(Jc.indptr, Jc.indices, Jc.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period,
                           kn=0.0, h=params.h, t_stop=params.t_stop, n_states=2, seeds=seeds, objective="maxcut")
    for r, res in enumerate(got):
        assert (res.rank, res.world, res.rows) == (r, 2, (r * n // 2, (r + 1) * n // 2))
        b = res.batch
        assert b.steps == want.steps == 250
        d = np.abs(b.final_phases - want.final_phases)
        assert (2 * np.pi * np.minimum(d, 1 - d)).max() < 1e-9
        assert np.array_equal(b.trace_t, want.trace_t) and np.array_equal(b.trace_ks, want.trace_ks)
        assert np.array_equal(b.best_objective, want.best_objective)
        assert np.array_equal(b.best_states.astype(np.int64), want.best_states)
        assert np.array_equal(b.best_trace, want.best_trace)
        assert np.abs(b.energy - want.energy).max() < 1e-8
    assert np.array_equal(got[0].batch.final_phases, got[1].batch.final_phases)


# ---------------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def pkg():
    import paper_2505_22631_b200 as p
    from paper_2505_22631_b200 import _native, dynamics
    assert _native.device_count() > 0, "no CUDA device: " + _native.last_error()
    old = dynamics.DENSE_DEVICE_MIN_N
    dynamics.DENSE_DEVICE_MIN_N = 0          # exercise the dense kernels on test-sized graphs
    yield p
    dynamics.DENSE_DEVICE_MIN_N = old


@pytest.mark.gpu
@pytest.mark.parametrize("weights", [(-1.0, 1.0), (0.0, 0.0, 1.0, -2.5, 0.75)])
def test_dense_handle_matches_oracle(pkg, oracle, weights):
    """Dense storage (int8 for +-1, float for general couplings) through the generic entry points
    vs the oracle on the CSR of the same couplings."""
    from paper_2505_22631_b200.dynamics import _step_raw
    from conftest import circ_dist_rad
    n = 70
    J = sk_graph(n, 5, weights)
    Jd = pkg.CouplingMatrix.from_dense(J, storage="dense")
    Js = pkg.CouplingMatrix.from_dense(J, storage="sparse")
    rng = np.random.default_rng(1)
    for R in (1, 11):
        phi = rng.random((R, n))
        noise = rng.standard_normal((R, n))
        want = oracle.step(Js.indptr, Js.indices, Js.data, phi, noise, 0.05, 0.7, 0.01, 0.03, 2)
        assert circ_dist_rad(_step_raw(Jd, phi, noise, 0.05, 0.7, 0.01, 0.03, 2, "f64", None), want).max() <= 1e-12
        assert circ_dist_rad(_step_raw(Jd, phi, noise, 0.05, 0.7, 0.01, 0.03, 2, "f32", None), want).max() <= 3e-6
        piu, pjv, pw = Js.pairs()
        for N, kind in ((2, "maxcut"), (3, "coloring")):
            ws, wo = oracle.score(phi, N, piu, pjv, pw, kind == "maxcut")
            gs, go = pkg.score_phases(Jd, phi, N, kind)
            assert np.array_equal(gs, ws)
            assert np.allclose(go, wo, rtol=0, atol=1e-9)
            if all(float(x).is_integer() for x in weights):
                assert np.array_equal(go, wo)
        en = np.array([oracle.continuous_energy(phi[r], piu, pjv, pw) for r in range(R)])
        assert np.abs(pkg.sample_energy(Jd, phi) - en).max() <= 1e-9 * max(1.0, np.abs(pw).sum())
    params = pkg.SolverParams(K=0.05, ks_max=1.0, ks_period=1.0, kn=0.0, h=0.01, t_stop=2.0, seed=4)
    seeds = [4, 5, 6]
    ref = oracle.simulate(Js.indptr, Js.indices, Js.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period,
                          kn=0.0, h=params.h, t_stop=params.t_stop, n_states=2, seeds=seeds, objective="maxcut")
    got = pkg.run_batch(Jd, params, "maxcut", seeds, precision="f64", kernel="stream")
    assert got.kernel == "stream"
    assert circ_dist_rad(got.final_phases, ref.final_phases).max() <= 1e-9          # N = 200 steps
    assert np.array_equal(got.best_objective, ref.best_objective)
    assert np.array_equal(got.best_states.astype(np.int64), ref.best_states)
    assert np.array_equal(got.trace_t, ref.trace_t)
    assert np.abs(got.energy - ref.energy).max() <= 1e-8
    short = pkg.run_batch(Jd, params, "maxcut", seeds, precision="f32", steps=30, kernel="stream")
    ref30 = pkg.run_batch(Jd, params, "maxcut", seeds, precision="f64", steps=30, kernel="stream")
    assert circ_dist_rad(short.final_phases, ref30.final_phases).max() <= 1e-4       # N = 30 steps


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_row_shards_reassemble_the_full_step(pkg, precision):
    """Two shard handles on one GPU (rows split in halves): their slices, concatenated, are the
    full handle's step bit for bit -- noise on, so the (seed, step, oscillator) indexing is checked
    across the shard boundary too."""
    import torch
    from paper_2505_22631_b200.dense_sharded import CudaDenseShard
    n, R = 96, 5
    J = sk_graph(n, 9)
    full = CudaDenseShard(J, n, 0, n, 0, precision)
    halves = [CudaDenseShard(J[:48], n, 0, 48, 0, precision), CudaDenseShard(J[48:], n, 48, 96, 0, precision)]
    phi = full.from_host(np.random.default_rng(2).random((n, R)))
    seeds = full.seeds([7, 8, 9, 10, 2**64 - 1])
    out_full = full.tensor((n, R))
    outs = [h.tensor((48, R)) for h in halves]
    args = (seeds, 0.05, 0.6, 0.01, 0.015, 2, True, 123)
    full.step(phi, out_full, *args)
    for h, o in zip(halves, outs):
        h.step(phi, o, *args)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs, dim=0), out_full)
    part_full = full.tensor((R,), torch.float64)
    parts = [h.tensor((R,), torch.float64) for h in halves]
    full.objective(phi, 2, True, part_full)
    for h, p_ in zip(halves, parts):
        h.objective(phi, 2, True, p_)
    torch.cuda.synchronize()
    assert torch.equal(parts[0] + parts[1], part_full)
    full.energy(phi, part_full)
    for h, p_ in zip(halves, parts):
        h.energy(phi, p_)
    torch.cuda.synchronize()
    assert torch.allclose(parts[0] + parts[1], part_full, rtol=0, atol=1e-9)
    assert full.nonfinite() == [-1, -1, -1]


@pytest.mark.gpu
def test_sharded_driver_equals_single_handle_run(pkg):
    """world = 1: the sharded loop (shard kernels + Python bookkeeping) reproduces oscb_run on the
    dense handle exactly, noise on."""
    from paper_2505_22631_b200.dense_sharded import CudaDenseShard, run_dense_sharded
    n = 64
    J = sk_graph(n, 21)
    Jd = pkg.CouplingMatrix.from_dense(J, storage="dense")
    params = pkg.SolverParams(K=0.05, ks_max=1.0, ks_period=1.0, kn=0.2, h=0.01, t_stop=1.5, seed=30)
    seeds = [30, 31, 32, 33]
    for precision in ("f32", "f64"):
        want = pkg.run_batch(Jd, params, "maxcut", seeds, precision=precision, kernel="stream")
        shard = CudaDenseShard(J, n, 0, n, 0, precision)
        got = run_dense_sharded(shard, params, "maxcut", seeds, pair_count=n * (n - 1) // 2).batch
        assert np.array_equal(got.final_phases, want.final_phases)
        assert np.array_equal(got.best_objective, want.best_objective)
        assert np.array_equal(got.best_states, want.best_states)
        assert np.array_equal(got.trace_t, want.trace_t)
        assert np.array_equal(got.best_trace, want.best_trace)
        assert np.abs(got.energy - want.energy).max() <= 1e-6 * n * n
