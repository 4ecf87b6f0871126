"""Multi-GPU host logic on CPU: world_size-2 gloo process group, the per-rank integrator
replaced by the CPU oracle (test infrastructure) through the `runner` hook.  Checks the
replica partition, seed derivation, global replica indices and the best-of tie rule."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2505_22631_b200.sharding import best_of, shard_bounds  # noqa: E402


def test_shard_bounds_partition():
    for replicas in (1, 2, 7, 8, 1024, 1025):
        for world in (1, 2, 3, 8):
            blocks = [shard_bounds(replicas, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == replicas
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(4, 2, 2)


def oracle_runner(J, params, objective, seeds, trace_stride=None, **kw):
    """BatchResult produced by the CPU oracle instead of the GPU (tests only)."""
    from oracle import oracle as O
    from paper_2505_22631_b200.dynamics import BatchResult
    r = O.simulate(J.indptr, J.indices, J.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period,
                   kn=params.kn, h=params.h, t_stop=params.t_stop, n_states=params.n_states, seeds=list(seeds),
                   objective=objective, trace_stride=trace_stride)
    return BatchResult(r.final_phases, r.best_states.astype(np.uint8), r.best_objective, r.trace_t, r.trace_ks,
                       r.energy, r.best_trace, np.full(len(seeds), -1), r.steps, 0.0, 0, "oracle", 0, 0, 0.0)


def _problem():
    import paper_2505_22631_b200 as pkg
    from conftest import random_graph_arrays
    iu, iv, w = random_graph_arrays(24, 0.3, seed=5, weights=(1.0,))
    J = pkg.CouplingMatrix.from_edges(24, (iu, iv, w))
    params = pkg.SolverParams(K=0.5, ks_max=1.0, ks_period=1.0, kn=0.3, h=0.01, t_stop=2.0, seed=2**64 - 3)
    return J, params


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import pickle
    import torch.distributed as dist
    from paper_2505_22631_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    J, params = _problem()
    best = sharding.run_replicas_sharded(J, params, "maxcut", replicas=7, runner=oracle_runner)
    allr = sharding.run_replica_set_sharded(J, params, "maxcut", replicas=7, runner=oracle_runner)
    with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump((best, allr), f)
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_process(tmp_path):
    import pickle
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    got = [pickle.load(open(tmp_path / f"rank{r}.pkl", "rb")) for r in range(2)]
    # single-process ground truth: all 7 replicas at once
    from paper_2505_22631_b200 import sharding
    J, params = _problem()
    solo = sharding.run_replica_block(J, params, "maxcut", 7, rank=0, world=1, runner=oracle_runner)
    assert [r.replica_index for r in solo] == list(range(7))
    want_best = best_of(solo, "maxcut")
    for rank in range(2):
        best, allr = got[rank]
        assert best.replica_index == want_best.replica_index
        assert best.best_objective == want_best.best_objective
        assert np.array_equal(best.final_phases.phases, want_best.final_phases.phases)
    assert got[1][1] is None
    allr = got[0][1]
    assert [r.replica_index for r in allr] == list(range(7))
    for a, b in zip(allr, solo):
        assert np.array_equal(a.final_phases.phases, b.final_phases.phases)    # seeds wrap mod 2^64 correctly
        assert a.best_objective == b.best_objective and a.energy_trace == b.energy_trace


def test_best_of_tie_rule():
    from types import SimpleNamespace as NS
    rs = [NS(best_objective=5.0, replica_index=3), NS(best_objective=7.0, replica_index=2),
          NS(best_objective=7.0, replica_index=1), NS(best_objective=6.0, replica_index=0)]
    assert best_of(rs, "maxcut").replica_index == 1
    assert best_of(rs, "coloring").replica_index == 3
    assert best_of([], "maxcut") is None
