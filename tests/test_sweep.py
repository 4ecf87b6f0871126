"""The batched K x ks_max sweep (paper_2505_22631_b200/sweep.py; reference cli.py:283-324): cell sharding over a
world_size-2 gloo group with the CPU oracle as the per-cell integrator, and on the GPU the concurrent cells against
the one-cell-at-a-time path."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from paper_2505_22631_b200 import sweep as sw  # noqa: E402
from test_sharding import oracle_runner  # noqa: E402


def test_cells_of_rank_partition_the_grid():
    for n_cells in (1, 5, 16):
        for world in (1, 2, 3, 8):
            got = sorted(c for r in range(world) for c in sw.cells_of_rank(n_cells, world, r))
            assert got == list(range(n_cells))
    with pytest.raises(ValueError):
        sw.cells_of_rank(4, 2, 2)


def _problem():
    import paper_2505_22631_b200 as pkg
    from conftest import random_graph_arrays
    iu, iv, w = random_graph_arrays(20, 0.3, seed=8, weights=(1.0,))
    J = pkg.CouplingMatrix.from_edges(20, (iu, iv, w))
    labels, cells = sw.grid_cells(20, 2, 5, [0.3, 0.6, 0.9], [0.5, 1.0], {"t_stop": 1.5, "kn": 0.2})
    return J, labels, cells


def _runner(J, params, objective, seeds, graph=None, device=None, want_states=True, want_traces=True, **kw):
    return oracle_runner(J, params, objective, seeds)


def test_grid_cells_follow_the_reference_order():
    _, labels, cells = _problem()
    assert labels == [(0.3, 0.5), (0.3, 1.0), (0.6, 0.5), (0.6, 1.0), (0.9, 0.5), (0.9, 1.0)]
    assert all(c.seed == 5 and c.t_stop == 1.5 and c.kn == 0.2 for c in cells)
    assert [(c.K, c.ks_max) for c in cells] == labels


def _worker(rank, world, port, out_dir):
    import pickle
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    J, labels, cells = _problem()
    got = sw.run_cells_sharded(J, cells, "maxcut", 3, runner=_runner, concurrency=2)
    with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump(got, f)
    dist.destroy_process_group()


def test_two_rank_gloo_sweep_equals_the_sequential_one(tmp_path):
    import pickle
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    got0, got1 = (pickle.load(open(tmp_path / f"rank{r}.pkl", "rb")) for r in range(2))
    assert got1 is None and len(got0) == 6
    J, labels, cells = _problem()
    want = sw.run_cells(J, cells, "maxcut", 3, runner=_runner, concurrency=1)      # one cell after another, one process
    for a, b in zip(got0, want):
        assert np.array_equal(a, b) and a.shape == (3,)


@pytest.mark.gpu
def test_concurrent_cells_equal_one_cell_at_a_time():
    """A cell's replicas see the same seeds and kernels whatever runs beside them: the concurrent sweep equals the
    sequential one number for number, and equals run_replica_set + the host read-out of the reference's cmd_sweep."""
    import paper_2505_22631_b200 as pkg
    from paper_2505_22631_b200 import workloads
    from paper_2505_22631_b200.model import Graph, cut_value, threshold_phases
    u, v, w = workloads.random_gnm(300, 1500, seed=2)
    J = pkg.CouplingMatrix.from_edges(300, (u, v, w))
    labels, cells = sw.grid_cells(300, 2, 11, [0.1, 0.2, 0.4], [0.5, 1.0, 1.5], {"t_stop": 4.0})
    together = sw.run_cells(J, cells, "maxcut", 6, concurrency=5)
    alone = sw.run_cells(J, cells, "maxcut", 6, concurrency=1)
    g = Graph(300, u, v, w)
    for p, a, b in zip(cells, together, alone):
        assert np.array_equal(a, b)
        ref = [cut_value(g, threshold_phases(r.final_phases, 2)) for r in pkg.run_replica_set(J, p, "maxcut", replicas=6)]
        assert np.array_equal(a, np.array(ref))
