"""The K x ks_max sweep as ONE batched, multi-GPU workload (reference cli.py:283-324).

Every cell of the heat map is `replicas` independent replicas of the SAME graph with its own (K, ks_max) -- the
reference runs the cells strictly one after another.  Here

  * the cells shard across the ranks of the process group (cell c goes to rank c mod world; no data-path
    collective, the per-cell scores are gathered once at the end) -- replicas and cells are both independent units
    (dynamics.py:243-247);
  * inside a rank the cells run CONCURRENTLY: each worker thread owns a device handle of the graph (its own CUDA
    stream) and drives whole solves through the C ABI, which releases the GIL; a cell of a few replicas occupies a few
    SMs, so the persistent kernels of many cells share the GPU instead of queueing behind one another;
  * a cell's score is the reference's: the objective of the FINAL thresholded state of every replica (not the
    best-of harvest), thresholded and counted on the device (`oscb_score`).

A cell's result does not depend on what runs beside it (same seeds, same kernels), so the heat map equals the
sequential one number for number.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as nat
from .dynamics import BatchResult, DeviceGraph, _default_device, _raise, replica_seed, run_batch
from .model import CouplingMatrix, SolverParams

CellRunner = Callable[..., BatchResult]


def cells_of_rank(n_cells: int, world: int, rank: int) -> List[int]:
    """Round-robin: neighbouring cells (similar cost) land on different ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard arguments")
    return list(range(rank, n_cells, world))


def final_state_objective(graph: DeviceGraph, phases: np.ndarray, n_states: int, objective: str) -> np.ndarray:
    """Objective of the thresholded FINAL phases of every replica (cli.py:310-322), on the device."""
    phi = np.ascontiguousarray(phases, dtype=np.float64)
    R, n = phi.shape
    states = np.empty((R, n), dtype=np.int64)
    obj = np.empty(R, dtype=np.float64)
    rc = nat.lib().oscb_score(graph.handle, R, nat.ptr(phi), n_states, int(objective == "maxcut"), nat.ptr(states), nat.ptr(obj))
    if rc != nat.OK:
        _raise(rc, "oscb_score")
    return obj


def run_cells(J: CouplingMatrix, cells: Sequence[SolverParams], objective: str, replicas: int, *,
              device: Optional[int] = None, concurrency: Optional[int] = None, runner: Optional[CellRunner] = None,
              **run_kw) -> List[np.ndarray]:
    """Final-state objectives [replicas] of every cell (one SolverParams each), the cells running concurrently on
    `device`.  `runner(J, params, objective, seeds, graph=..., **run_kw) -> BatchResult` replaces the GPU integrator
    in the CPU tests."""
    if replicas < 1:
        raise ValueError("replicas must be >= 1")
    if not cells:
        return []
    device = _default_device() if device is None else device
    workers = max(1, min(len(cells), concurrency or int(os.environ.get("OSCB_SWEEP_CONCURRENCY", "8"))))
    integrate = runner or run_batch

    def make_graph():
        if runner is not None:
            return None
        return DeviceGraph.from_csr(device, J.n, J.indptr, J.indices, J.data)

    graphs = [make_graph() for _ in range(workers)]          # one handle (one stream) per worker thread
    free = list(range(workers))

    def one(params: SolverParams) -> np.ndarray:
        slot = free.pop()                                    # (list.pop / append are atomic under the GIL)
        try:
            g = graphs[slot]
            seeds = [replica_seed(params.seed, r) for r in range(replicas)]
            b = integrate(J, params, objective, seeds, graph=g, device=device, want_states=False, want_traces=False, **run_kw)
            if g is None:
                from .model import PhaseState, threshold_phases       # CPU test path: the host rule
                s = np.stack([threshold_phases(PhaseState(p), params.n_states).states for p in b.final_phases])
                iu, jv, w = J.pairs()
                return ((w[None, :] * (s[:, iu] != s[:, jv])).sum(axis=1) if objective == "maxcut"
                        else (s[:, iu] == s[:, jv]).sum(axis=1).astype(np.float64))
            return final_state_objective(g, b.final_phases, params.n_states, objective)
        finally:
            free.append(slot)

    try:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            return list(pool.map(one, cells))
    finally:
        for g in graphs:
            if g is not None:
                g.close()


def run_cells_sharded(J: CouplingMatrix, cells: Sequence[SolverParams], objective: str, replicas: int, **kw) -> Optional[List[np.ndarray]]:
    """`run_cells` across the ranks of the default process group: rank r integrates cells r, r + world, ...; the
    complete list (cell order) is returned on rank 0, None elsewhere.  Without a group: the single-GPU run."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return run_cells(J, cells, objective, replicas, **kw)
    rank, world = dist.get_rank(), dist.get_world_size()
    mine_idx = cells_of_rank(len(cells), world, rank)
    mine = run_cells(J, [cells[c] for c in mine_idx], objective, replicas, **kw)
    parts: Optional[List] = [None] * world if rank == 0 else None
    dist.gather_object(list(zip(mine_idx, mine)), parts, dst=0)
    if rank != 0:
        return None
    out: List[Optional[np.ndarray]] = [None] * len(cells)
    for part in parts:
        for c, obj in part:
            out[c] = obj
    return out


def grid_cells(n: int, n_states: int, seed: int, K_values: Sequence[float], ks_values: Sequence[float],
               overrides: Optional[dict] = None) -> Tuple[List[Tuple[float, float]], List[SolverParams]]:
    """The cells of a K x ks_max grid in the reference's order (K outer, ks_max inner; the same base seed in every
    cell so replica r sees the same noise stream everywhere, cli.py:299-309)."""
    over = dict(overrides or {})
    labels = [(K, ks) for K in K_values for ks in ks_values]
    return labels, [SolverParams.tuned_for(n, n_states=n_states, seed=seed, **{**over, "K": K, "ks_max": ks}) for K, ks in labels]
