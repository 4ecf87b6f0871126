"""Multi-GPU execution of the replica batch: one process per GPU, contiguous replica blocks.

Replica r of a run depends only on (J, params, seed + r) (reference dynamics.py:243-247,
test_dynamics.py:257-267), so replicas shard across ranks with NO data-path collective: every
rank uploads the (small) graph, integrates its own block on its own GPU and keeps its results.
The only communication is the final best-of reduction -- 16 bytes per rank -- done with
`torch.distributed` (NCCL on GPUs, gloo in the CPU tests), with the reference's tie rule
(strict improvement, ties to the lowest replica index, dynamics.py:507-513).

The single oversized dense graph (SK 16384) is the one case with a per-step exchange; its
row-sharded kernel lives with the dense path (multi-GPU).
"""
from __future__ import annotations

import time
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from .dynamics import (BatchResult, RunResult, _default_device, _results_from_batch, _validate_run_args, replica_seed,
                       resolve_workers, run_batch)
from .model import CouplingMatrix, SolverParams

Runner = Callable[..., BatchResult]
MAX_REPLICAS_PER_CALL = 65536          # oscb_run's limit (include/oscb.h)


def shard_bounds(replicas: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block [start, stop) of replica indices owned by `rank`; the first
    `replicas % world` ranks hold one extra replica."""
    if replicas < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard arguments")
    base, extra = divmod(replicas, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def _dist():
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return None
    return dist


def run_replica_block(J: CouplingMatrix, params: SolverParams, objective: str, replicas: int, *,
                      rank: int, world: int, runner: Optional[Runner] = None, **run_kw) -> List[RunResult]:
    """This rank's share of `run_replica_set`: results carry GLOBAL replica indices."""
    _validate_run_args(J, params, objective)
    if replicas < 1:
        raise ValueError("replicas must be >= 1")
    start, stop = shard_bounds(replicas, world, rank)
    if stop == start:
        return []
    # oscb_run takes at most 65536 replicas per call: chunk the block like run_replica_set does
    out: List[RunResult] = []
    for lo in range(start, stop, MAX_REPLICAS_PER_CALL):
        hi = min(stop, lo + MAX_REPLICAS_PER_CALL)
        seeds = [replica_seed(params.seed, r) for r in range(lo, hi)]
        b = (runner or run_batch)(J, params, objective, seeds, **run_kw)
        out.extend(_results_from_batch(J, params, objective, b, lo))
    return out


def best_of(results: Sequence[RunResult], objective: str) -> Optional[RunResult]:
    """Strict improvement in replica-index order: ties go to the lowest index (dynamics.py:507-513)."""
    best = None
    for res in sorted(results, key=lambda r: r.replica_index):
        if best is None or ((res.best_objective > best.best_objective) if objective == "maxcut"
                            else (res.best_objective < best.best_objective)):
            best = res
    return best


def run_replicas_sharded(J: CouplingMatrix, params: SolverParams, objective: str = "maxcut", replicas: int = 1,
                         workers: Optional[int] = None, trace_stride: Optional[float] = None, *,
                         runner: Optional[Runner] = None, **run_kw) -> RunResult:
    """`run_replicas` across all ranks of the default process group (every rank returns the
    same winner).  Without an initialised group it is the single-GPU `run_replicas`."""
    import torch

    resolve_workers(workers)
    dist = _dist()
    rank, world = (dist.get_rank(), dist.get_world_size()) if dist else (0, 1)
    t0 = time.perf_counter()
    mine = run_replica_block(J, params, objective, replicas, rank=rank, world=world, runner=runner,
                             trace_stride=trace_stride, **run_kw)
    local = best_of(mine, objective)
    if dist is None:
        local.wall_time = time.perf_counter() - t0
        return local
    # (objective, replica index) per rank; ranks without replicas send a sentinel
    worst = -np.inf if objective == "maxcut" else np.inf
    # the GPU this rank computes on (OSCB_DEVICE / LOCAL_RANK, or the caller's `device`), not torch's current device:
    # without a set_device every rank's "cuda" would be cuda:0 and NCCL would see one GPU twice
    dev = torch.device("cuda", int(run_kw.get("device", _default_device()) or 0)) if dist.get_backend() == "nccl" else "cpu"
    mine_t = torch.tensor([local.best_objective if local else worst, float(local.replica_index) if local else -1.0],
                          dtype=torch.float64, device=dev)
    gathered = [torch.zeros_like(mine_t) for _ in range(world)]
    dist.all_gather(gathered, mine_t)
    table = [(float(t[0]), int(t[1]), rk) for rk, t in enumerate(gathered) if int(t[1]) >= 0]
    table.sort(key=lambda x: x[1])
    win = table[0]
    for cand in table[1:]:
        if (cand[0] > win[0]) if objective == "maxcut" else (cand[0] < win[0]):
            win = cand
    box = [local if rank == win[2] else None]
    dist.broadcast_object_list(box, src=win[2])
    best = box[0]
    best.wall_time = time.perf_counter() - t0
    return best


def run_replica_set_sharded(J: CouplingMatrix, params: SolverParams, objective: str = "maxcut", replicas: int = 1,
                            workers: Optional[int] = None, trace_stride: Optional[float] = None, *,
                            runner: Optional[Runner] = None, **run_kw) -> Optional[List[RunResult]]:
    """`run_replica_set` across all ranks; the full list (replica order) is returned on rank 0,
    None elsewhere."""
    resolve_workers(workers)
    dist = _dist()
    rank, world = (dist.get_rank(), dist.get_world_size()) if dist else (0, 1)
    mine = run_replica_block(J, params, objective, replicas, rank=rank, world=world, runner=runner,
                             trace_stride=trace_stride, **run_kw)
    if dist is None:
        return mine
    parts = [None] * world if rank == 0 else None
    dist.gather_object(mine, parts, dst=0)
    if rank != 0:
        return None
    out = [r for part in parts for r in part]
    out.sort(key=lambda r: r.replica_index)
    return out
