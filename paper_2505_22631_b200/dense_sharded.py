"""One oversized dense (all-to-all) graph, row-sharded over several GPUs.

Rank g holds the rows J[g*n/G:(g+1)*n/G, :] and owns the phases of those oscillators.  Every
Euler step each rank computes the new phases of ITS rows from the full (cos, sin) vector
(`oscb_dense_shard_step`, CUDA), then the slices are all-gathered (NCCL over NVLink through
`torch.distributed.all_gather_into_tensor`) into the next full phase array -- phases, not pairs,
travel (4 bytes per oscillator-replica; every rank rebuilds the pairs locally).  Scoring steps add
one all-reduce of R partial objectives.  All bookkeeping (best objective, best phases, traces) is
replicated on every rank from all-reduced values, so every rank returns the same result.

The loop mirrors the reference's `_simulate` (dynamics.py:333-431): same step count, sample
schedule, scoring cadence and strict-improvement rule.  The arithmetic lives behind a small
backend object so the orchestration can be exercised on CPU with a gloo group
(tests/test_dense_sharded.py); the product backend is `CudaDenseShard` (liboscb + torch device
tensors).  There is no CPU fallback in the product path.
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _native as nat
from .dynamics import (BatchResult, KsSchedule, NumericalError, _initial_phases_host, _objective_cadence_for,
                       _raise, _sample_steps)
from .model import SolverParams, _threshold


class CudaDenseShard:
    """The CUDA backend: one `oscb_graph` row shard on `device`, state in torch device tensors
    laid out [n][R] (oscillator-major, replica-minor) like the dense kernels expect."""

    def __init__(self, J_rows: np.ndarray, n: int, row_begin: int, row_end: int, device: int, precision: str = "f32"):
        import torch
        self.torch = torch
        self.n, self.row_begin, self.row_end = n, row_begin, row_end
        self.device = device
        self.precision = precision
        self.dtype = torch.float32 if precision == "f32" else torch.float64
        J_rows = np.ascontiguousarray(J_rows, dtype=np.float64)
        if J_rows.shape != (row_end - row_begin, n):
            raise ValueError(f"J_rows must have shape ({row_end - row_begin}, {n})")
        h = C.c_void_p()
        rc = nat.lib().oscb_graph_create_dense(device, n, nat.ptr(J_rows), row_begin, row_end, C.byref(h))
        if rc != nat.OK:
            _raise(rc, "oscb_graph_create_dense")
        self.handle = h

    def close(self):
        if self.handle:
            nat.lib().oscb_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def tensor(self, shape, dtype=None):
        return self.torch.empty(shape, dtype=dtype or self.dtype, device=f"cuda:{self.device}")

    def from_host(self, a: np.ndarray, dtype=None):
        return self.torch.as_tensor(a).to(device=f"cuda:{self.device}", dtype=dtype or self.dtype)

    def seeds(self, seeds: Sequence[int]):
        s = np.array([int(x) % 2**64 for x in seeds], dtype=np.uint64).view(np.int64)
        return self.torch.as_tensor(s).to(device=f"cuda:{self.device}")

    def _stream(self):
        return C.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def step(self, phi_full, phi_rows_out, seeds_dev, K, ks, h, kn_sqrt_h, n_states, noise_on, step):
        p = nat.ShardStepParams(K, ks, h, kn_sqrt_h, n_states, nat.PREC[self.precision], int(bool(noise_on)), 0, step)
        R = phi_full.shape[1]
        rc = nat.lib().oscb_dense_shard_step(self.handle, R, C.byref(p), C.c_void_p(phi_full.data_ptr()),
                                             C.c_void_p(phi_rows_out.data_ptr()), C.c_void_p(seeds_dev.data_ptr()),
                                             self._stream())
        if rc != nat.OK:
            _raise(rc, "oscb_dense_shard_step")

    def objective(self, phi_full, n_states, maximize, out):
        rc = nat.lib().oscb_dense_shard_objective(self.handle, phi_full.shape[1], nat.PREC[self.precision],
                                                  C.c_void_p(phi_full.data_ptr()), n_states, int(bool(maximize)),
                                                  C.c_void_p(out.data_ptr()), self._stream())
        if rc != nat.OK:
            _raise(rc, "oscb_dense_shard_objective")

    def energy(self, phi_full, out):
        rc = nat.lib().oscb_dense_shard_energy(self.handle, phi_full.shape[1], nat.PREC[self.precision],
                                               C.c_void_p(phi_full.data_ptr()), C.c_void_p(out.data_ptr()), self._stream())
        if rc != nat.OK:
            _raise(rc, "oscb_dense_shard_energy")

    def nonfinite(self):
        w = (C.c_int64 * 3)(-1, -1, -1)
        rc = nat.lib().oscb_graph_nonfinite(self.handle, w, 1)
        if rc != nat.OK:
            _raise(rc, "oscb_graph_nonfinite")
        return [int(x) for x in w]


@dataclass
class ShardedRun:
    batch: BatchResult
    rank: int
    world: int
    rows: tuple


def run_dense_sharded(backend, params: SolverParams, objective: str, seeds: Sequence[int], *,
                      pair_count: int, phi0: Optional[np.ndarray] = None, trace_stride: Optional[float] = None,
                      steps: Optional[int] = None, noise_off: bool = False, group=None) -> ShardedRun:
    """Integrate R = len(seeds) replicas of one dense graph whose rows are sharded over the ranks
    of `group` (default process group; a single process works too).  `backend` is this rank's
    shard (`CudaDenseShard`); `pair_count` is the number of coupled pairs of the WHOLE graph (it
    sets the scoring cadence, dynamics.py:325-330).  Every rank returns the same ShardedRun."""
    import torch
    import torch.distributed as dist

    if objective not in ("maxcut", "coloring"):
        raise ValueError(f"unknown objective kind: {objective!r}")
    if objective == "maxcut" and params.n_states != 2:
        raise ValueError("maxcut runs require n_states=2")
    have_group = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if have_group else 0
    world = dist.get_world_size(group) if have_group else 1
    n, R = backend.n, len(seeds)
    rows = backend.row_end - backend.row_begin
    if rows * world != n or backend.row_begin != rank * rows:
        raise ValueError("rows must be split evenly: rank r owns [r*n/world, (r+1)*n/world)")
    maximize = objective == "maxcut"
    stride = params.ks_period / 2.0 if trace_stride is None else float(trace_stride)
    if stride <= 0:
        raise ValueError("trace_stride must be > 0")
    nsteps = int(math.ceil(params.t_stop / params.h)) if steps is None else int(steps)
    cadence = _objective_cadence_for(n, pair_count)
    sample_after = set(_sample_steps(nsteps, params.h, stride))
    schedule = KsSchedule(params.ks_max, params.ks_period)
    kn_sqrt_h = params.kn * math.sqrt(params.h)
    noise_on = (not noise_off) and params.kn != 0.0

    if phi0 is None:
        phi0 = _initial_phases_host(getattr(backend, "device", 0), seeds, n)      # [R, n], the reference's stream
    phi = backend.from_host(np.ascontiguousarray(np.asarray(phi0, dtype=np.float64).reshape(R, n).T))   # [n][R]
    phi_next = backend.tensor((n, R))
    mine = backend.tensor((rows, R))
    seeds_dev = backend.seeds(seeds)
    f64 = torch.float64
    part = backend.tensor((R,), f64)
    best_obj = torch.full_like(part, -math.inf if maximize else math.inf)
    best_phi = phi.clone()
    trace_t: List[float] = []
    trace_ks: List[float] = []
    energies, bests = [], []

    def reduce_(t):
        if world > 1:
            dist.all_reduce(t, group=group)

    def score():
        nonlocal best_obj
        backend.objective(phi, params.n_states, maximize, part)
        reduce_(part)
        better = part > best_obj if maximize else part < best_obj
        best_obj = torch.where(better, part, best_obj)
        best_phi[:, better] = phi[:, better]

    def sample(t_now):
        score()
        en = backend.tensor((R,), f64)
        backend.energy(phi, en)
        reduce_(en)
        trace_t.append(t_now)
        trace_ks.append(schedule.value(t_now))
        energies.append(en)
        bests.append(best_obj.clone())

    t0 = time.perf_counter()
    sample(0.0)
    for step in range(nsteps):
        backend.step(phi, mine, seeds_dev, params.K, schedule.value(step * params.h), params.h, kn_sqrt_h,
                     params.n_states, noise_on, step)
        if world > 1:
            dist.all_gather_into_tensor(phi_next, mine, group=group)     # rank r's rows land at [r*rows, (r+1)*rows)
        else:
            phi_next.copy_(mine)
        phi, phi_next = phi_next, phi
        if step in sample_after:
            sample((step + 1) * params.h)
        elif step % cadence == 0:
            score()
    where = backend.nonfinite()
    flag = torch.tensor([where[2] if where[2] >= 0 else 2**62, where[0], where[1]], dtype=torch.int64,
                        device=part.device)
    if world > 1:
        gathered = [torch.zeros_like(flag) for _ in range(world)]
        dist.all_gather(gathered, flag, group=group)
        flag = min(gathered, key=lambda f: (int(f[0]), int(f[1]), int(f[2])))
    if int(flag[0]) < 2**62:
        raise NumericalError(f"non-finite phase for oscillator {int(flag[2])} (replica row {int(flag[1])}) "
                             f"after step {int(flag[0])}; parameters are numerically unstable")
    wall = time.perf_counter() - t0

    final = phi.to(f64).cpu().numpy().T.copy()                 # [R, n]
    bphi = best_phi.to(f64).cpu().numpy().T
    states = _threshold(bphi, params.n_states).astype(np.uint8)
    S = len(trace_t)
    b = BatchResult(final, states, best_obj.cpu().numpy().copy(), np.array(trace_t), np.array(trace_ks),
                    torch.stack(energies, dim=1).cpu().numpy() if S else np.zeros((R, 0)),
                    torch.stack(bests, dim=1).cpu().numpy() if S else np.zeros((R, 0)),
                    np.full(R, -1, dtype=np.int64), nsteps, 1e3 * wall, 0, "dense-sharded", 0, 0, wall)
    return ShardedRun(b, rank, world, (backend.row_begin, backend.row_end))
