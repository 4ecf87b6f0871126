"""One oversized dense graph, row-sharded over several GPUs, FUSED.

Rank g holds the 128-row aligned shard J[row_begin:row_end, :] (integer couplings |J| <= 127) and
runs ONE persistent tensor-core kernel for the whole integration (`csrc/oscb_umma.cuh`).  The
per-step exchange is inside the kernel: the epilogue of every Euler step stores the new (cos, sin)
digit planes of the rank's rows into EVERY rank's next-step image through peer-mapped memory
(NVLink / NVSwitch), adds its part of the cut into every rank's event record with system-scope
atomics and arrives on every rank's step counter -- the all-gather and the all-reduce of
`dense_sharded.run_dense_sharded` (one kernel launch + one NCCL call per step, driven from Python)
become stores and atomics of the compute kernel.  The host only sets the run up:

    create -> export -> (all-gather the 96-byte blobs) -> connect -> prepare -> (barrier) -> launch -> finish

`torch.distributed` carries the blobs, the barrier and the final gather of the row slices (any
backend; nothing on the data path).  The same protocol runs several "virtual ranks" inside one
process (tests: two shards on one GPU, bit-identical to the single-handle run).

Mirrors the reference's `_simulate` (dynamics.py:333-431): same steps, sample schedule, scoring
cadence, strict-improvement best tracking and traces.
"""
from __future__ import annotations

import ctypes as C
import math
import time
from typing import List, Optional, Sequence

import numpy as np

from . import _native as nat
from .dynamics import BatchResult, _initial_phases_host, _raise, _sample_capacity
from .model import SolverParams

MAX_REPLICAS = 28      # replicas per session on the int8 stream (9 B columns per replica)


class FusedDenseRank:
    """One rank's session: a dense int8 row shard on `device` + the exchange block of one run of
    R <= 28 replicas."""

    def __init__(self, J_rows: np.ndarray, n: int, row_begin: int, row_end: int, device: int, params: SolverParams,
                 R: int, pair_count: int, world: int, rank: int, *, precision: str = "f32", steps: Optional[int] = None,
                 trace_stride: Optional[float] = None, noise_off: bool = False, first_step: int = 0, graph=None,
                 stream_bits: int = 0):
        self.n, self.row_begin, self.row_end, self.device = n, row_begin, row_end, device
        self.R, self.world, self.rank = R, world, rank
        self.own_graph = graph is None
        if graph is None:
            J_rows = np.ascontiguousarray(J_rows, dtype=np.float64)
            if J_rows.shape != (row_end - row_begin, n):
                raise ValueError(f"J_rows must have shape ({row_end - row_begin}, {n})")
            h = C.c_void_p()
            rc = nat.lib().oscb_graph_create_dense(device, n, nat.ptr(J_rows), row_begin, row_end, C.byref(h))
            if rc != nat.OK:
                _raise(rc, "oscb_graph_create_dense")
            graph = h
        self.graph = graph
        stride = params.ks_period / 2.0 if trace_stride is None else float(trace_stride)
        if stride <= 0:
            raise ValueError("trace_stride must be > 0")
        self.nsteps = int(math.ceil(params.t_stop / params.h)) if steps is None else int(steps)
        self.cap = _sample_capacity(self.nsteps, params.h, stride)
        p = nat.RunParams()
        p.K, p.ks_max, p.ks_period, p.kn = params.K, params.ks_max, params.ks_period, params.kn
        p.h, p.t_stop, p.n_states = params.h, params.t_stop, params.n_states
        p.objective = nat.OBJ["maxcut"]
        p.precision = nat.PREC[precision]
        p.noise_mode = nat.NOISE_NONE if noise_off else nat.NOISE_DEVICE
        p.kernel = nat.KERNEL["dense-tc"]
        p.steps = self.nsteps if steps is not None else 0
        p.trace_stride = stride
        p.first_step = int(first_step)
        if stream_bits not in (0, 4, 8):
            raise ValueError("stream_bits must be 0 (this shard's own choice), 4 (packed e2m1) or 8 (int8)")
        p.variant = int(stream_bits)               # the stream all ranks agreed on (agree_stream); 0 = this shard's own choice
        self.handle = C.c_void_p()
        rc = nat.lib().oscb_dense_fused_create(self.graph, C.byref(p), R, pair_count, world, rank, C.byref(self.handle))
        if rc != nat.OK:
            self.handle = None
            self.close()
            _raise(rc, "oscb_dense_fused_create")
        rows = C.c_int64(0)
        nat.lib().oscb_dense_fused_rows(self.handle, C.byref(rows))
        self.rows = int(rows.value)
        ctas, splits = C.c_int32(0), C.c_int32(0)
        nat.lib().oscb_dense_fused_grid(self.handle, C.byref(ctas), C.byref(splits))
        self.ctas, self.splits = int(ctas.value), int(splits.value)      # CTAs of this rank's kernel; CTAs per row tile (split-K)

    def close(self):
        if getattr(self, "handle", None):
            nat.lib().oscb_dense_fused_destroy(self.handle)
            self.handle = None
        if getattr(self, "own_graph", False) and getattr(self, "graph", None):
            nat.lib().oscb_graph_destroy(self.graph)
            self.graph = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export(self) -> bytes:
        buf = C.create_string_buffer(nat.FUSED_MEM_BYTES)
        rc = nat.lib().oscb_dense_fused_export(self.handle, buf)
        if rc != nat.OK:
            _raise(rc, "oscb_dense_fused_export")
        return buf.raw

    def connect(self, blobs: Sequence[bytes]):
        if len(blobs) != self.world or any(len(b) != nat.FUSED_MEM_BYTES for b in blobs):
            raise ValueError("connect needs one exchange blob per rank, in rank order")
        joined = C.create_string_buffer(b"".join(blobs), nat.FUSED_MEM_BYTES * self.world)
        rc = nat.lib().oscb_dense_fused_connect(self.handle, joined)
        if rc != nat.OK:
            _raise(rc, "oscb_dense_fused_connect")

    def prepare(self, seeds: Sequence[int], phi0: Optional[np.ndarray] = None):
        s = np.array([int(x) % 2**64 for x in seeds], dtype=np.uint64)
        if len(s) != self.R:
            raise ValueError(f"need {self.R} seeds")
        if phi0 is not None:
            phi0 = np.ascontiguousarray(phi0, dtype=np.float64).reshape(self.R, self.n)
        rc = nat.lib().oscb_dense_fused_prepare(self.handle, nat.ptr(s), nat.ptr(phi0))
        if rc != nat.OK:
            _raise(rc, "oscb_dense_fused_prepare")

    def launch(self):
        rc = nat.lib().oscb_dense_fused_launch(self.handle)
        if rc != nat.OK:
            _raise(rc, "oscb_dense_fused_launch")

    def finish(self) -> BatchResult:
        """This rank's rows of the final phases / best states ([R, rows]); objectives, traces and
        energies of the whole graph."""
        R, cap = self.R, self.cap
        final = np.empty((R, self.rows), dtype=np.float64)
        states = np.empty((R, self.rows), dtype=np.uint8)
        best = np.empty(R, dtype=np.float64)
        tt = np.zeros(cap); tks = np.zeros(cap)
        en = np.zeros((R, cap)); bt = np.zeros((R, cap))
        first = np.full(R, -1, dtype=np.int64)
        o = nat.RunOutputs()
        o.final_phases, o.best_states, o.best_objective = nat.ptr(final), nat.ptr(states), nat.ptr(best)
        o.trace_t, o.trace_ks, o.energy, o.best_trace = nat.ptr(tt), nat.ptr(tks), nat.ptr(en), nat.ptr(bt)
        o.first_hit_step = nat.ptr(first)
        o.max_samples = cap
        t0 = time.perf_counter()
        rc = nat.lib().oscb_dense_fused_finish(self.handle, C.byref(o))
        wall = time.perf_counter() - t0
        if rc != nat.OK:
            _raise(rc, "oscb_dense_fused_finish")
        S = int(o.n_samples)
        return BatchResult(final, states, best, tt[:S].copy(), tks[:S].copy(), en[:, :S].copy(), bt[:, :S].copy(), first,
                           int(o.steps_executed), float(o.device_ms), int(o.kernel_launches), "dense-tc",
                           int(o.replicas_per_cta), int(o.smem_bytes), wall)


def shard_stream_bits(graph, n_states: int, R: int) -> int:
    """Bits per coupling this shard would stream on its own for a call of R replicas: 4 (packed e2m1: every coupling of
    THESE rows in {0, +-1, +-2, +-3, +-4, +-6} and R small enough) or 8 (int8)."""
    bits, per = C.c_int32(0), C.c_int32(0)
    rc = nat.lib().oscb_dense_tc_stream(graph, n_states, R, C.byref(bits), C.byref(per))
    if rc != nat.OK:
        _raise(rc, "oscb_dense_tc_stream")
    return int(bits.value)


def agree_stream(local_bits: Sequence[int]) -> int:
    """The stream of a row-sharded run: every rank writes phase digits into every peer's B image, so all ranks must use
    ONE layout -- packed e2m1 only if every shard can take it, else int8 everywhere."""
    return 4 if all(b == 4 for b in local_bits) else 8


def assemble(parts: Sequence[BatchResult]) -> BatchResult:
    """Concatenate the ranks' row slices (rank order) into the result of the whole graph."""
    p0 = parts[0]
    return BatchResult(np.concatenate([p.final_phases for p in parts], axis=1),
                       np.concatenate([p.best_states for p in parts], axis=1),
                       p0.best_objective, p0.trace_t, p0.trace_ks, p0.energy, p0.best_trace, p0.first_hit_step, p0.steps,
                       max(p.device_ms for p in parts), sum(p.kernel_launches for p in parts), "dense-tc",
                       p0.replicas_per_cta, p0.smem_bytes, max(p.wall_time for p in parts))


def run_fused_in_process(shards: Sequence[tuple], n: int, params: SolverParams, seeds: Sequence[int], *,
                         pair_count: int, device: int = 0, phi0: Optional[np.ndarray] = None, **kw) -> BatchResult:
    """All ranks of a fused run driven from ONE process (several GPUs, or several virtual ranks on
    one GPU when every rank's CTAs fit on it together).  shards = [(J_rows, row_begin, row_end,
    device), ...] in rank order."""
    world = len(shards)
    ranks: List[FusedDenseRank] = []
    graphs = []
    try:
        # upload the shards first and agree on one stream for all of them
        for J, rb, re, dev in shards:
            h = C.c_void_p()
            rc = nat.lib().oscb_graph_create_dense(dev, n, nat.ptr(np.ascontiguousarray(J, dtype=np.float64)), rb, re, C.byref(h))
            if rc != nat.OK:
                _raise(rc, "oscb_graph_create_dense")
            graphs.append(h)
        bits = agree_stream([shard_stream_bits(h, params.n_states, len(seeds)) for h in graphs]) if world > 1 else 0
        for r, (J, rb, re, dev) in enumerate(shards):
            rk = FusedDenseRank(None, n, rb, re, dev, params, len(seeds), pair_count, world, r, graph=graphs[r], stream_bits=bits, **kw)
            rk.own_graph = False
            ranks.append(rk)
        blobs = [rk.export() for rk in ranks]
        for rk in ranks:
            rk.connect(blobs)
        for rk in ranks:
            rk.prepare(seeds, phi0)
        for rk in ranks:
            rk.launch()
        return assemble([rk.finish() for rk in ranks])
    finally:
        for rk in ranks:
            rk.close()
        for h in graphs:
            nat.lib().oscb_graph_destroy(h)


def run_dense_fused(J_rows: Optional[np.ndarray], n: int, row_begin: int, row_end: int, params: SolverParams,
                    seeds: Sequence[int], *, device: int, pair_count: int, phi0: Optional[np.ndarray] = None, group=None,
                    graph=None, **kw) -> BatchResult:
    """This process's rank of a fused run over the ranks of `group` (torch.distributed; one process
    per GPU).  Every rank returns the assembled result of the whole graph.  `graph` reuses an
    already uploaded shard handle (`oscb_graph_create_dense` with the same rows; J_rows may then be
    None) and leaves it alive."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        rank, world = 0, 1
    else:
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    if phi0 is None:
        phi0 = _initial_phases_host(device, seeds, n)          # the reference's Philox stream, identical on every rank
    phi0 = np.asarray(phi0, dtype=np.float64).reshape(len(seeds), n)
    keep_graph = graph is not None
    out: List[BatchResult] = []
    try:
        if graph is None:
            h = C.c_void_p()
            rc = nat.lib().oscb_graph_create_dense(device, n, nat.ptr(np.ascontiguousarray(J_rows, dtype=np.float64)), row_begin,
                                                   row_end, C.byref(h))
            if rc != nat.OK:
                _raise(rc, "oscb_graph_create_dense")
            graph = h
        for r0 in range(0, len(seeds), MAX_REPLICAS):
            chunk = list(seeds[r0:r0 + MAX_REPLICAS])
            bits = 0
            if world > 1:
                # one stream for all ranks: e2m1 only if EVERY shard's couplings allow it (the OSCB_UMMA_FP4 environment of
                # a single process must not split the ranks either)
                mine_bits = shard_stream_bits(graph, params.n_states, len(seeds))
                all_bits: List[Optional[int]] = [None] * world
                dist.all_gather_object(all_bits, mine_bits, group=group)
                bits = agree_stream(all_bits)
            rk = FusedDenseRank(None, n, row_begin, row_end, device, params, len(chunk), pair_count, world, rank,
                                graph=graph, stream_bits=bits, **kw)
            rk.own_graph = False
            graph = rk.graph
            try:
                blobs: List[Optional[bytes]] = [None] * world
                if world > 1:
                    dist.all_gather_object(blobs, rk.export(), group=group)
                else:
                    blobs = [rk.export()]
                rk.connect(blobs)
                rk.prepare(chunk, phi0[r0:r0 + len(chunk)])
                if world > 1:
                    dist.barrier(group=group)                  # every block is clean before any rank pushes into it
                rk.launch()
                mine = rk.finish()
                parts: List[Optional[BatchResult]] = [None] * world
                if world > 1:
                    dist.all_gather_object(parts, mine, group=group)
                else:
                    parts = [mine]
                out.append(assemble(parts))
                if world > 1:
                    dist.barrier(group=group)                  # nobody unmaps a block a peer may still read
            finally:
                rk.close()
    finally:
        if graph and not keep_graph:
            nat.lib().oscb_graph_destroy(graph)
    if len(out) == 1:
        return out[0]
    cat = lambda f: np.concatenate([f(b) for b in out], axis=0)
    b0 = out[0]
    return BatchResult(cat(lambda b: b.final_phases), cat(lambda b: b.best_states), cat(lambda b: b.best_objective),
                       b0.trace_t, b0.trace_ks, cat(lambda b: b.energy), cat(lambda b: b.best_trace),
                       cat(lambda b: b.first_hit_step), b0.steps, sum(b.device_ms for b in out),
                       sum(b.kernel_launches for b in out), "dense-tc", b0.replicas_per_cta, b0.smem_bytes,
                       sum(b.wall_time for b in out))
