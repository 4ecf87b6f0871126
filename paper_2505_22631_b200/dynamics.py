"""Noisy Forward-Euler integration of the OIM/OPM phase dynamics -- on the GPU.

    dphi_i/dt = K * sum_j J_ij sin(2 pi (phi_i - phi_j)) - Ks(t) * sin(2 pi N phi_i) + noise

This module keeps the reference solver's public API name for name
(/root/reference/pkg/src/oscim/dynamics.py: KsSchedule :69-92, NoiseSource :95-129,
RunResult :132-144, phase_drift :254-273, euler_step :286-314, run :443-460,
run_replica_set :469-493, run_replicas :496-515, replica_seed :243-247, resolve_workers
:226-240) so it is a drop-in for that path, but none of the arithmetic happens here: every
function hands numpy buffers to liboscb.so (include/oscb.h) through ctypes and the CUDA
kernels do the work.  There is no CPU fallback.

What differs from the reference, by design:
  * all replicas of a call advance together in one device loop (the reference runs groups
    of <= ~32 MB of noise one after another, dynamics.py:463-466, :486-492);
  * the Gaussian noise is the device's counter-based Philox4x32-10 + Box-Muller stream,
    a pure function of (seed, step, oscillator) as the reference documents for its own
    stream (dynamics.py:97-105); the reference's numpy Ziggurat stream cannot be replayed
    in parallel, so noisy runs agree in distribution, not draw for draw.  Initial phases
    ARE the reference's bit for bit (numpy Philox4x64-10, replayed on the device);
  * `precision="f64"` keeps the reference's float64 arithmetic and operation order
    (parity mode); `precision="f32"` is the throughput mode (the paper's precision);
  * `workers` / `batch_size` are accepted and validated like the reference's but do not
    change anything (they never changed results there either, test_dynamics.py:320-333).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import time
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as nat
from .model import CouplingMatrix, PhaseState, SolverParams, StateAssignment

TWO_PI = 2.0 * np.pi
NOISE_CHUNK = 256  # kept for API compatibility; the device stream is not chunked
WORKER_ENV_VAR = "OSCIM_MAX_WORKERS"
PRECISION_ENV_VAR = "OSCB_PRECISION"
DEVICE_ENV_VAR = "OSCB_DEVICE"

__all__ = [
    "KsSchedule", "NoiseSource", "RunResult", "NumericalError", "ks_at", "phase_drift",
    "euler_step", "run", "run_replicas", "run_replica_set", "replica_seed", "resolve_workers",
    "score_phases", "sample_energy", "run_batch", "BatchResult", "default_precision",
]


class NumericalError(ArithmeticError):
    """A phase became non-finite during integration (dynamics.py:65-66)."""


def default_precision() -> str:
    p = os.environ.get(PRECISION_ENV_VAR, "f32")
    if p not in nat.PREC:
        raise ValueError(f"{PRECISION_ENV_VAR} must be one of {sorted(nat.PREC)}, got {p!r}")
    return p


def _default_device() -> int:
    env = os.environ.get(DEVICE_ENV_VAR)
    if env is not None:
        return int(env)
    return int(os.environ.get("LOCAL_RANK", "0")) if "LOCAL_RANK" in os.environ else 0


def _precision(p: Optional[str]) -> str:
    p = default_precision() if p is None else p
    if p not in nat.PREC:
        raise ValueError(f"precision must be one of {sorted(nat.PREC)}, got {p!r}")
    return p


def _raise(rc: int, what: str):
    msg = nat.last_error()
    if rc == nat.EINVAL:
        raise ValueError(msg)
    if rc == nat.ENONFINITE:
        raise NumericalError(msg)
    if rc == nat.ENOMEM:
        raise MemoryError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")


# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class KsSchedule:
    """Triangular annealing waveform (dynamics.py:69-88): 0 at cycle start, ks_max at
    mid-cycle, back to 0 at the period.  The device evaluates the same expression in float64
    from the step index."""

    ks_max: float
    period: float

    def __post_init__(self) -> None:
        if not (self.ks_max >= 0 and np.isfinite(self.ks_max)):
            raise ValueError("ks_max must be finite and >= 0")
        if not (self.period > 0 and np.isfinite(self.period)):
            raise ValueError("period must be finite and > 0")

    def value(self, t: float) -> float:
        tm = t % self.period
        half = 0.5 * self.period
        if tm <= half:
            return self.ks_max * (tm / half)
        return self.ks_max * (2.0 - tm / half)


def ks_at(schedule: KsSchedule, t: float) -> float:
    return schedule.value(t)


@dataclass(frozen=True)
class NoiseSource:
    """Counter-indexed noise keyed by a 64-bit seed (dynamics.py:95-129).

    `initial_phases` replays the reference's numpy stream exactly (Philox4x64-10, counter
    1 << 192) on the device.  `step_normals` returns the DEVICE stream the integrator uses:
    Philox4x32-10 at counter (oscillator // 4, step) keyed by the seed, Box-Muller; a pure
    function of (seed, oscillator, step), independent of n, order and batch."""

    seed: int
    precision: Optional[str] = None
    device: Optional[int] = None

    def __post_init__(self) -> None:
        if not (0 <= self.seed < 2**64):
            raise ValueError("seed must fit in 64 bits")

    def _dev(self) -> int:
        return _default_device() if self.device is None else self.device

    def step_normals(self, step: int, n: int) -> np.ndarray:
        if step < 0:
            raise ValueError("step must be >= 0")
        out = np.empty(n, dtype=np.float64)
        rc = nat.lib().oscb_device_normals(self._dev(), self.seed, step, n, nat.PREC[_precision(self.precision)],
                                           nat.ptr(out))
        if rc != nat.OK:
            _raise(rc, "oscb_device_normals")
        return out

    def normal_chunk(self, chunk_index: int, n: int) -> np.ndarray:
        """Draws for NOISE_CHUNK consecutive steps, shape (NOISE_CHUNK, n)."""
        start = chunk_index * NOISE_CHUNK
        return np.stack([self.step_normals(start + s, n) for s in range(NOISE_CHUNK)])

    def initial_phases(self, n: int) -> np.ndarray:
        """Uniform [0, 1) starting phases, identical to the reference's."""
        return _initial_phases_host(self._dev(), [self.seed], n)[0]


def _initial_phases_host(device: int, seeds: Sequence[int], n: int) -> np.ndarray:
    """Philox4x64-10 initial phases need no graph; a one-node handle carries the call."""
    h = _scratch_graph(device, n)
    seeds_a = np.array([int(s) % 2**64 for s in seeds], dtype=np.uint64)
    out = np.empty((len(seeds_a), n), dtype=np.float64)
    rc = nat.lib().oscb_initial_phases(h.handle, nat.ptr(seeds_a), len(seeds_a), nat.ptr(out))
    if rc != nat.OK:
        _raise(rc, "oscb_initial_phases")
    return out


@dataclass
class RunResult:
    """Outcome of one solver run (or the best replica of a batch) (dynamics.py:132-144)."""

    best_assignment: StateAssignment
    best_objective: float
    final_phases: PhaseState
    energy_trace: List[Tuple[float, float, float]]  # (t, continuous energy, Ks)
    best_trace: List[float]
    wall_time: float
    steps_executed: int
    objective_kind: str
    replica_index: int = 0
    # not in the reference's RunResult: the arithmetic this result was computed in -- "f32" (throughput mode, the
    # DEFAULT of this package) or "f64" (the reference's own arithmetic) -- and the kernel that ran
    precision: str = "f32"
    kernel: str = ""


# ---------------------------------------------------------------------------
# device graphs
class DeviceGraph:
    """Owns one `oscb_graph` handle (device CSR or dense J) for a CouplingMatrix."""

    def __init__(self, handle, device: int):
        self.handle = handle
        self.device = device

    @classmethod
    def from_csr(cls, device: int, n: int, indptr, indices, data) -> "DeviceGraph":
        indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        indices = np.ascontiguousarray(indices, dtype=np.int64)
        data = np.ascontiguousarray(data, dtype=np.float64)
        h = C.c_void_p()
        rc = nat.lib().oscb_graph_create_csr(device, n, nat.ptr(indptr), nat.ptr(indices), nat.ptr(data), C.byref(h))
        if rc != nat.OK:
            _raise(rc, "oscb_graph_create_csr")
        return cls(h, device)

    @classmethod
    def from_dense(cls, device: int, J: np.ndarray, row_begin: int = 0, row_end: Optional[int] = None) -> "DeviceGraph":
        J = np.ascontiguousarray(J, dtype=np.float64)
        n = J.shape[1]
        row_end = n if row_end is None else row_end
        h = C.c_void_p()
        rc = nat.lib().oscb_graph_create_dense(device, n, nat.ptr(J), row_begin, row_end, C.byref(h))
        if rc != nat.OK:
            _raise(rc, "oscb_graph_create_dense")
        return cls(h, device)

    def info(self) -> nat.GraphInfo:
        gi = nat.GraphInfo()
        rc = nat.lib().oscb_graph_get_info(self.handle, C.byref(gi))
        if rc != nat.OK:
            _raise(rc, "oscb_graph_get_info")
        return gi

    def tc_stream(self, n_states: int, replicas: int) -> Tuple[int, int]:
        """(bits per coupling, replicas per launch) of a tensor-core dense run of `replicas` replicas."""
        bits, per = C.c_int32(0), C.c_int32(0)
        rc = nat.lib().oscb_dense_tc_stream(self.handle, n_states, replicas, C.byref(bits), C.byref(per))
        if rc != nat.OK:
            _raise(rc, "oscb_dense_tc_stream")
        return bits.value, per.value

    def close(self) -> None:
        if self.handle:
            nat.lib().oscb_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_scratch = {}


def _scratch_graph(device: int, n: int) -> DeviceGraph:
    key = (device, n)
    if key not in _scratch:
        _scratch.clear()
        _scratch[key] = DeviceGraph.from_csr(device, n, np.zeros(n + 1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    return _scratch[key]


# Couplings stored dense (model.py:21, :190-192) get the dense device path (J in HBM, O(n^2)
# kernels) only from this size on; below it the device CSR + the persistent shared-memory kernel
# is the faster home even for a complete graph (rows of up to 1020 neighbours fit its stream).
DENSE_DEVICE_MIN_N = 1021


def device_graph(J: CouplingMatrix, device: Optional[int] = None) -> DeviceGraph:
    """The (cached) device mirror of J on `device`: dense J for large couplings stored dense,
    device CSR otherwise (north_star subsystem 1)."""
    device = _default_device() if device is None else device
    cache = J._device
    if cache is None:
        cache = {}
        J._device = cache
    if device not in cache:
        if J.storage_kind == "dense" and J._dense is not None and J.n >= DENSE_DEVICE_MIN_N:
            cache[device] = DeviceGraph.from_dense(device, J._dense)
        else:
            cache[device] = DeviceGraph.from_csr(device, J.n, J.indptr, J.indices, J.data)
    return cache[device]


# ---------------------------------------------------------------------------
def resolve_workers(requested: Optional[int]) -> int:
    """Same validation as the reference (dynamics.py:226-240).  The value has no effect on
    the GPU path (it never affected results in the reference either)."""
    cap = os.cpu_count() or 1
    env = os.environ.get(WORKER_ENV_VAR)
    if env is not None:
        try:
            cap = min(cap, max(1, int(env)))
        except ValueError:
            raise ValueError(f"{WORKER_ENV_VAR} must be an integer, got {env!r}") from None
    if requested is None:
        return 1
    if requested < 1:
        raise ValueError("workers must be >= 1")
    return min(requested, cap)


def replica_seed(seed: int, index: int) -> int:
    """(seed + index) mod 2^64 (dynamics.py:243-247)."""
    return (seed + index) % 2**64


def phase_drift(J: CouplingMatrix, phi: PhaseState, i: int, K: float, ks_t: float, n_states: int,
                device: Optional[int] = None) -> float:
    """Deterministic part of dphi_i/dt (dynamics.py:254-273), evaluated by the float64 parity
    kernel: one noise-free step of size h = 1 from `phi` moves oscillator i by exactly the
    drift (before the wrap), so drift = unwrap(step(phi)[i] - phi[i])."""
    if not 0 <= i < J.n:
        raise IndexError(f"oscillator index {i} out of range for n={J.n}")
    if J.n != phi.n:
        raise ValueError(f"dimension mismatch: coupling n={J.n} vs phases n={phi.n}")
    # a small h keeps the move inside (-0.5, 0.5) so the wrap can be undone exactly
    lo, hi = int(J.indptr[i]), int(J.indptr[i + 1])
    bound = abs(K) * float(np.abs(J.data[lo:hi]).sum()) + abs(ks_t)      # |drift| <= bound, also for K < 0
    if not math.isfinite(bound):
        raise ValueError("K, ks_t and the couplings must be finite")
    h = 2.0 ** -math.ceil(math.log2(max(bound, 1.0)) + 2)
    out = _step_raw(J, phi.phases[None, :], None, K, ks_t, h, 0.0, n_states, "f64", device)[0]
    d = out[i] - phi.phases[i]
    d -= round(d)
    return d / h


def _step_raw(J: CouplingMatrix, phi2d: np.ndarray, noise2d: Optional[np.ndarray], K: float, ks: float, h: float,
              kn_sqrt_h: float, n_states: int, precision: str, device: Optional[int]) -> np.ndarray:
    g = device_graph(J, device)
    phi2d = np.ascontiguousarray(phi2d, dtype=np.float64)
    R, n = phi2d.shape
    if noise2d is not None:
        noise2d = np.ascontiguousarray(noise2d, dtype=np.float64).reshape(R, n)
    out = np.empty_like(phi2d)
    nf = np.full(2, -1, dtype=np.int64)
    rc = nat.lib().oscb_step(g.handle, R, nat.ptr(phi2d), nat.ptr(noise2d), K, ks, h, kn_sqrt_h, n_states,
                             nat.PREC[precision], nat.ptr(out), nat.ptr(nf))
    if rc != nat.OK:
        _raise(rc, "oscb_step")
    return out


def euler_step(phi: PhaseState, J: CouplingMatrix, params: SolverParams, t: float, noise: NoiseSource,
               step_index: int, precision: Optional[str] = None, device: Optional[int] = None) -> PhaseState:
    """One synchronous Forward-Euler update of all phases (dynamics.py:286-314)."""
    if J.n != phi.n:
        raise ValueError(f"dimension mismatch: coupling n={J.n} vs phases n={phi.n}")
    prec = _precision(precision)
    schedule = KsSchedule(params.ks_max, params.ks_period)
    src = NoiseSource(noise.seed, prec, device if device is not None else noise.device)
    kick = src.step_normals(step_index, phi.n)[None, :] if params.kn != 0.0 else None
    g = device_graph(J, device)
    p = np.ascontiguousarray(phi.phases[None, :], dtype=np.float64)
    out = np.empty_like(p)
    nf = np.full(2, -1, dtype=np.int64)
    rc = nat.lib().oscb_step(g.handle, 1, nat.ptr(p), nat.ptr(None if kick is None else np.ascontiguousarray(kick)),
                             params.K, schedule.value(t), params.h, params.kn * math.sqrt(params.h),
                             params.n_states, nat.PREC[prec], nat.ptr(out), nat.ptr(nf))
    if rc == nat.ENONFINITE:
        raise NumericalError(f"non-finite phase for oscillator {int(nf[1])} (replica row {int(nf[0])}) "
                             f"after step {step_index}; parameters are numerically unstable")
    if rc != nat.OK:
        _raise(rc, "oscb_step")
    return PhaseState(out[0])


def score_phases(J: CouplingMatrix, phi2d: np.ndarray, n_states: int, objective: str,
                 device: Optional[int] = None) -> Tuple[np.ndarray, np.ndarray]:
    """Threshold + objective of every row of `phi2d` on the device: the drop-in for
    `_score_kernel` (dynamics.py:193-223).  Returns (states int64 [R, n], objective [R])."""
    g = device_graph(J, device)
    phi2d = np.ascontiguousarray(np.atleast_2d(phi2d), dtype=np.float64)
    R, n = phi2d.shape
    if n != J.n:
        raise ValueError(f"dimension mismatch: coupling n={J.n} vs phases n={n}")
    states = np.empty((R, n), dtype=np.int64)
    obj = np.empty(R, dtype=np.float64)
    rc = nat.lib().oscb_score(g.handle, R, nat.ptr(phi2d), n_states, int(objective == "maxcut"), nat.ptr(states), nat.ptr(obj))
    if rc != nat.OK:
        _raise(rc, "oscb_score")
    return states, obj


def sample_energy(J: CouplingMatrix, phi2d: np.ndarray, device: Optional[int] = None) -> np.ndarray:
    """sum_{i<j} J_ij cos(2 pi (phi_i - phi_j)) per row, on the device (dynamics.py:380)."""
    g = device_graph(J, device)
    phi2d = np.ascontiguousarray(np.atleast_2d(phi2d), dtype=np.float64)
    R, n = phi2d.shape
    if n != J.n:
        raise ValueError(f"dimension mismatch: coupling n={J.n} vs phases n={n}")
    out = np.empty(R, dtype=np.float64)
    rc = nat.lib().oscb_energy(g.handle, R, nat.ptr(phi2d), nat.ptr(out))
    if rc != nat.OK:
        _raise(rc, "oscb_energy")
    return out


# ---------------------------------------------------------------------------
@dataclass
class BatchResult:
    """Raw arrays of one `oscb_run` call (all replicas)."""

    final_phases: np.ndarray      # [R, n] float64
    best_states: np.ndarray       # [R, n] uint8
    best_objective: np.ndarray    # [R] in-loop value of the best sample
    trace_t: np.ndarray           # [S]
    trace_ks: np.ndarray          # [S]
    energy: np.ndarray            # [R, S]
    best_trace: np.ndarray        # [R, S]
    first_hit_step: np.ndarray    # [R] (-1: target never reached / not requested)
    steps: int
    device_ms: float
    kernel_launches: int
    kernel: str
    replicas_per_cta: int
    smem_bytes: int
    wall_time: float
    precision: str = "f32"


def _objective_cadence_for(n: int, pair_count: int) -> int:
    """Steps between best-of objective checks (dynamics.py:325-330)."""
    return max(1, min(10, round(pair_count / max(n, 1))))


def _sample_steps(steps: int, h: float, stride: float) -> List[int]:
    """Steps after which the reference takes a trace sample (dynamics.py:385, :404-408), with the
    same float arithmetic."""
    out, next_sample = [], stride
    for step in range(steps):
        t_next = (step + 1) * h
        if t_next >= next_sample or step == steps - 1:
            while next_sample <= t_next:
                next_sample += stride
            out.append(step)
    return out


def _sample_capacity(steps: int, h: float, stride: float) -> int:
    return int(min(steps + 2, steps * h / stride + 8))


def run_batch(J: CouplingMatrix, params: SolverParams, objective: str, seeds: Sequence[int], *,
              trace_stride: Optional[float] = None, precision: Optional[str] = None,
              device: Optional[int] = None, kernel: str = "auto", steps: Optional[int] = None,
              cadence: Optional[int] = None, phi0: Optional[np.ndarray] = None,
              noise: Optional[np.ndarray] = None, noise_off: bool = False,
              target: Optional[float] = None, first_step: int = 0, replicas_per_cta: int = 0,
              want_phases: bool = True, want_states: bool = True, want_traces: bool = True,
              graph: Optional[DeviceGraph] = None) -> BatchResult:
    """Advance the replicas `seeds` together on one GPU: the drop-in for `_simulate`
    (dynamics.py:333-431).  `noise` ([steps, R, n]) injects host-supplied normals (parity
    hook); `noise_off` integrates with kn treated as 0.  `graph` runs on an already uploaded
    device graph (J may then be None -- e.g. a dense J too large to also hold as CSR)."""
    g = device_graph(J, device) if graph is None else graph
    prec = _precision(precision)
    n, R = (J.n if graph is None else int(graph.info().n)), len(seeds)
    stride = params.ks_period / 2.0 if trace_stride is None else float(trace_stride)
    if stride <= 0:
        raise ValueError("trace_stride must be > 0")
    nsteps = int(math.ceil(params.t_stop / params.h)) if steps is None else int(steps)
    cap = _sample_capacity(nsteps, params.h, stride)
    seeds_a = np.array([int(s) % 2**64 for s in seeds], dtype=np.uint64)

    p = nat.RunParams()
    p.K, p.ks_max, p.ks_period, p.kn = params.K, params.ks_max, params.ks_period, params.kn
    p.h, p.t_stop, p.n_states = params.h, params.t_stop, params.n_states
    p.objective = nat.OBJ.get(objective, -1)
    p.precision = nat.PREC[prec]
    p.noise_mode = nat.NOISE_HOST if noise is not None else (nat.NOISE_NONE if noise_off else nat.NOISE_DEVICE)
    if kernel not in nat.KERNEL:
        raise ValueError(f"kernel must be one of {sorted(nat.KERNEL)}")
    p.kernel = nat.KERNEL[kernel]
    p.variant = 1 if kernel == "resident-generic" else 0
    p.use_target = int(target is not None)
    p.target_objective = 0.0 if target is None else float(target)
    p.steps = nsteps if steps is not None else 0
    p.cadence = 0 if cadence is None else int(cadence)
    p.trace_stride = stride
    p.first_step = int(first_step)
    p.replicas_per_cta = int(replicas_per_cta)

    final = np.empty((R, n), dtype=np.float64) if want_phases else None
    states = np.empty((R, n), dtype=np.uint8) if want_states else None
    best = np.empty(R, dtype=np.float64)
    tt = np.zeros(cap); tks = np.zeros(cap)
    en = np.zeros((R, cap)) if want_traces else None
    bt = np.zeros((R, cap)) if want_traces else None
    first = np.full(R, -1, dtype=np.int64)
    o = nat.RunOutputs()
    o.final_phases, o.best_states, o.best_objective = nat.ptr(final), nat.ptr(states), nat.ptr(best)
    o.trace_t, o.trace_ks, o.energy, o.best_trace = nat.ptr(tt), nat.ptr(tks), nat.ptr(en), nat.ptr(bt)
    o.first_hit_step = nat.ptr(first)
    o.max_samples = cap
    if phi0 is not None:
        phi0 = np.ascontiguousarray(phi0, dtype=np.float64).reshape(R, n)
    if noise is not None:
        noise = np.ascontiguousarray(noise, dtype=np.float64).reshape(nsteps, R, n)
    t0 = time.perf_counter()
    rc = nat.lib().oscb_run(g.handle, C.byref(p), nat.ptr(seeds_a), R, nat.ptr(phi0), nat.ptr(noise), C.byref(o))
    wall = time.perf_counter() - t0
    if rc != nat.OK:
        _raise(rc, "oscb_run")
    S = int(o.n_samples)
    return BatchResult(final, states, best, tt[:S].copy(), tks[:S].copy(),
                       en[:, :S].copy() if en is not None else np.zeros((R, 0)),
                       bt[:, :S].copy() if bt is not None else np.zeros((R, 0)),
                       first, int(o.steps_executed), float(o.device_ms), int(o.kernel_launches),
                       nat.KERNEL_NAME.get(int(o.kernel_used), "?"), int(o.replicas_per_cta), int(o.smem_bytes), wall, prec)


def _objective_from_states(states_row: np.ndarray, iu, jv, w, kind: str) -> float:
    """Objective of one assignment on the canonical pair order (dynamics.py:317-322)."""
    if kind == "maxcut":
        return float((w * (states_row[iu] != states_row[jv])).sum())
    return float((states_row[iu] == states_row[jv]).sum())


def _validate_run_args(J: CouplingMatrix, params: SolverParams, objective: str) -> None:
    if J.n < 1:
        raise ValueError("problem must have at least one oscillator")
    if objective not in ("maxcut", "coloring"):
        raise ValueError(f"unknown objective kind: {objective!r}")
    if objective == "maxcut" and params.n_states != 2:
        raise ValueError("maxcut runs require n_states=2")


def _results_from_batch(J: CouplingMatrix, params: SolverParams, objective: str, b: BatchResult,
                        first_index: int = 0) -> List[RunResult]:
    iu, jv, w = J.pairs()
    out = []
    for r in range(b.final_phases.shape[0]):
        states = b.best_states[r].astype(np.int64)
        trace = [(float(b.trace_t[k]), float(b.energy[r, k]), float(b.trace_ks[k])) for k in range(len(b.trace_t))]
        out.append(RunResult(
            best_assignment=StateAssignment(params.n_states, states),
            best_objective=_objective_from_states(states, iu, jv, w, objective),
            final_phases=PhaseState(b.final_phases[r]),
            energy_trace=trace,
            best_trace=[float(x) for x in b.best_trace[r]],
            wall_time=b.wall_time,
            steps_executed=b.steps,
            objective_kind=objective,
            replica_index=first_index + r,
            precision=b.precision,
            kernel=b.kernel,
        ))
    return out


def run(J: CouplingMatrix, params: SolverParams, objective: str = "maxcut", workers: Optional[int] = None,
        trace_stride: Optional[float] = None, *, precision: Optional[str] = None,
        device: Optional[int] = None, kernel: str = "auto") -> RunResult:
    """Integrate from the seed's initial phases and return the best assignment found at any
    scored step (dynamics.py:443-460)."""
    _validate_run_args(J, params, objective)
    resolve_workers(workers)
    b = run_batch(J, params, objective, [params.seed % 2**64], trace_stride=trace_stride,
                  precision=precision, device=device, kernel=kernel)
    return _results_from_batch(J, params, objective, b)[0]


def run_replica_set(J: CouplingMatrix, params: SolverParams, objective: str = "maxcut", replicas: int = 1,
                    workers: Optional[int] = None, trace_stride: Optional[float] = None, *,
                    precision: Optional[str] = None, device: Optional[int] = None,
                    kernel: str = "auto") -> List[RunResult]:
    """All replica results; replica r uses seed replica_seed(params.seed, r)
    (dynamics.py:469-493).  Every replica advances in the same device loop."""
    _validate_run_args(J, params, objective)
    if replicas < 1:
        raise ValueError("replicas must be >= 1")
    resolve_workers(workers)
    seeds = [replica_seed(params.seed, r) for r in range(replicas)]
    results: List[RunResult] = []
    group = 65536
    for start in range(0, replicas, group):
        b = run_batch(J, params, objective, seeds[start:start + group], trace_stride=trace_stride,
                      precision=precision, device=device, kernel=kernel)
        results.extend(_results_from_batch(J, params, objective, b, start))
    return results


def run_replicas(J: CouplingMatrix, params: SolverParams, objective: str = "maxcut", replicas: int = 1,
                 workers: Optional[int] = None, trace_stride: Optional[float] = None, *,
                 precision: Optional[str] = None, device: Optional[int] = None,
                 kernel: str = "auto") -> RunResult:
    """Best-of-replicas; ties go to the lowest replica index (dynamics.py:496-515)."""
    t0 = time.perf_counter()
    results = run_replica_set(J, params, objective, replicas, workers, trace_stride,
                              precision=precision, device=device, kernel=kernel)
    maximize = objective == "maxcut"
    best = results[0]
    for res in results[1:]:
        if (res.best_objective > best.best_objective) if maximize else (res.best_objective < best.best_objective):
            best = res
    best.wall_time = time.perf_counter() - t0
    return best
