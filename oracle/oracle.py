"""ctypes front-end for oracle/liboscim_oracle.so -- TEST INFRASTRUCTURE ONLY.

The oracle is the CPU restatement of the reference algorithm (see the header of
oscim_oracle.c for the file:line map).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module; the product package never does.

Array conventions follow the reference kernels (pkg/src/oscim/dynamics.py:155-223):
int64 CSR, float64 phases [R, n] row-major.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboscim_oracle.so"
_lib = None

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> Path:
    """Compile the oracle with the committed Makefile (gcc + numpy's libnpyrandom.a)."""
    src = _HERE / "oscim_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(_HERE), "-B"], check=True, capture_output=True)
    return _LIB_PATH


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = C.CDLL(str(_LIB_PATH))
        L.osc_philox4x64_10.argtypes = [_u64p, _u64p, _u64p]
        L.osc_philox4x64_10.restype = None
        L.osc_initial_phases.argtypes = [C.c_uint64, C.c_int64, _f64p]
        L.osc_initial_phases.restype = None
        L.osc_normal_chunk.argtypes = [C.c_uint64, C.c_int64, C.c_int64, _f64p]
        L.osc_normal_chunk.restype = None
        L.osc_ks_value.argtypes = [C.c_double, C.c_double, C.c_double]
        L.osc_ks_value.restype = C.c_double
        L.osc_step.argtypes = [_i64p, _i64p, _f64p, C.c_int64, C.c_int64, _f64p, C.c_void_p,
                               C.c_double, C.c_double, C.c_double, C.c_double, C.c_int64,
                               _f64p, _f64p, C.c_int]
        L.osc_step.restype = None
        L.osc_score.argtypes = [_f64p, C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p, _f64p,
                                C.c_int64, C.c_int, _i64p, _f64p, C.c_int]
        L.osc_score.restype = None
        L.osc_continuous_energy.argtypes = [_f64p, _i64p, _i64p, _f64p, C.c_int64]
        L.osc_continuous_energy.restype = C.c_double
        L.osc_objective_cadence.argtypes = [C.c_int64, C.c_int64]
        L.osc_objective_cadence.restype = C.c_int64
        L.osc_simulate.argtypes = [
            _i64p, _i64p, _f64p, C.c_int64, _i64p, _i64p, _f64p, C.c_int64,
            C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
            C.c_int64, _u64p, C.c_int64, C.c_int, C.c_double, C.c_void_p, C.c_int,
            _f64p, _i64p, _f64p, _f64p, _f64p, _f64p, _f64p,
            C.c_int64, _i64p, _i64p, _i64p,
        ]
        L.osc_simulate.restype = C.c_int
        L.osc_max_threads.argtypes = []
        L.osc_max_threads.restype = C.c_int
        _lib = L
    return _lib


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def pairs_from_csr(indptr, indices, data):
    """Canonical upper-triangle pairs (model.py:238-242)."""
    indptr = np.asarray(indptr, dtype=np.int64)
    n = len(indptr) - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
    idx = np.asarray(indices, dtype=np.int64)
    up = rows < idx
    return _c(rows[up], np.int64), _c(idx[up], np.int64), _c(np.asarray(data)[up], np.float64)


def philox4x64_10(counter: int, seed: int) -> np.ndarray:
    ctr = np.array([(counter >> (64 * k)) & (2**64 - 1) for k in range(4)], dtype=np.uint64)
    key = np.array([seed, 0], dtype=np.uint64)
    out = np.zeros(4, dtype=np.uint64)
    lib().osc_philox4x64_10(ctr, key, out)
    return out


def initial_phases(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib().osc_initial_phases(seed, n, out)
    return out


def normal_chunk(seed: int, chunk_index: int, n: int) -> np.ndarray:
    out = np.empty((256, n), dtype=np.float64)
    lib().osc_normal_chunk(seed, chunk_index, n, out)
    return out


def step_normals(seed: int, step: int, n: int) -> np.ndarray:
    return normal_chunk(seed, step // 256, n)[step % 256]


def ks_value(ks_max: float, period: float, t: float) -> float:
    return float(lib().osc_ks_value(ks_max, period, t))


def objective_cadence(n: int, pair_count: int) -> int:
    return int(lib().osc_objective_cadence(n, pair_count))


def step(indptr, indices, data, phi, noise, K, ks, h, kn_sqrt_h, n_states, threads=1):
    phi = _c(np.atleast_2d(phi), np.float64)
    R, n = phi.shape
    out = np.empty_like(phi)
    scratch = np.empty(3 * R * n, dtype=np.float64)
    if noise is not None:
        noise = _c(np.atleast_2d(noise), np.float64)
        nptr = noise.ctypes.data_as(C.c_void_p)
    else:
        nptr = None
    lib().osc_step(_c(indptr, np.int64), _c(indices, np.int64), _c(data, np.float64), R, n, phi,
                   nptr, K, ks, h, kn_sqrt_h, n_states, out, scratch, threads)
    return out


def score(phi, n_states, iu, jv, w, maximize, threads=1):
    phi = _c(np.atleast_2d(phi), np.float64)
    R, n = phi.shape
    states = np.zeros((R, n), dtype=np.int64)
    obj = np.zeros(R, dtype=np.float64)
    iu, jv, w = _c(iu, np.int64), _c(jv, np.int64), _c(w, np.float64)
    lib().osc_score(phi, R, n, n_states, iu, jv, w, len(iu), int(bool(maximize)), states, obj, threads)
    return states, obj


def continuous_energy(phi_row, iu, jv, w) -> float:
    iu, jv, w = _c(iu, np.int64), _c(jv, np.int64), _c(w, np.float64)
    return float(lib().osc_continuous_energy(_c(phi_row, np.float64), iu, jv, w, len(iu)))


@dataclass
class OracleRun:
    final_phases: np.ndarray        # [R, n]
    best_states: np.ndarray         # [R, n] int64
    best_objective: np.ndarray      # [R]
    trace_t: np.ndarray             # [S]
    trace_ks: np.ndarray            # [S]
    energy: np.ndarray              # [R, S]
    best_trace: np.ndarray          # [R, S]
    steps: int


class OracleNumericalError(ArithmeticError):
    def __init__(self, replica, oscillator, step):
        self.replica, self.oscillator, self.step = replica, oscillator, step
        super().__init__(f"non-finite phase for oscillator {oscillator} (replica row {replica}) after step {step}")


def simulate(indptr, indices, data, *, K, ks_max, ks_period, kn, h, t_stop, n_states,
             seeds: Sequence[int], objective: str = "maxcut", trace_stride: Optional[float] = None,
             phi0=None, threads: int = 1) -> OracleRun:
    """The whole of dynamics.py:_simulate for the replica group `seeds`."""
    indptr, indices, data = _c(indptr, np.int64), _c(indices, np.int64), _c(data, np.float64)
    n = len(indptr) - 1
    iu, jv, w = pairs_from_csr(indptr, indices, data)
    R = len(seeds)
    steps = int(math.ceil(t_stop / h))
    stride = ks_period / 2.0 if trace_stride is None else float(trace_stride)
    if stride <= 0:
        raise ValueError("trace_stride must be > 0")
    max_samples = int(min(steps + 2, steps * h / stride + 8))
    seeds_a = np.array([int(s) % 2**64 for s in seeds], dtype=np.uint64)
    final = np.empty((R, n)); states = np.zeros((R, n), dtype=np.int64); best = np.zeros(R)
    tt = np.zeros(max_samples); tks = np.zeros(max_samples)
    en = np.zeros((R, max_samples)); bt = np.zeros((R, max_samples))
    ns = np.zeros(1, dtype=np.int64); st = np.zeros(1, dtype=np.int64); nf = np.zeros(3, dtype=np.int64)
    if phi0 is not None:
        phi0 = _c(phi0, np.float64).reshape(R, n)
        p0 = phi0.ctypes.data_as(C.c_void_p)
    else:
        p0 = None
    rc = lib().osc_simulate(indptr, indices, data, n, iu, jv, w, len(iu),
                            K, ks_max, ks_period, kn, h, t_stop, n_states, seeds_a, R,
                            int(objective == "maxcut"), stride, p0, threads,
                            final, states, best, tt, tks, en, bt, max_samples, ns, st, nf)
    if rc == 3:
        raise OracleNumericalError(int(nf[0]), int(nf[1]), int(nf[2]))
    if rc != 0:
        raise RuntimeError(f"osc_simulate failed rc={rc}")
    S = int(ns[0])
    return OracleRun(final, states, best, tt[:S].copy(), tks[:S].copy(), en[:, :S].copy(),
                     bt[:, :S].copy(), int(st[0]))


def max_threads() -> int:
    env = os.environ.get("OMP_NUM_THREADS")
    if env:
        try:
            return max(1, int(env))
        except ValueError:
            pass
    return max(1, min(int(lib().osc_max_threads()), os.cpu_count() or 1))
