"""ctypes binding of liboscb.so (include/oscb.h) -- the only way Python reaches the GPU here.

There is deliberately no fallback: if the shared library is missing, or no CUDA device is
usable, every solver entry point raises.  The library is built in-tree by
`__graft_entry__.build()` (nvcc, sm_100a) as `paper_2505_22631_b200/liboscb.so`.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from pathlib import Path
from typing import Optional

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "liboscb.so"
CSRC = PKG_DIR / "csrc"

OK, EINVAL, ECUDA, ENONFINITE, ENOMEM = 0, 1, 2, 3, 4
OBJ = {"maxcut": 0, "coloring": 1}
PREC = {"f32": 32, "f64": 64}
NOISE_DEVICE, NOISE_HOST, NOISE_NONE = 0, 1, 2
FUSED_MEM_BYTES = 96
KERNEL = {"auto": 0, "stream": 1, "resident": 2, "resident-generic": 2, "dense-tc": 3, "cluster": 4, "lowdeg": 5}
KERNEL_NAME = {0: "auto", 1: "stream", 2: "resident", 3: "dense-tc", 4: "cluster", 5: "lowdeg"}

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-shared", "-Xcompiler", "-fPIC"]


class GraphInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("pairs", C.c_int64), ("device", C.c_int32),
                ("is_dense", C.c_int32), ("unit_weights", C.c_int32), ("int_weights", C.c_int32),
                ("row_begin", C.c_int64), ("row_end", C.c_int64), ("max_degree", C.c_int64)]


class RunParams(C.Structure):
    _fields_ = [("K", C.c_double), ("ks_max", C.c_double), ("ks_period", C.c_double), ("kn", C.c_double),
                ("h", C.c_double), ("t_stop", C.c_double),
                ("n_states", C.c_int32), ("objective", C.c_int32), ("precision", C.c_int32),
                ("noise_mode", C.c_int32), ("kernel", C.c_int32), ("use_target", C.c_int32),
                ("steps", C.c_int64), ("cadence", C.c_int64), ("trace_stride", C.c_double),
                ("target_objective", C.c_double), ("first_step", C.c_int64),
                ("replicas_per_cta", C.c_int32), ("variant", C.c_int32)]


class RunOutputs(C.Structure):
    _fields_ = [("final_phases", C.c_void_p), ("best_states", C.c_void_p), ("best_objective", C.c_void_p),
                ("trace_t", C.c_void_p), ("trace_ks", C.c_void_p), ("energy", C.c_void_p),
                ("best_trace", C.c_void_p), ("first_hit_step", C.c_void_p), ("max_samples", C.c_int64),
                ("n_samples", C.c_int64), ("steps_executed", C.c_int64), ("nonfinite", C.c_int64 * 3),
                ("device_ms", C.c_double), ("kernel_launches", C.c_int64), ("kernel_used", C.c_int32),
                ("replicas_per_cta", C.c_int32), ("smem_bytes", C.c_int64)]


class ShardStepParams(C.Structure):
    _fields_ = [("K", C.c_double), ("ks", C.c_double), ("h", C.c_double), ("kn_sqrt_h", C.c_double),
                ("n_states", C.c_int32), ("precision", C.c_int32), ("noise_on", C.c_int32), ("reserved", C.c_int32),
                ("step", C.c_int64)]


# every symbol include/oscb.h declares: name -> (restype, argtypes)
_P = C.c_void_p
SYMBOLS = {
    "oscb_last_error": (C.c_char_p, []),
    "oscb_version": (C.c_int, []),
    "oscb_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "oscb_pool_trim": (C.c_int, []),
    "oscb_csr_from_edges": (C.c_int, [C.c_int, C.c_int64, C.c_int64, _P, _P, _P, _P, _P, _P, C.POINTER(C.c_int64),
                                      C.POINTER(C.c_double)]),
    "oscb_graph_create_csr": (C.c_int, [C.c_int, C.c_int64, _P, _P, _P, C.POINTER(_P)]),
    "oscb_graph_create_dense": (C.c_int, [C.c_int, C.c_int64, _P, C.c_int64, C.c_int64, C.POINTER(_P)]),
    "oscb_graph_destroy": (C.c_int, [_P]),
    "oscb_graph_get_info": (C.c_int, [_P, C.POINTER(GraphInfo)]),
    "oscb_initial_phases": (C.c_int, [_P, _P, C.c_int64, _P]),
    "oscb_device_normals": (C.c_int, [C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_int32, _P]),
    "oscb_step": (C.c_int, [_P, C.c_int64, _P, _P, C.c_double, C.c_double, C.c_double, C.c_double,
                            C.c_int32, C.c_int32, _P, _P]),
    "oscb_score": (C.c_int, [_P, C.c_int64, _P, C.c_int32, C.c_int32, _P, _P]),
    "oscb_energy": (C.c_int, [_P, C.c_int64, _P, _P]),
    "oscb_dense_shard_step": (C.c_int, [_P, C.c_int64, C.POINTER(ShardStepParams), _P, _P, _P, _P]),
    "oscb_dense_shard_objective": (C.c_int, [_P, C.c_int64, C.c_int32, _P, C.c_int32, C.c_int32, _P, _P]),
    "oscb_dense_shard_energy": (C.c_int, [_P, C.c_int64, C.c_int32, _P, _P, _P]),
    "oscb_graph_nonfinite": (C.c_int, [_P, _P, C.c_int32]),
    "oscb_dense_fused_create": (C.c_int, [_P, C.POINTER(RunParams), C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.POINTER(_P)]),
    "oscb_dense_fused_export": (C.c_int, [_P, _P]),
    "oscb_dense_fused_connect": (C.c_int, [_P, _P]),
    "oscb_dense_fused_prepare": (C.c_int, [_P, _P, _P]),
    "oscb_dense_fused_launch": (C.c_int, [_P]),
    "oscb_dense_fused_finish": (C.c_int, [_P, C.POINTER(RunOutputs)]),
    "oscb_dense_fused_rows": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "oscb_dense_fused_grid": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "oscb_dense_fused_destroy": (C.c_int, [_P]),
    "oscb_dense_tc_stream": (C.c_int, [_P, C.c_int32, C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "oscb_selftest_sign_state": (C.c_int, [C.c_int, C.POINTER(C.c_uint64)]),
    "oscb_resident_plan_host": (C.c_int, [C.c_int64, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                          C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                          C.POINTER(C.c_int64), _P, _P, _P, _P]),
    "oscb_lowdeg_plan_host": (C.c_int, [C.c_int64, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int64), C.POINTER(C.c_int64), _P, _P, _P, _P, _P]),
    "oscb_lowdeg_pair_plan_host": (C.c_int, [C.c_int64, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                             C.POINTER(C.c_int64), C.POINTER(C.c_int64), _P, _P, _P, _P, _P]),
    "oscb_run": (C.c_int, [_P, C.POINTER(RunParams), _P, C.c_int64, _P, _P, C.POINTER(RunOutputs)]),
}

_lib: Optional[C.CDLL] = None
_lock = threading.Lock()


def sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.hpp")) + [
        PKG_DIR.parent / "include" / "oscb.h"]


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile liboscb.so for sm_100a with nvcc (cross-compiles without a GPU)."""
    newest = max(p.stat().st_mtime for p in sources())
    if not force and LIB_PATH.exists() and LIB_PATH.stat().st_mtime >= newest:
        return LIB_PATH
    # one object per translation unit (compiled in parallel, rebuilt only when stale), then one link
    from concurrent.futures import ThreadPoolExecutor
    objdir = PKG_DIR / "build"
    objdir.mkdir(exist_ok=True)
    units = sorted(CSRC.glob("*.cu"))

    def deps(src, seen=None):
        """`src` plus the local headers it includes, transitively."""
        import re
        seen = set() if seen is None else seen
        if src in seen or not src.exists():
            return seen
        seen.add(src)
        for inc in re.findall(r'#include\s+"([^"]+)"', src.read_text()):
            deps((src.parent / inc).resolve(), seen)
        return seen

    def compile_unit(src):
        obj = objdir / (src.stem + ".o")
        stamp = max(p.stat().st_mtime for p in deps(src))
        if not force and obj.exists() and obj.stat().st_mtime >= stamp:
            return obj, ""
        cmd = ["nvcc", *[f for f in NVCC_FLAGS if f != "-shared"], "-c", "-o", str(obj), str(src)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stdout}\n{res.stderr}")
        return obj, res.stderr

    with ThreadPoolExecutor(max_workers=len(units)) as ex:
        results = list(ex.map(compile_unit, units))
    if verbose:
        for _, log in results:
            print(log)
    cmd = ["nvcc", *NVCC_FLAGS, "-o", str(LIB_PATH), *[str(o) for o, _ in results]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stdout}\n{res.stderr}")
    return LIB_PATH


def lib() -> C.CDLL:
    """The loaded library.  Raises if it has not been built -- there is no CPU path."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                    " (nvcc, sm_100a).  This package has no CPU fallback.")
            L = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SYMBOLS.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def last_error() -> str:
    msg = lib().oscb_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def device_count() -> int:
    c = C.c_int(0)
    rc = lib().oscb_device_count(C.byref(c))
    return int(c.value) if rc == OK else 0


def ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)
