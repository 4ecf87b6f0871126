#!/usr/bin/env python
"""bench.py -- oscillator-edge updates/s of the OIM/OPM Euler integrator on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload NAME]

A "step" is one pass of the hot path over one batch: a complete solve -- the whole default
schedule ceil(t_stop / h) (66 875 Euler steps on the G22 shape; `--window N` takes N consecutive
steps instead) -- of ALL replicas of the workload, including threshold + cut scoring at the
reference cadence, best-state tracking and the trace samples (SURVEY.md 8d "unit of work").  The default
workload is BASELINE.json configs[1]: G22-shape max-cut (n=2000, 19990 edges, synthetic
G(n,m), OIM N=2, GSET tuning K=0.2 ks_max=1.0 kn=0.15), 1024 replicas per GPU.

  value   : updates/s = replicas * nnz * window * K / (device time of the K steps), phases
            resident on the device (Philox initial phases generated there), CUDA events on
            the stream the kernels run on, max over ranks.
  e2e     : the same metric through the public API with HOST buffers: initial phases
            handed in from host memory, final phases / best states / objectives / traces
            copied back, wall clock around the K calls.
  roofline: algorithmic HBM bytes (2*R*n*4 + nnz*(4+0|4) + (n+1)*4 per Euler step)
            / kernel time, against MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline / --impl reference: the CPU oracle port of the reference algorithm
            (oracle/, C + OpenMP, numpy's own Ziggurat) on the box's host cores, bounded sample.

Multi-GPU (torchrun, one process per GPU): independent replicas shard across ranks with no
data-path collective (weak scaling: 1024 replicas per GPU); the only communication is the
barrier and the max-over-ranks of the timing.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (shape, replicas per GPU, tuning overrides)
    "G22x1024": ("G22", 1024, dict(K=0.2, ks_max=1.0, kn=0.15)),
    "G1x1": ("G1", 1, dict(K=0.2, ks_max=1.0, kn=0.15)),
    "flat200x4096": ("flat200", 4096, {}),
    "G81x296": ("G81", 296, {}),
}


def load_workload(name):
    from paper_2505_22631_b200 import workloads
    from paper_2505_22631_b200.model import CouplingMatrix, SolverParams
    shape, R, tune = WORKLOADS[name]
    if shape == "flat200":
        # the reference's own generator call, generate_colorable_graph(200, 479, 3, seed=0)
        # (problems.py:255-276; the package's port returns the reference's edge list bit for bit --
        # tests/test_oracle_golden.py::test_flat200_graph_is_the_reference_generators)
        from paper_2505_22631_b200 import problems
        g = problems.generate_colorable_graph(200, 479, 3, seed=0)
        n, (u, v, w), N, kind = g.node_count, (g.u, g.v, g.w), 3, "coloring"
    else:
        n, (u, v, w), N, kind = workloads.shape_graph(shape)
    J = CouplingMatrix.from_edges(n, (u, v, w))
    params = SolverParams.tuned_for(n, N, seed=0, **tune)
    return shape, J, params, kind, R


def default_steps(params):
    """The reference's step count of a full run: ceil(t_stop / h) (dynamics.py:349)."""
    import math
    return int(math.ceil(params.t_stop / params.h))


def workload_label(shape, J, params, R, window):
    """The `config.workload` string shared by both arms."""
    return (f"{shape}-shape graph n={J.n} nnz={J.nnz} N={params.n_states} "
            f"K={params.K} ks_max={params.ks_max} kn={params.kn} h={params.h}, {R} replicas per GPU, "
            f"{window} Euler steps ({'the whole default schedule t_stop=%g' % params.t_stop if window == default_steps(params) else 'a window of the schedule'}) "
            f"incl. scoring at the reference cadence")


def algorithmic_bytes_per_euler_step(J, R, unit_weights, s_phi=4):
    """every phase read once and written once, graph read once per step."""
    return 2 * R * J.n * s_phi + J.nnz * (4 + (0 if unit_weights else 4)) + (J.n + 1) * 4


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def samples(self):
        try:
            return sum(1 for line in open(self.path) if line.count(",") >= 6)
        except Exception:
            return 0

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 7:
                    continue
                try:
                    sm.append(float(f[0])); mx.append(float(f[1]))
                except ValueError:
                    continue
                for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), f[3:7]):
                    if val.lower().startswith("active"):
                        reasons.add(name)
            os.unlink(self.path)
        except Exception:
            pass
        if sm:
            out.update(sm_mhz=statistics.median(sm), sm_max_mhz=max(mx), reasons=sorted(reasons), samples=len(sm))
        return out


def cpu_oracle_throughput(J, params, kind, R_cpu, window, threads=None):
    """The CPU port of the reference algorithm (oracle/) on the host cores: one bounded sample."""
    from oracle import oracle as O
    O.build()
    threads = threads or O.max_threads()
    t0 = time.perf_counter()
    O.simulate(J.indptr, J.indices, J.data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period,
               kn=params.kn, h=params.h, t_stop=window * params.h, n_states=params.n_states,
               seeds=list(range(R_cpu)), objective=kind, threads=threads)
    dt = time.perf_counter() - t0
    return R_cpu * J.nnz * window / dt, dt, threads


CPU_SAMPLE_STEPS = 2048     # Euler steps of the CPU arm's bounded sample

_REF = None


def reference_package():
    """The UNMODIFIED reference package `oscim` (numpy + numba), pip-installed once from
    /root/reference/pkg into baseline/_ref (git-ignored, travels to the GPU box).
    None when it (or numba) cannot be imported -- the oracle port is then the only CPU arm."""
    global _REF
    if _REF is None:
        _REF = False
        ref = ROOT / "baseline" / "_ref"
        if (ref / "oscim").is_dir():
            os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "oscb_numba_cache"))
            sys.path.insert(0, str(ref))
            try:
                import oscim  # noqa: F401
                _REF = oscim
            except Exception as e:          # numba missing / broken install: say so, fall back to the port
                print(f"bench.py: reference package not importable ({e!r}); CPU arm = oracle port", file=sys.stderr)
            finally:
                sys.path.remove(str(ref))
    return _REF or None


def reference_throughput(indptr, indices, data, n, params, kind, R_cpu, steps, workers=None):
    """`oscim.run_replica_set` (dynamics.py:469-493) of the unmodified reference on the same CSR, parameters
    and a fixed step count; the time is the reference's own RunResult.wall_time (dynamics.py:356, :411:
    RNG init + integrate + scoring + trace) summed over its sequential replica groups."""
    oscim = reference_package()
    workers = workers or (os.cpu_count() or 1)
    Jr = oscim.CouplingMatrix(n, np.asarray(indptr), np.asarray(indices), np.asarray(data), "sparse")
    pr = oscim.SolverParams(K=params.K, ks_max=params.ks_max, ks_period=params.ks_period, kn=params.kn, h=params.h,
                            t_stop=steps * params.h, n_states=params.n_states, seed=0)
    res = oscim.run_replica_set(Jr, pr, kind, replicas=R_cpu, workers=workers)
    assert all(r.steps_executed == steps for r in res)
    group = oscim.dynamics._group_size(n, R_cpu)
    dt = sum(res[k].wall_time for k in range(0, R_cpu, group))      # one wall_time per group (shared by its replicas)
    from oscim.dynamics import resolve_workers
    return R_cpu * len(data) * steps / dt, dt, resolve_workers(workers), group


def reference_sample(n, nnz, R, window):
    """(replicas, steps) of the reference's bounded sample: whole replica groups (dynamics.py:463-466: the reference
    runs groups one after another, so its cost is linear in the replica count), ~10-20 s at ~0.15 G updates/s."""
    group = max(1, 4_000_000 // max(1, n * 256))
    replicas = max(1, min(R, group))
    steps = int(min(window, max(64, 2.5e9 / (nnz * replicas))))
    return replicas, steps


def cpu_sample(J, R, window, scale=1.0):
    """(replicas, steps) of the CPU arm's bounded sample: ~10-20 s of work at ~80 M updates/s/core,
    never more replicas than the workload has (a 1-replica workload is timed with 1 replica), a
    slice of CPU_SAMPLE_STEPS steps of the schedule unless few replicas leave room for more."""
    cores = os.cpu_count() or 1
    target_updates = 12.0 * 80e6 * cores * scale
    steps = min(window, CPU_SAMPLE_STEPS)
    replicas = int(max(1, min(256, R, target_updates / (J.nnz * steps))))
    steps = int(min(window, max(steps, target_updates / (J.nnz * replicas))))
    return replicas, steps


def run_reference_arm(args, rank, world):
    """`--impl reference`: the reference's own CPU implementation on the box's host cores -- the unmodified Python
    package when baseline/_ref imports (kind "reference"), else the oracle port (kind "port").  The port's number
    rides along as `cpu_baseline_port` either way."""
    if rank != 0:
        return
    shape, J, params, kind, R = load_workload(args.workload)
    window = args.window or default_steps(params)
    # bounded sample: many replicas (they are what the CPU threads share) x a slice of the schedule --
    # the CPU cost of an Euler step does not depend on where in the schedule it sits
    R_cpu, steps_cpu = cpu_sample(J, R, window, scale=0.5)
    for _ in range(min(1, args.warmup)):
        cpu_oracle_throughput(J, params, kind, max(1, R_cpu // 8), max(32, steps_cpu // 16))
    port_v, port_dt, port_threads = cpu_oracle_throughput(J, params, kind, R_cpu, steps_cpu)
    port = {"value": port_v, "unit": "updates/s", "cores": port_threads, "kind": "port",
            "sample": f"{R_cpu} replicas x {steps_cpu} Euler steps in {port_dt:.1f} s (oracle/ C+OpenMP port of the reference)"}
    if reference_package() is not None:
        R_ref, steps_ref = reference_sample(J.n, J.nnz, R, window)
        for _ in range(min(1, args.warmup)):        # numba JIT + thread pool
            reference_throughput(J.indptr, J.indices, J.data, J.n, params, kind, min(R_ref, 2), 64)
        t_all = upd = 0.0
        threads = group = 1
        for _ in range(args.steps):
            v, dt, threads, group = reference_throughput(J.indptr, J.indices, J.data, J.n, params, kind, R_ref, steps_ref)
            t_all += dt
            upd += R_ref * J.nnz * steps_ref
        kind_label = "reference"
        sample = (f"oscim.run_replica_set (unmodified reference, numpy + numba, workers={threads}): {R_ref} replicas "
                  f"(one group of {group}) x {steps_ref} Euler steps per step (of {R} replicas x {window} steps per GPU); "
                  f"the reference runs its groups one after another, so its time is linear in replicas and steps")
    else:
        t_all, upd, threads = 0.0, 0.0, 1
        for _ in range(args.steps):
            v, dt, threads = cpu_oracle_throughput(J, params, kind, R_cpu, steps_cpu)
            t_all += dt
            upd += R_cpu * J.nnz * steps_cpu
        kind_label = "port"
        sample = (f"{R_cpu} replicas x {steps_cpu} Euler steps per step (of {R} replicas x {window} steps per GPU), "
                  f"linear in replicas and steps")
    value = upd / t_all
    line = {
        "impl": "reference", "metric": "oscillator-edge updates/sec", "value": value, "unit": "updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_label(shape, J, params, R, window), "replicas_per_gpu": R, "window": window,
                   "sample": sample},
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": threads, "kind": kind_label, "sample": sample},
        "cpu_baseline_port": port,
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def dense_csr(J8):
    """CSR (int64/float64, the reference's layout) of a dense int8 J with zero diagonal -- the CPU arm's input."""
    n = J8.shape[0]
    mask = ~np.eye(n, dtype=bool)
    indices = np.broadcast_to(np.arange(n, dtype=np.int64), (n, n))[mask]
    data = J8[mask].astype(np.float64)
    indptr = np.arange(n + 1, dtype=np.int64) * (n - 1)
    return indptr, indices, data


def dense_cpu_sample(J8, params, steps, threads=None):
    """The CPU oracle port on the dense graph: R = 1, a few Euler steps (~0.3 s each on 16 cores)."""
    from oracle import oracle as O
    O.build()
    threads = threads or O.max_threads()
    indptr, indices, data = dense_csr(J8)
    t0 = time.perf_counter()
    O.simulate(indptr, indices, data, K=params.K, ks_max=params.ks_max, ks_period=params.ks_period, kn=params.kn,
               h=params.h, t_stop=steps * params.h, n_states=2, seeds=[0], objective="maxcut", threads=threads)
    dt = time.perf_counter() - t0
    return len(data) * steps / dt, dt, threads


def bench_dense(args, rank, world, local_rank):
    """configs[4]: dense +-1 SK graph.  One GPU: the persistent tensor-core kernel (csrc/oscb_umma.cuh)
    integrates the whole window in ONE launch.  Several GPUs: J row-sharded over the ranks, phases
    all-gathered every Euler step (strong scaling: the graph is fixed, the rows per GPU shrink)."""
    import torch
    import torch.distributed as dist
    from paper_2505_22631_b200 import workloads
    from paper_2505_22631_b200.model import SolverParams
    n = int(args.workload[2:].split("x")[0])
    R = args.replicas or int(args.workload.split("x")[1])
    window = args.window or 1024
    params = SolverParams.tuned_for(n, 2, seed=0)
    seeds = list(range(R))
    nnz = n * (n - 1)
    peaks, peak_kind = measured_peaks()
    s_phi = 4 if args.precision == "f32" else 8
    label = (f"dense +-1 SK graph n={n} N=2 K={params.K} ks_max={params.ks_max} kn={params.kn} h={params.h}, {R} replica(s), "
             f"window {window} Euler steps incl. scoring every 10")
    if args.impl == "reference":
        if rank != 0:
            return
        J8 = workloads.sk_dense(n)
        steps_cpu = max(2, min(window, int(12.0 * 80e6 * (os.cpu_count() or 1) / nnz)))
        for _ in range(min(1, args.warmup)):
            dense_cpu_sample(J8, params, 2)
        t_all = upd = 0.0
        threads = 1
        for _ in range(args.steps):
            v, dt, threads = dense_cpu_sample(J8, params, steps_cpu)
            t_all += dt
            upd += nnz * steps_cpu
        value = upd / t_all
        sample = f"1 replica x {steps_cpu} Euler steps per step (of {R} x {window}), linear in replicas and steps"
        print(json.dumps({
            "impl": "reference", "metric": "oscillator-edge updates/sec", "value": value, "unit": "updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": label, "replicas": R, "window": window, "sample": sample},
            "cpu_baseline": {"value": value, "unit": "updates/s", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}, "gpu_launches": 0}), flush=True)
        return

    J8 = workloads.sk_dense(n)                                   # int8, symmetric, zero diagonal
    if world == 1:
        from paper_2505_22631_b200 import dynamics as dyn
        g = dyn.DeviceGraph.from_dense(local_rank, J8.astype(np.float64))

        def device_step():
            return dyn.run_batch(None, params, "maxcut", seeds, precision=args.precision, device=local_rank, steps=window,
                                 want_phases=False, want_states=False, want_traces=False, graph=g)

        for _ in range(args.warmup):
            device_step()
        torch.cuda.synchronize()
        sampler = ClockSampler(local_rank)
        sampler.start()
        dev_ms, launches, last = 0.0, 0, None
        for _ in range(args.steps):
            last = device_step()
            dev_ms += last.device_ms
            launches += last.kernel_launches
        torch.cuda.synchronize()
        # a dense window is tens of milliseconds, nvidia-smi needs a few hundred to deliver its first sample: keep the
        # same kernel running (untimed) until the sampler has seen the load
        t_s = time.perf_counter()
        while sampler.proc is not None and sampler.samples() < 3 and time.perf_counter() - t_s < 5.0:
            device_step()
            torch.cuda.synchronize()
        clocks = sampler.stop()
        phi0_pinned = torch.empty((R, n), dtype=torch.float64, pin_memory=True)
        phi0 = phi0_pinned.numpy()
        phi0[...] = dyn._initial_phases_host(local_rank, seeds, n)
        dyn.run_batch(None, params, "maxcut", seeds, precision=args.precision, device=local_rank, steps=window,
                      phi0=phi0, graph=g)                           # untimed: first use of the host-buffer path sizes the block pool
        t0 = time.perf_counter()
        h2d = d2h = 0
        for _ in range(args.steps):
            b = dyn.run_batch(None, params, "maxcut", seeds, precision=args.precision, device=local_rank, steps=window,
                              phi0=phi0, graph=g)
            h2d = phi0.nbytes + 8 * R
            d2h = b.final_phases.nbytes + b.best_states.nbytes + b.best_objective.nbytes + b.energy.nbytes + b.best_trace.nbytes
        e2e_s = time.perf_counter() - t0
        value = R * nnz * window * args.steps / (dev_ms / 1e3)
        e2e_value = R * nnz * window * args.steps / e2e_s
        bits, per_launch = g.tc_stream(2, R)                      # 8 = int8 J tiles, 4 = packed e2m1 tiles (R <= 12)
        chunks = -(-R // per_launch)                              # launches per window
        # algorithmic HBM bytes per Euler step: J once (bits / 8 bytes per coupling) per launch + phases read and written
        bytes_step = chunks * n * n * bits // 8 + 2 * R * n * s_phi
        kernel_ms = dev_ms / args.steps
        achieved = bytes_step * window / (kernel_ms * 1e-3) / 1e9
        traffic = None
        tpath = ROOT / "profiles" / "dram_traffic.json"
        if tpath.exists():
            tj = json.loads(tpath.read_text())
            t = tj.get(f"{args.workload}:{last.kernel}-{bits}b:{args.precision}:{window}") or \
                (tj.get(f"{args.workload}:{last.kernel}:{args.precision}:{window}") if bits == 8 else None)
            if t:
                traffic = t["dram_bytes_per_launch"]
        # tensor work issued: 2 * 128-row tiles * N columns * n per step (N = 16-padded digit planes: 9 per replica
        # against the int8 tiles, 21 against the e2m1 tiles)
        nb = -(-(9 if bits == 8 else 21) * min(R, per_launch) // 16) * 16
        tensor_tops = 2.0 * n * n * nb * chunks * window / (kernel_ms * 1e-3) / 1e12
        line = {
            "metric": "oscillator-edge updates/sec", "value": value, "unit": "updates/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": kernel_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": args.precision + (" epilogue, int8 x int8 -> int32 tensor-core sums" if bits == 8 else
                                                           " epilogue, e2m1 x e2m1 -> f32 tensor-core sums (exact integers)"),
            "data": "synthetic",
            "config": {"workload": label, "replicas": R, "window": window, "kernel": last.kernel, "coupling_bits": bits,
                       "replicas_per_launch": last.replicas_per_cta, "smem_bytes": last.smem_bytes, "parallelism": "one GPU",
                       "l2": "J (%.0f MB at %d bits per coupling) exceeds the 126 MB L2 and is re-read from HBM every Euler step "
                             "(ncu: DRAM bytes per step = the image size); no flush needed" % (n * n * bits / 8e6, bits)},
            "e2e": {"value": e2e_value, "unit": "updates/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "clocks": {"sm_mhz": clocks["sm_mhz"], "sm_max_mhz": clocks["sm_max_mhz"], "reasons": clocks["reasons"]},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": traffic, "peak_kind": peak_kind, "kernel": "k_dense_umma",
                         "algorithmic_bytes_per_launch": bytes_step * window / chunks, "bytes_per_update": bytes_step / (R * nnz),
                         "tensor_tops_issued": tensor_tops,
                         "note": ("one persistent launch = the whole window; per Euler step it streams J (int8) once from HBM" if bits == 8 else
                                  "one persistent launch = the whole window; per Euler step it streams J (packed e2m1, n^2/2 bytes) once "
                                  "from HBM (kind::mxf4 MMAs against e2m1 base-9 digit planes); the same step on the int8 stream "
                                  "(OSCB_UMMA_FP4=0) sits at 1.0 of HBM with twice the bytes")},
        }
        if not args.no_cpu_baseline:
            steps_cpu = max(2, min(window, int(12.0 * 80e6 * (os.cpu_count() or 1) / nnz)))
            v, dt, threads = dense_cpu_sample(J8, params, steps_cpu)
            line["cpu_baseline"] = {"value": v, "unit": "updates/s", "cores": threads, "kind": "port",
                                    "sample": f"1 replica x {steps_cpu} Euler steps of the same graph in {dt:.1f} s "
                                              f"(oracle/ C+OpenMP port of the reference; linear in replicas and steps)"}
        print(json.dumps(line), flush=True)
        return

    # several GPUs: J row-sharded (128-row aligned), ONE fused persistent kernel per rank; the per-step phase
    # exchange is stores into the peers' exchange blocks from inside the kernel (dense_fused.py)
    from paper_2505_22631_b200 import dense_fused, dynamics as dyn
    rows = (n // world) // 128 * 128
    lo, hi = rank * rows, (n if rank == world - 1 else (rank + 1) * rows)
    g = dyn.DeviceGraph.from_dense(local_rank, J8[lo:hi].astype(np.float64), lo, hi)
    del J8
    pairs = n * (n - 1) // 2
    phi0 = dyn._initial_phases_host(local_rank, seeds, n)

    nccl_backend = None
    if args.exchange == "nccl":
        from paper_2505_22631_b200 import dense_sharded
        if (n // world) * world != n:
            raise SystemExit("--exchange nccl needs n divisible by the rank count")
        rows = n // world
        lo, hi = rank * rows, (rank + 1) * rows
        g.close()
        nccl_backend = dense_sharded.CudaDenseShard(workloads.sk_dense(n)[lo:hi].astype(np.float64), n, lo, hi, local_rank, args.precision)

    def one():
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        if nccl_backend is not None:
            run = dense_sharded.run_dense_sharded(nccl_backend, params, "maxcut", seeds, pair_count=pairs, phi0=phi0, steps=window)
            res = run.batch
        else:
            res = dense_fused.run_dense_fused(None, n, lo, hi, params, seeds, device=local_rank, pair_count=pairs, phi0=phi0,
                                              graph=g.handle, precision=args.precision, steps=window)
        torch.cuda.synchronize()
        return time.perf_counter() - t0, res

    for _ in range(args.warmup):
        one()
    sampler = ClockSampler(local_rank)
    sampler.start()
    total = dev_ms = 0.0
    for _ in range(args.steps):
        dt, res = one()
        total += dt
        dev_ms += res.device_ms
    clocks = sampler.stop()
    t = torch.tensor([total, dev_ms / 1e3], dtype=torch.float64,
                     device=f"cuda:{local_rank}" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total, dev_s = (float(x) for x in t.cpu())
    value = R * nnz * window * args.steps / dev_s
    e2e_value = R * nnz * window * args.steps / total
    # per GPU: its shard of J once per Euler step and session (sessions of <= 28 replicas; one of <= 12 streams e2m1 tiles)
    sessions = [min(dense_fused.MAX_REPLICAS, R - r0) for r0 in range(0, R, dense_fused.MAX_REPLICAS)]
    chunks = len(sessions)
    bytes_step = (sum((hi - lo) * n * g.tc_stream(2, r)[0] // 8 for r in sessions) if nccl_backend is None      # (int8 J on the SIMT path)
                  else (hi - lo) * n) + 2 * R * n * s_phi
    achieved = bytes_step * window * args.steps / dev_s / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": "oscillator-edge updates/sec", "value": value, "unit": "updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dev_s / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": args.precision + " epilogue, int8 x int8 -> int32 tensor-core sums", "data": "synthetic",
            "config": {"workload": label + f"; J row-sharded over {world} GPUs, phase digits pushed to the peers from inside the kernel every Euler step",
                       "replicas": R, "window": window, "kernel": "dense-tc" if nccl_backend is None else "dense-sharded (SIMT step + ncclAllGather)",
                       "exchange": args.exchange, "parallelism": f"row-shard x{world}",
                       "l2": "a J shard below ~100 MB (n=16384 at 4+ GPUs) stays L2 resident between Euler steps; the roofline below still charges it to HBM"},
            "e2e": {"value": e2e_value, "unit": "updates/s", "h2d_bytes_per_step": int(8 * R * n + 8 * R),
                    "d2h_bytes_per_step": int(9 * R * (hi - lo) + 8 * R * 4),
                    "note": "run_dense_fused: host phases in, host results out, session set-up (IPC exchange, barrier) included; wall clock"},
            "gpu_launches": int(chunks * args.steps),
            "clocks": {"sm_mhz": clocks["sm_mhz"], "sm_max_mhz": clocks["sm_max_mhz"], "reasons": clocks["reasons"]},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": None, "peak_kind": peak_kind, "kernel": "k_dense_umma",
                         "note": "per GPU"},
        }), flush=True)


def reference_target():
    """0.99 x the best `best_objective` of 96 CPU-oracle replicas (numpy's noise stream, whole default schedule)
    on the synthetic G22-shape graph -- tests/golden/fullsize_fixtures.npz, written by
    tests/golden/make_fullsize_fixtures.py."""
    f = ROOT / "tests" / "golden" / "fullsize_fixtures.npz"
    if not f.exists():
        return None
    z = np.load(f)
    return float(z["g22_target_best"]), int(len(z["g22_best"]))


def torch_sm_count(device):
    import torch
    return int(torch.cuda.get_device_properties(device).multi_processor_count)


def time_to_target(dyn, J, params, kind, seeds, args, local_rank, phi0, R):
    """Time-to-99 %-best-cut on the G22 shape, both arms against the SAME reference-derived target."""
    anchor = reference_target()
    run = lambda **kw: dyn.run_batch(J, params, kind, seeds, precision=args.precision, device=local_rank, kernel=args.kernel,
                                     want_phases=False, want_traces=False, **kw)
    if anchor is None:
        best, how_target = float(run(want_states=False).best_objective.max()), "0.99 x best cut of this GPU batch (fixture missing)"
    else:
        best, how_target = anchor[0], f"0.99 x best best_objective of {anchor[1]} CPU-oracle seeds (tests/golden/fullsize_fixtures.npz)"
    target = 0.99 * best
    hit = run(target=target, want_states=False)
    hits = hit.first_hit_step[hit.first_hit_step >= 0]
    first = int(hits.min()) if len(hits) else -1
    measured = e2e_hit = None
    if first >= 0:
        # the solve actually stopped at the step that reaches the target: device time, and wall clock
        # through the API with host phases in and the best states / objectives out
        stop = max(1, first + 1)
        for _ in range(2):
            short = run(steps=stop, phi0=phi0)
        t0 = time.perf_counter()
        short = run(steps=stop, phi0=phi0)
        e2e_hit = time.perf_counter() - t0
        measured = short.device_ms / 1e3
        assert float(short.best_objective.max()) >= target
    out = {"best_cut_reference": best, "target": target, "target_from": how_target, "first_hit_step": first,
           "steps_total": hit.steps, "seconds": measured, "e2e_seconds": e2e_hit, "gpu_best_cut": float(hit.best_objective.max()),
           "how": "a run of first_hit_step + 1 Euler steps of all replicas: CUDA-event time of the launch, and wall clock "
                  "of the API call with host buffers",
           "full_run_seconds": hit.device_ms / 1e3, "replicas": R}
    # The metric does not prescribe the batch: fewer replicas mean a shorter Euler step (one replica per SM: ~5.6 us; 9
    # replicas on 16-CTA clusters, the latency kernel: ~3.5 us) at the price of a later first hit.  Same target, same seeds 0..R-1.
    sm = torch_sm_count(local_rank)
    small = []
    for R_try, rt in ((2 * sm, 2), (sm, 1), (max(1, sm // 16), 0)):
        sd = list(range(R_try))
        h = dyn.run_batch(J, params, kind, sd, precision=args.precision, device=local_rank, target=target, replicas_per_cta=rt,
                          want_phases=False, want_states=False, want_traces=False)
        hs = h.first_hit_step[h.first_hit_step >= 0]
        rec = {"replicas": R_try, "kernel": h.kernel, "replicas_per_cta": h.replicas_per_cta, "first_hit_step": int(hs.min()) if len(hs) else -1,
               "seconds": None, "e2e_seconds": None}
        if len(hs):
            stop = int(hs.min()) + 1
            p0 = np.ascontiguousarray(phi0[:R_try]) if R_try <= len(phi0) else dyn._initial_phases_host(local_rank, sd, J.n)
            for _ in range(2):
                sh = dyn.run_batch(J, params, kind, sd, precision=args.precision, device=local_rank, steps=stop, phi0=p0, replicas_per_cta=rt,
                                   want_phases=False, want_traces=False)
            t0 = time.perf_counter()
            sh = dyn.run_batch(J, params, kind, sd, precision=args.precision, device=local_rank, steps=stop, phi0=p0, replicas_per_cta=rt,
                               want_phases=False, want_traces=False)
            rec.update(seconds=sh.device_ms / 1e3, e2e_seconds=time.perf_counter() - t0, reached=bool(sh.best_objective.max() >= target))
        small.append(rec)
    out["smaller_batches"] = small
    done = [r for r in small if r["seconds"] is not None] + ([{"replicas": R, "seconds": measured}] if measured is not None else [])
    if done:
        best_rec = min(done, key=lambda r: r["seconds"])
        out["fastest"] = {"replicas": best_rec["replicas"], "seconds": best_rec["seconds"]}
    if not args.no_cpu_baseline:
        # the CPU arm to the same target: one replica per host thread (seeds 0..T-1), best-so-far sampled every 50 steps
        # (dynamics.py:377-384 best_trace); then the run that stops at the first sample reaching the target is timed
        from oracle import oracle as O
        O.build()
        T = O.max_threads()
        sim = lambda t_stop, stride: O.simulate(J.indptr, J.indices, J.data, K=params.K, ks_max=params.ks_max,
                                                ks_period=params.ks_period, kn=params.kn, h=params.h, t_stop=t_stop,
                                                n_states=params.n_states, seeds=list(range(T)), objective=kind,
                                                trace_stride=stride, threads=T)
        t0 = time.perf_counter()
        full = sim(params.t_stop, 50 * params.h)
        full_s = time.perf_counter() - t0
        reached = np.nonzero(full.best_trace.max(axis=0) >= target)[0]
        cpu = {"replicas": T, "cores": T, "kind": "port", "full_run_seconds": full_s, "best_cut": float(full.best_objective.max())}
        if len(reached):
            t_hit = float(full.trace_t[reached[0]])
            t0 = time.perf_counter()
            part = sim(max(t_hit, 2 * params.h), 50 * params.h)
            cpu.update(seconds=time.perf_counter() - t0, first_hit_t=t_hit, first_hit_step=int(round(t_hit / params.h)),
                       reached=bool(part.best_objective.max() >= target))
        else:
            cpu.update(seconds=None, note="target not reached by this batch within the default schedule")
        out["cpu"] = cpu
    return out


def self_launch(n_ranks):
    """Re-run this command line under torch.distributed.run with `n_ranks` local ranks.  NCCL's communicator
    INIT lines go to stderr (NCCL_DEBUG=INFO unless the caller set it) so the rank count is visible from outside."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n_ranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="G22x1024", help="one of %s, or SK<n>x<replicas> (dense, row-sharded)" % sorted(WORKLOADS))
    ap.add_argument("--window", type=int, default=0,
                    help="Euler steps per bench step; 0 = the workload's whole default schedule ceil(t_stop / h) "
                         "(dense SK workloads: 1024)")
    ap.add_argument("--precision", default="f32", choices=["f32", "f64"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "stream", "resident", "lowdeg", "cluster"])
    ap.add_argument("--replicas", type=int, default=0, help="override replicas per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl"],
                    help="row-sharded dense runs (SK<n>x<R> under torchrun): 'fused' = phase digits pushed into the peers' B images "
                         "from inside the persistent tensor-core kernel; 'nccl' = the baseline it replaces, one SIMT step launch + "
                         "ncclAllGather of the phase slices per Euler step (dense_sharded.py)")
    ap.add_argument("--no-target", action="store_true", help="skip the time-to-99%%-best-cut run")
    ap.add_argument("--no-parity-mode", action="store_true", help="skip the float64 sub-record of the same workload")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl != "reference":
        # `python bench.py --gpus N` without a launcher: become N ranks (one process per GPU, rendezvous on 127.0.0.1)
        raise SystemExit(self_launch(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus if args.impl == "reference" else 1)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("OSCB_BENCH_DRYRUN"):
        # launcher check (tests/test_bench_launch.py): rendezvous only, no device work
        import torch.distributed as dist
        import torch
        if world > 1:
            dist.init_process_group("gloo")
            t = torch.ones(1)
            dist.all_reduce(t)
            seen = int(t.item())
            dist.destroy_process_group()
        else:
            seen = 1
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_seen": seen, "gpus_arg": args.gpus}), flush=True)
        return
    if args.impl == "reference":
        if args.workload.startswith("SK"):
            bench_dense(args, rank, world, 0)
        else:
            run_reference_arm(args, rank, world)
        return

    import torch
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    # OSCB_BENCH_BACKEND=gloo lets several ranks share one GPU (a functional check of the multi-rank
    # paths on a single-GPU box; the timings of such a run mean nothing)
    backend = os.environ.get("OSCB_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local_rank = local_rank % torch.cuda.device_count()
    elif world > torch.cuda.device_count() and "LOCAL_RANK" in os.environ:
        raise SystemExit(f"bench.py --gpus {world}: this node has {torch.cuda.device_count()} GPU(s); "
                         f"OSCB_BENCH_BACKEND=gloo shares one GPU between the ranks for a functional check")
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)

    if args.workload.startswith("SK"):
        bench_dense(args, rank, world, local_rank)
        if dist is not None:
            dist.destroy_process_group()
        return

    from paper_2505_22631_b200 import _native as nat
    from paper_2505_22631_b200 import dynamics as dyn
    shape, J, params, kind, R = load_workload(args.workload)
    if args.replicas:
        R = args.replicas
    window = args.window or default_steps(params)
    seeds = [rank * R + r for r in range(R)]           # contiguous replica-index block per rank
    g = dyn.device_graph(J, local_rank)
    info = g.info()
    info_sm_count = torch.cuda.get_device_properties(local_rank).multi_processor_count
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local_rank}")

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    def device_step(first_step):
        # phases generated on the device, nothing copied back: inputs resident when the clock starts
        return dyn.run_batch(J, params, kind, seeds, precision=args.precision, device=local_rank, kernel=args.kernel,
                             steps=window, first_step=first_step, want_phases=False, want_states=False, want_traces=False)

    for w in range(args.warmup):
        device_step(0)
        flush.zero_()
    barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    dev_ms, launches, wall0 = 0.0, 0, time.perf_counter()
    last = None
    for k in range(args.steps):
        last = device_step(0)
        dev_ms += last.device_ms
        launches += last.kernel_launches
        flush.zero_()                                   # L2 flush between timed iterations
    barrier()
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()

    # end to end through the public API with host buffers
    phi0_pinned = torch.empty((R, J.n), dtype=torch.float64, pin_memory=True)     # pinned host source of the h2d copy
    phi0 = phi0_pinned.numpy()
    phi0[...] = dyn._initial_phases_host(local_rank, seeds, J.n)
    barrier()
    e2e0 = time.perf_counter()
    h2d = d2h = 0
    for k in range(args.steps):
        b = dyn.run_batch(J, params, kind, seeds, precision=args.precision, device=local_rank, kernel=args.kernel,
                          steps=window, phi0=phi0)
        h2d = phi0.nbytes + 8 * R
        d2h = b.final_phases.nbytes + b.best_states.nbytes + b.best_objective.nbytes + b.energy.nbytes + b.best_trace.nbytes + 8 * R
    barrier()
    e2e_s = time.perf_counter() - e2e0

    t_dev = torch.tensor([dev_ms / 1e3, e2e_s, wall], dtype=torch.float64,
                         device=f"cuda:{local_rank}" if dist is None or dist.get_backend() == "nccl" else "cpu")
    if dist is not None:
        dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
    t_dev_s, t_e2e_s, t_wall_s = (float(x) for x in t_dev.cpu())
    updates_per_step = world * R * J.nnz * window
    value = updates_per_step * args.steps / t_dev_s
    e2e_value = updates_per_step * args.steps / t_e2e_s

    peaks, peak_kind = measured_peaks()
    s_phi = 4 if args.precision == "f32" else 8
    bytes_per_launch = algorithmic_bytes_per_euler_step(J, R, bool(info.unit_weights), s_phi) * window
    if last.kernel in ("resident", "lowdeg", "cluster"):
        kernel_ms = dev_ms / args.steps           # one persistent launch integrates the whole window
        launch_bytes = bytes_per_launch
        launch_updates = R * J.nnz * window
    else:
        kernel_ms = dev_ms / args.steps / window  # per Euler-step launch (scoring launches included in the time)
        launch_bytes = bytes_per_launch / window
        launch_updates = R * J.nnz
    achieved = launch_bytes / (kernel_ms * 1e-3) / 1e9
    # the resource that actually binds the resident kernel: every update gathers one (cos, sin)
    # pair from shared memory (8 B float32 / 16 B float64); the SM array moves 128 B/clk/SM
    sm_mhz = clocks["sm_mhz"] or peaks.get("sm_max_mhz", 1965.0)
    smem_peak = 128.0 * info_sm_count * sm_mhz * 1e6 / 1e9
    smem_achieved = launch_updates * (2 * s_phi) / (kernel_ms * 1e-3) / 1e9
    kernel_name = {"resident": "k_resident_fast" if args.precision == "f32" else "k_resident",
                   # (N = 2 rows of more than one group run two replicas per lane: oscb_lowdeg_host.hpp)
                   "lowdeg": "k_lowdeg_pair" if (params.n_states == 2 and int(np.diff(J.indptr).max()) > 4 and last.replicas_per_cta > 1)
                             else "k_lowdeg"}.get(last.kernel, last.kernel)
    # DRAM bytes per launch cannot be counted from inside an untraced run: the figure is the one transcribed from the
    # committed `ncu --set full` capture of this exact (workload, kernel, precision, window); anything else says so
    traffic, traffic_source = None, "not captured for this (workload, kernel, precision, window)"
    tpath = ROOT / "profiles" / "dram_traffic.json"
    if tpath.exists():
        t = json.loads(tpath.read_text()).get(f"{args.workload}:{last.kernel}:{args.precision}:{window}")
        if t:
            traffic, traffic_source = t["dram_bytes_per_launch"], t.get("source", "profiles/dram_traffic.json")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": traffic, "traffic_source": traffic_source, "peak_kind": peak_kind,
                "kernel": kernel_name,
                "algorithmic_bytes_per_launch": launch_bytes, "bytes_per_update": launch_bytes / launch_updates,
                "binding_resource": {"name": "shared-memory gather wavefronts", "achieved": smem_achieved, "peak": smem_peak,
                                     "unit": "GB/s", "frac": smem_achieved / smem_peak,
                                     "how": "updates x 8 B (cos, sin) pair / kernel time vs 128 B/clk/SM x SMs x measured SM clock"},
                "note": "the persistent kernel keeps phases and pairs on chip for the whole window, so DRAM traffic is ~0 "
                        "by design and the HBM fraction is small by construction; shared-memory gather bandwidth and "
                        "instruction issue bind (DESIGN.md section 4)"}
    if last.kernel in ("resident", "lowdeg", "cluster") and last.kernel_launches > 1:
        # the mixed-tile schedule of k_lowdeg_pair: windows of two concurrent grids (tiles of 8 and of 4 replicas); the unit
        # the figures above are quoted per is the whole schedule of one bench step, not one of its launches
        roofline["launches_per_step"] = int(last.kernel_launches)
        roofline["note"] += ("; one bench step is a schedule of %d launches (windows x two concurrent grids on two streams), "
                             "achieved = algorithmic bytes of the step / its device time" % last.kernel_launches)

    line = {
        "metric": "oscillator-edge updates/sec", "value": value, "unit": "updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_dev_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": workload_label(shape, J, params, R, window), "replicas_per_gpu": R, "window": window,
                   "kernel": last.kernel, "replicas_per_cta": last.replicas_per_cta, "smem_bytes": last.smem_bytes,
                   "l2": "256 MB flush write between timed iterations", "parallelism": f"replica-shard x{world}",
                   "wall_s_timed_region": t_wall_s},
        "e2e": {"value": e2e_value, "unit": "updates/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "clocks": {"sm_mhz": clocks["sm_mhz"], "sm_max_mhz": clocks["sm_max_mhz"], "reasons": clocks["reasons"]},
        "roofline": roofline,
    }

    if rank == 0 and not args.no_parity_mode and args.precision == "f32":
        # the same workload in the reference's own arithmetic (float64 state, the reference's operation order:
        # dynamics.py:155-190) -- the throughput the parity mode sustains, beside the float32 headline
        k64 = args.kernel if args.kernel in ("auto", "stream", "resident") else "auto"     # (the others are float32 only)
        dyn.run_batch(J, params, kind, seeds, precision="f64", device=local_rank, kernel=k64, steps=min(window, 256),
                      want_phases=False, want_states=False, want_traces=False)
        p64 = dyn.run_batch(J, params, kind, seeds, precision="f64", device=local_rank, kernel=k64, steps=window,
                            want_phases=False, want_states=False, want_traces=False)
        b64 = algorithmic_bytes_per_euler_step(J, R, bool(info.unit_weights), 8) * window
        ach64 = b64 / (p64.device_ms * 1e-3) / 1e9
        line["parity_mode"] = {"precision": "f64", "value": R * J.nnz * window / (p64.device_ms * 1e-3), "unit": "updates/s",
                               "ms_per_step": p64.device_ms, "kernel": p64.kernel, "replicas_per_cta": p64.replicas_per_cta,
                               "frac": ach64 / peaks["hbm_gbs"], "achieved_gbs": ach64,
                               "note": "one solve of the same workload (this rank's replicas) with precision='f64', CUDA-event time; "
                                       "frac = algorithmic bytes at 8 B per phase / time / measured HBM peak"}

    if rank == 0 and not args.no_target and shape == "G22":
        line["time_to_99pct_best_cut"] = time_to_target(dyn, J, params, kind, seeds, args, local_rank, phi0, R)

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        R_cpu, steps_cpu = cpu_sample(J, R, window)
        v, dt, threads = cpu_oracle_throughput(J, params, kind, R_cpu, steps_cpu)
        port = {"value": v, "unit": "updates/s", "cores": threads, "kind": "port",
                "sample": f"{R_cpu} replicas x {steps_cpu} Euler steps of the same workload in {dt:.1f} s "
                          f"(oracle/ C+OpenMP port of the reference; linear in replicas and steps)"}
        line["cpu_baseline"] = port
        if reference_package() is not None:
            try:
                R_ref, steps_ref = reference_sample(J.n, J.nnz, R, window)
                reference_throughput(J.indptr, J.indices, J.data, J.n, params, kind, min(R_ref, 2), 64)   # JIT warm-up
                rv, rdt, rthreads, group = reference_throughput(J.indptr, J.indices, J.data, J.n, params, kind, R_ref, steps_ref)
                line["cpu_baseline"] = {
                    "value": rv, "unit": "updates/s", "cores": rthreads, "kind": "reference",
                    "sample": f"oscim.run_replica_set of the unmodified reference (baseline/_ref, numpy + numba, workers={rthreads}): "
                              f"{R_ref} replicas (one group of {group}) x {steps_ref} Euler steps of the same workload in {rdt:.1f} s; "
                              f"groups run one after another in the reference, so linear in replicas and steps"}
                line["cpu_baseline_port"] = port
            except Exception as e:
                line["cpu_baseline_reference_error"] = repr(e)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
