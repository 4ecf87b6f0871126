"""Command-line front end on top of the GPU solver: `solve`, `bench`, `sweep`, `scaling`.

Same sub-commands, flags, output schemas and exit codes as the reference's CLI
(/root/reference/pkg/src/oscim/cli.py: flags :64-74, report :94-126, trace CSV :129-133,
manifest bench :175-259, sweep :283-324, scaling :335-360, exit codes :36-39, :414-436), so
scripts written against `python -m oscim ...` run unchanged against
`python -m paper_2505_22631_b200 ...`.  Extra flags select GPU specifics: --precision, --device,
--kernel.  Exit codes: 0 success, 1 usage error, 2 input/parse error, 3 numerical failure.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import sys
from pathlib import Path
from typing import Dict, List, Optional

import numpy as np

from .dynamics import NumericalError, resolve_workers, run_replica_set, run_replicas
from .model import Graph, SolverParams, coloring_conflicts, cut_value, threshold_phases
from .problems import ParseError, build_maxcut_coupling, load_instance

EXIT_OK, EXIT_USAGE, EXIT_INPUT, EXIT_NUMERIC = 0, 1, 2, 3

TRACE_HEADER = "t,energy,ks,best_objective"
BENCH_COLUMNS = ["instance", "kind", "n", "best_objective", "reference", "accuracy_pct", "satisfied_fraction",
                 "wall_time_s", "steps", "seed", "replicas", "error"]
SWEEP_HEADER = "K,ks_max,accuracy"
SCALING_HEADER = "n,workers,wall_time_s"

# SolverParams fields settable from flags / manifest columns, with their casts
TUNABLES = {"K": float, "ks_max": float, "ks_period": float, "kn": float, "h": float, "t_stop": float, "batch_size": int}


class UsageError(Exception):
    """Bad flag combination (exit code 1)."""


class _ArgParser(argparse.ArgumentParser):
    def error(self, message):          # the documented contract is exit 1, argparse's default is 2
        self.print_usage(sys.stderr)
        print(f"{self.prog}: error: {message}", file=sys.stderr)
        raise SystemExit(EXIT_USAGE)


def _gpu_kwargs(args) -> dict:
    return {"precision": getattr(args, "precision", None), "device": getattr(args, "device", None),
            "kernel": getattr(args, "kernel", "auto")}


def _tuned(args, n: int, n_states: int, seed: int, extra: Optional[dict] = None) -> SolverParams:
    over = {k: getattr(args, k) for k in TUNABLES if getattr(args, k, None) is not None}
    over.update(extra or {})
    return SolverParams.tuned_for(n, n_states=n_states, seed=seed, **over)


def _load(args):
    if args.problem == "maxcut" and args.colors is not None:
        raise UsageError("--colors is only valid with --problem coloring")
    return load_instance(args.path, args.problem, args.colors if args.problem == "coloring" else 2)


def _report(inst, params: SolverParams, result, replicas: int, workers: int, reference: Optional[float]) -> dict:
    satisfied = accuracy = None
    if inst.kind == "coloring":
        _, satisfied = coloring_conflicts(inst.graph, result.best_assignment)
        if reference is not None:
            accuracy = 100.0 * satisfied
    elif reference is not None:
        accuracy = 100.0 * result.best_objective / reference
    fields = ("K", "ks_max", "ks_period", "kn", "h", "t_stop", "n_states", "seed", "batch_size")
    return {"instance": inst.source_name, "problem": inst.kind, "n": inst.graph.node_count, "edges": inst.graph.edge_count,
            "params": {f: getattr(params, f) for f in fields}, "replicas": replicas, "workers": workers,
            "best_objective": result.best_objective, "satisfied_fraction": satisfied, "reference": reference,
            "accuracy_pct": accuracy, "wall_time_s": result.wall_time, "steps": result.steps_executed, "seed": params.seed,
            # (beyond the reference's report: the arithmetic of this run -- float32 is this package's default)
            "precision": getattr(result, "precision", "f32")}


def _emit(text: str, out: Optional[str]) -> None:
    if out:
        Path(out).write_text(text)
    else:
        sys.stdout.write(text)


# ---------------------------------------------------------------------------------------------
def cmd_solve(args) -> int:
    inst = _load(args)
    params = _tuned(args, inst.graph.node_count, inst.n_states, args.seed)
    workers = resolve_workers(args.workers)
    result = run_replicas(inst.coupling(), params, inst.kind, replicas=args.replicas, workers=workers, **_gpu_kwargs(args))
    _emit(json.dumps(_report(inst, params, result, args.replicas, workers, args.reference), indent=2, sort_keys=True) + "\n",
          args.out)
    if args.trace:
        rows = [TRACE_HEADER] + [f"{t!r},{e!r},{ks!r},{b!r}" for (t, e, ks), b in zip(result.energy_trace, result.best_trace)]
        Path(args.trace).write_text("\n".join(rows) + "\n")
    return EXIT_OK


def _manifest_rows(path: str) -> List[Dict[str, str]]:
    kept = [ln for ln in Path(path).read_text().splitlines() if ln.strip() and not ln.lstrip().startswith("#")]
    if not kept:
        return []
    reader = csv.DictReader(io.StringIO("\n".join(kept)))
    if reader.fieldnames is None or not {"path", "kind", "reference"} <= set(reader.fieldnames):
        raise ParseError(f"manifest must have columns path,kind,reference (got {reader.fieldnames})")
    return list(reader)


def _cell(row: Dict[str, str], key: str, cast, default=None):
    raw = row.get(key)
    return default if raw is None or not str(raw).strip() else cast(raw)


def cmd_bench(args) -> int:
    base = Path(args.manifest).parent
    table, accuracies = [], []
    failures, numeric, total = 0, False, 0.0
    for row in _manifest_rows(args.manifest):
        rec = dict.fromkeys(BENCH_COLUMNS, "")
        where = Path(row["path"])
        where = where if where.is_absolute() else base / where
        rec["instance"] = where.name
        try:
            kind = row["kind"].strip()
            if kind not in ("maxcut", "coloring"):
                raise ParseError(f"unknown kind {kind!r} in manifest")
            inst = load_instance(where, kind, _cell(row, "colors", int, 3) if kind == "coloring" else 2)
            extra = {k: _cell(row, k, cast) for k, cast in TUNABLES.items() if _cell(row, k, cast) is not None}
            seed = _cell(row, "seed", int, args.seed)
            replicas = _cell(row, "replicas", int, args.replicas)
            reference = _cell(row, "reference", float, None)
            params = _tuned(args, inst.graph.node_count, inst.n_states, seed, extra)
            workers = resolve_workers(args.workers)
            result = run_replicas(inst.coupling(), params, inst.kind, replicas=replicas, workers=workers, **_gpu_kwargs(args))
            rep = _report(inst, params, result, replicas, workers, reference)
            blank = lambda v: "" if v is None else v      # noqa: E731
            rec.update(kind=inst.kind, n=inst.graph.node_count, best_objective=rep["best_objective"],
                       reference=blank(reference), accuracy_pct=blank(rep["accuracy_pct"]),
                       satisfied_fraction=blank(rep["satisfied_fraction"]), wall_time_s=rep["wall_time_s"],
                       steps=rep["steps"], seed=seed, replicas=replicas)
            if rep["accuracy_pct"] is not None:
                accuracies.append(rep["accuracy_pct"])
            total += rep["wall_time_s"]
        except NumericalError as exc:
            rec["error"], failures, numeric = str(exc), failures + 1, True
        except (ParseError, OSError, ValueError) as exc:
            rec["error"], failures = str(exc), failures + 1
        table.append(rec)
    aggregate = {"instances": len(table), "failures": failures,
                 "min_accuracy_pct": min(accuracies) if accuracies else None,
                 "mean_accuracy_pct": float(np.mean(accuracies)) if accuracies else None,
                 "total_wall_time_s": total}
    if args.json:
        _emit(json.dumps({"rows": table, "aggregate": aggregate}, indent=2, sort_keys=True) + "\n", args.out)
    else:
        buf = io.StringIO()
        writer = csv.DictWriter(buf, fieldnames=BENCH_COLUMNS)
        writer.writeheader()
        writer.writerows(table)
        _emit(buf.getvalue(), args.out)
        print(f"bench: {aggregate['instances']} instances, {failures} failures, min acc {aggregate['min_accuracy_pct']}, "
              f"mean acc {aggregate['mean_accuracy_pct']}, total {total:.2f}s", file=sys.stderr)
    return EXIT_NUMERIC if numeric else (EXIT_INPUT if failures else EXIT_OK)


def _span(raw: str, what: str):
    try:
        lo, hi = (float(x) for x in raw.split(":"))
    except ValueError:
        raise UsageError(f"{what} must look like LO:HI with numbers, got {raw!r}") from None
    if hi < lo:
        raise UsageError(f"empty {what}: {raw!r}")
    return lo, hi


def _axis(lo: float, hi: float, count: int) -> List[float]:
    if count < 1:
        raise UsageError("grid steps must be >= 1")
    return [lo] if count == 1 else [float(x) for x in np.linspace(lo, hi, count)]


def cmd_sweep(args) -> int:
    """K x ks_max heat map.  Every cell uses the same base seed and scores the FINAL thresholded
    state of each replica (cli.py:310-322), not the best-of harvest."""
    inst = _load(args)
    if inst.kind == "maxcut" and args.reference is None:
        raise UsageError("sweep over maxcut requires --reference for the accuracy axis")
    k_lo, k_hi = _span(args.k_range, "--k-range")
    s_lo, s_hi = _span(args.ks_range, "--ks-range")
    try:
        n_k, n_s = (int(x) for x in args.grid.lower().split("x"))
    except ValueError:
        raise UsageError(f"--grid must look like RxC with integers, got {args.grid!r}") from None
    resolve_workers(args.workers)
    J = inst.coupling()
    # all cells are independent replicas of one graph: they run as ONE batched workload -- concurrently on the GPU and,
    # under a torch.distributed launch (WORLD_SIZE > 1), sharded over the ranks (sweep.py); rank 0 writes the table
    from . import sweep as sw
    over = {k: getattr(args, k) for k in TUNABLES if getattr(args, k, None) is not None}
    labels, cells = sw.grid_cells(inst.graph.node_count, inst.n_states, args.seed, _axis(k_lo, k_hi, n_k), _axis(s_lo, s_hi, n_s), over)
    group = _maybe_init_process_group()
    try:
        objs = sw.run_cells_sharded(J, cells, inst.kind, args.replicas, **_gpu_kwargs(args))
    finally:
        if group:
            import torch.distributed as dist
            dist.destroy_process_group()
    if objs is None:
        return EXIT_OK                                # not rank 0
    lines = [SWEEP_HEADER]
    m = inst.graph.edge_count
    for (K, ks_max), obj in zip(labels, objs):
        scores = 100.0 * obj / args.reference if inst.kind == "maxcut" else 100.0 * ((1.0 - obj / m) if m else np.ones_like(obj))
        lines.append(f"{K!r},{ks_max!r},{float(np.mean(scores))!r}")
    _emit("\n".join(lines) + "\n", args.out)
    return EXIT_OK


def _maybe_init_process_group() -> bool:
    """Under torchrun (WORLD_SIZE > 1) join the default process group -- NCCL with GPUs, gloo otherwise (or when
    OSCB_BENCH_BACKEND says so).  Returns True when this call created it."""
    if int(os.environ.get("WORLD_SIZE", "1")) <= 1:
        return False
    import torch
    import torch.distributed as dist
    if dist.is_initialized():
        return False
    backend = os.environ.get("OSCB_BENCH_BACKEND", "nccl" if torch.cuda.is_available() else "gloo")
    dist.init_process_group(backend)
    return True


def cmd_scaling(args) -> int:
    """Wall time of dense random +-1 instances at a fixed step count (cli.py:327-360)."""
    try:
        sizes = [int(x) for x in args.sizes.split(",") if x.strip()]
    except ValueError:
        raise UsageError(f"--sizes must be a comma list of integers, got {args.sizes!r}") from None
    if not sizes or min(sizes) < 2:
        raise UsageError("--sizes needs integers >= 2")
    if args.steps < 1:
        raise UsageError("--steps must be >= 1")
    multi = resolve_workers(args.workers)
    h = 0.01
    lines = [SCALING_HEADER]
    for n in sizes:
        iu, iv = np.triu_indices(n, 1)
        w = np.random.default_rng(n).choice([-1.0, 1.0], size=len(iu))
        J = build_maxcut_coupling(Graph(n, iu.astype(np.int64), iv.astype(np.int64), w))
        params = SolverParams.tuned_for(n, seed=args.seed, h=h, t_stop=(args.steps - 0.5) * h,
                                        ks_period=max(args.steps * h / 2, 2 * h))
        for workers in dict.fromkeys([1, multi]):
            res = run_replicas(J, params, "maxcut", replicas=1, workers=workers, **_gpu_kwargs(args))
            lines.append(f"{n},{workers},{res.wall_time!r}")
            print(f"scaling: n={n} workers={workers} steps={res.steps_executed} wall={res.wall_time:.3f}s", file=sys.stderr)
    _emit("\n".join(lines) + "\n", args.out)
    return EXIT_OK


# ---------------------------------------------------------------------------------------------
def _solver_flags(p, replicas_default=1, workers_default=1, with_k=True):
    if with_k:
        p.add_argument("--K", type=float, default=None, help="global coupling strength")
        p.add_argument("--ks-max", type=float, default=None, help="peak locking strength")
    p.add_argument("--ks-period", type=float, default=None, help="anneal cycle length (simulated time)")
    p.add_argument("--kn", type=float, default=None, help="noise strength")
    p.add_argument("--h", type=float, default=None, help="Euler time step")
    p.add_argument("--t-stop", type=float, default=None, help="total simulated time")
    p.add_argument("--seed", type=int, default=0, help="base RNG seed")
    p.add_argument("--replicas", type=int, default=replicas_default, help="independent restarts, best kept")
    p.add_argument("--batch-size", type=int, default=None, help="accepted for compatibility (no effect on the GPU)")
    p.add_argument("--workers", type=int, default=workers_default, help="accepted for compatibility (no effect on the GPU)")
    _gpu_flags(p)


def _gpu_flags(p):
    p.add_argument("--precision", choices=("f32", "f64"), default=None, help="f32 throughput mode (default) or f64 parity mode")
    p.add_argument("--device", type=int, default=None, help="CUDA device index")
    p.add_argument("--kernel", choices=("auto", "stream", "resident", "lowdeg", "cluster", "dense-tc"), default="auto")


def build_parser() -> argparse.ArgumentParser:
    parser = _ArgParser(prog="oscim-b200", description=__doc__)
    sub = parser.add_subparsers(dest="command", required=True)

    ps = sub.add_parser("solve", help="solve one instance, print a JSON report")
    ps.add_argument("path", help="instance file (GSET layout, or DIMACS .col)")
    ps.add_argument("--problem", choices=("maxcut", "coloring"), default="maxcut")
    ps.add_argument("--colors", type=int, default=None, help="number of colors (coloring only)")
    _solver_flags(ps)
    ps.add_argument("--reference", type=float, default=None, help="best-known objective for accuracy")
    ps.add_argument("--trace", default=None, metavar="PATH", help="write energy trace CSV")
    ps.add_argument("--out", default=None, metavar="PATH", help="write the report here instead of stdout")
    ps.set_defaults(func=cmd_solve)

    pb = sub.add_parser("bench", help="run a manifest of instances, emit a CSV/JSON table")
    pb.add_argument("manifest", help="CSV manifest: path,kind,reference[,colors,replicas,seed,...]")
    _solver_flags(pb)
    pb.add_argument("--json", action="store_true", help="emit JSON instead of CSV")
    pb.add_argument("--out", default=None, metavar="PATH")
    pb.set_defaults(func=cmd_bench)

    pw = sub.add_parser("sweep", help="grid sweep over K and ks_max, emit accuracy heat-map CSV")
    pw.add_argument("path")
    pw.add_argument("--problem", choices=("maxcut", "coloring"), default="maxcut")
    pw.add_argument("--colors", type=int, default=None)
    pw.add_argument("--k-range", required=True, metavar="LO:HI")
    pw.add_argument("--ks-range", required=True, metavar="LO:HI")
    pw.add_argument("--grid", default="5x5", metavar="RxC")
    _solver_flags(pw, replicas_default=8, with_k=False)
    pw.add_argument("--reference", type=float, default=None)
    pw.add_argument("--out", default=None, metavar="PATH")
    pw.set_defaults(func=cmd_sweep)

    pc = sub.add_parser("scaling", help="time dense random instances at a fixed step count")
    pc.add_argument("--sizes", required=True, help="comma list of node counts")
    pc.add_argument("--steps", type=int, default=60, help="integration steps per run")
    pc.add_argument("--seed", type=int, default=0)
    pc.add_argument("--workers", type=int, default=4, help="accepted for compatibility")
    pc.add_argument("--out", default=None, metavar="PATH")
    _gpu_flags(pc)
    pc.set_defaults(func=cmd_scaling)
    return parser


def main(argv: Optional[List[str]] = None) -> int:
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as exc:          # _ArgParser.error or --help
        return int(exc.code or 0)
    try:
        return args.func(args)
    except UsageError as exc:
        print(f"oscim-b200: error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except NumericalError as exc:
        print(f"oscim-b200: numerical failure: {exc}", file=sys.stderr)
        return EXIT_NUMERIC
    except ParseError as exc:
        print(f"oscim-b200: input error: {exc}", file=sys.stderr)
        return EXIT_INPUT
    except ValueError as exc:          # invalid parameter combinations
        print(f"oscim-b200: error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except OSError as exc:
        print(f"oscim-b200: input error: {exc}", file=sys.stderr)
        return EXIT_INPUT


if __name__ == "__main__":
    sys.exit(main())
