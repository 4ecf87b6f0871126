"""bench.py's launcher: `python bench.py --gpus N` without torchrun must become N ranks (one process per GPU,
rendezvous on 127.0.0.1) and report n_gpus = N.  OSCB_BENCH_DRYRUN=1 stops after the rendezvous, so this runs on CPU."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _run(args, extra_env=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["OSCB_BENCH_DRYRUN"] = "1"
    env.update(extra_env or {})
    out = subprocess.run([sys.executable, str(ROOT / "bench.py")] + args, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout          # rank 0 alone prints
    return json.loads(lines[0])


def test_gpus_flag_self_launches_that_many_ranks():
    line = _run(["--gpus", "2"])
    assert line["n_gpus"] == 2 and line["ranks_seen"] == 2 and line["gpus_arg"] == 2


def test_single_gpu_default_does_not_spawn():
    line = _run([])
    assert line["n_gpus"] == 1 and line["ranks_seen"] == 1


def test_under_torchrun_world_size_wins():
    """The driver's N>1 form: torchrun sets WORLD_SIZE; bench.py must not spawn again."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["OSCB_BENCH_DRYRUN"] = "1"
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
                          "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), "--gpus", "2"],
                         env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["ranks_seen"] == 2
