"""Device-side CSR build against the vectorised host build, on graphs of the sizes SURVEY.md 8(f4) names.

    python tools/csr_build_bench.py > gpurun_out/csr_build.jsonl

One JSON line per graph: entries per second of the kernels alone (CUDA events inside oscb_csr_from_edges), of the whole call with
its host<->device copies (pageable numpy buffers), and of CouplingMatrix.from_edges(build="host") on this box's cores; the
algorithmic bytes per edge are csrc/oscb_csr_build.cu's (count 24 + fill 24 + 32 + placement 32 + 32 = 144 B per edge)."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2505_22631_b200 as pkg                      # noqa: E402
from paper_2505_22631_b200 import model                  # noqa: E402


def gnm(n, m, seed):
    rng = np.random.default_rng(seed)
    i = rng.integers(0, n, size=m)
    j = (i + 1 + rng.integers(0, n - 1, size=m)) % n
    keys = np.minimum(i, j) * n + np.maximum(i, j)
    _, first = np.unique(keys, return_index=True)
    first = rng.permutation(first)
    return i[first], j[first], rng.choice([-1.0, 1.0], size=first.size)


def complete(n, seed):
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, 1)
    order = rng.permutation(iu.size)
    return iu[order].astype(np.int64), ju[order].astype(np.int64), rng.choice([-1.0, 1.0], size=iu.size)


CASES = [("G(10^6, 4x10^6) +-1", 1_000_000, lambda: gnm(1_000_000, 4_000_000, 1)),
         ("G(4x10^6, 1.6x10^7) +-1", 4_000_000, lambda: gnm(4_000_000, 16_000_000, 2)),
         ("custom_8000-like G(8000, 2x10^6)", 8000, lambda: gnm(8000, 2_000_000, 3)),
         ("complete SK 8192 (3.4x10^7 pairs)", 8192, lambda: complete(8192, 4))]

for name, n, make in CASES:
    i, j, x = make()
    model._device_csr(n, i[:1000], j[:1000], x[:1000])          # context, module load
    best = None
    for _ in range(3):
        timing = {}
        t0 = time.perf_counter()
        indptr, cols, vals = model._device_csr(n, i, j, x, timing=timing)
        wall = time.perf_counter() - t0
        best = (timing["device_ms"], wall) if best is None or wall < best[1] else best
    t0 = time.perf_counter()
    host = pkg.CouplingMatrix.from_edges(n, (i, j, x), storage="sparse", build="host")
    host_s = time.perf_counter() - t0
    same = bool(np.array_equal(indptr, host.indptr) and np.array_equal(cols, host.indices) and np.array_equal(vals, host.data))
    m = int(i.size)
    print(json.dumps({"graph": name, "n": n, "edges": m, "identical_to_host_build": same,
                      "device_kernels_ms": round(best[0], 3), "device_edges_per_s": m / (best[0] * 1e-3),
                      "device_algorithmic_GBps": 144.0 * m / (best[0] * 1e-3) / 1e9,
                      "call_with_copies_s": round(best[1], 4), "call_edges_per_s": m / best[1],
                      "host_numpy_s": round(host_s, 3), "host_edges_per_s": m / host_s}), flush=True)
