"""Per-step time of ONE rank's kernel of a row-sharded SK run, measured alone on one GPU: the rank's row shard of J is
uploaded and its persistent kernel runs as a world-of-one session, so it integrates its own rows against a B image whose
other rows never move.  Everything a rank does per Euler step is there (its J stream, MMAs, epilogue, grid barrier, split-K
exchange) except the NVLink pushes and the peers' arrivals.

    python tools/dense_rank_emulation.py [n] [steps]      -> one JSON line per (world, OSCB_UMMA_SPLITK) setting
"""
import json
import os
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_2505_22631_b200 as pkg
from paper_2505_22631_b200 import dense_fused, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 512
J8 = workloads.sk_dense(n)
params = pkg.SolverParams.tuned_for(n, 2, seed=0)
for world in (8, 4, 2, 1):
    rows = n // world
    Jr = J8[:rows].astype(np.float64)
    for splitk in ("1", None) + ((("2",) if world == 2 else ())):
        if splitk is None:
            os.environ.pop("OSCB_UMMA_SPLITK", None)
        else:
            os.environ["OSCB_UMMA_SPLITK"] = splitk
        rk = dense_fused.FusedDenseRank(Jr, n, 0, rows, 0, params, 1, n * (n - 1) // 2, 1, 0, steps=steps)
        try:
            rk.connect([rk.export()])
            best = None
            for _ in range(3):
                rk.prepare([0])
                rk.launch()
                b = rk.finish()
                best = b.device_ms if best is None else min(best, b.device_ms)
            print(json.dumps({"n": n, "emulated_world": world, "rows": rows, "row_tiles": rows // 128, "ctas": rk.ctas, "splits": rk.splits,
                              "us_per_step": 1e3 * best / (steps + 1), "steps": steps,
                              "updates_per_s_if_all_ranks_ran_at_this_pace": n * (n - 1) * (steps + 1) / (best * 1e-3)}), flush=True)
        finally:
            rk.close()
