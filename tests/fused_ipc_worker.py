"""Worker of tests/test_dense_fused_ipc.py: world_size processes, ALL on cuda:0, run one fused
row-sharded dense integration; the exchange blocks are mapped across processes with CUDA IPC."""
import os
import pickle
import sys

import numpy as np


def sk_graph(n, seed):
    rng = np.random.default_rng(seed)
    U = np.triu(rng.choice(np.array([-1.0, 1.0]), size=(n, n)), 1)
    return U + U.T


def main():
    rank, world, port, outdir = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import paper_2505_22631_b200 as pkg
    from paper_2505_22631_b200 import dense_fused
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    n, steps = 512, int(os.environ.get("FUSED_IPC_STEPS", "24"))
    J = sk_graph(n, 5)
    rows = n // world
    params = pkg.SolverParams(K=0.02, ks_max=1.0, ks_period=0.5, kn=0.2, h=0.01, t_stop=1.2, seed=40)
    seeds = [40, 41]
    got = dense_fused.run_dense_fused(J[rank * rows:(rank + 1) * rows], n, rank * rows, (rank + 1) * rows, params, seeds,
                                      device=0, pair_count=n * (n - 1) // 2, steps=steps)
    with open(os.path.join(outdir, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump(got, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
