import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden" / "reference_vectors.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def oracle():
    """The CPU oracle (test infrastructure): built on demand with gcc."""
    from oracle import oracle as O
    O.build()
    O.lib()
    return O


def graph_from_golden(golden, tag):
    return golden[f"{tag}_indptr"], golden[f"{tag}_indices"], golden[f"{tag}_data"]


def coupling_from_golden(golden, tag):
    from paper_2505_22631_b200.model import CouplingMatrix
    ip, ix, d = graph_from_golden(golden, tag)
    return CouplingMatrix(len(ip) - 1, ip, ix, d, "sparse")


def params_from_row(row, **over):
    from paper_2505_22631_b200.model import SolverParams
    K, ks_max, ks_period, kn, h, t_stop, N, seed = row
    kw = dict(K=float(K), ks_max=float(ks_max), ks_period=float(ks_period), kn=float(kn), h=float(h),
              t_stop=float(t_stop), n_states=int(N), seed=int(seed))
    kw.update(over)
    return SolverParams(**kw)


def circ_dist_rad(a, b):
    d = np.abs(np.asarray(a) - np.asarray(b))
    return 2 * np.pi * np.minimum(d, 1.0 - d)


def random_graph_arrays(n, density, seed, weights=(-1.0, 1.0)):
    """Same synthetic-graph generator the reference's tests share (tests/conftest.py:22-29)."""
    rng = np.random.default_rng(seed)
    iu, iv = np.triu_indices(n, 1)
    keep = rng.random(len(iu)) < density
    iu, iv = iu[keep], iv[keep]
    w = rng.choice(weights, size=len(iu))
    return iu.astype(np.int64), iv.astype(np.int64), w
