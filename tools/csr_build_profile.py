"""One device CSR build per row regime, for `ncu -k regex:k_csr` (see profiles/README.md): G(10^6, 4x10^6) (warp-ranked rows)
and the complete graph on 4096 oscillators (column-bitmap rows)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_22631_b200 import model                  # noqa: E402

rng = np.random.default_rng(1)
n, m = 1_000_000, 4_000_000
i = rng.integers(0, n, size=m)
j = (i + 1 + rng.integers(0, n - 1, size=m)) % n
_, first = np.unique(np.minimum(i, j) * n + np.maximum(i, j), return_index=True)
first = rng.permutation(first)
model._device_csr(n, i[first], j[first], np.ones(first.size))
iu, ju = np.triu_indices(4096, 1)
order = rng.permutation(iu.size)
model._device_csr(4096, iu[order].astype(np.int64), ju[order].astype(np.int64), np.ones(iu.size))
