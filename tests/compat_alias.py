"""pytest plugin (-p compat_alias): makes `import oscim` resolve to this package, so the reference's
own test modules can be run, unmodified and in place, against the GPU-backed drop-in."""
import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import paper_2505_22631_b200 as _pkg  # noqa: E402

sys.modules["oscim"] = _pkg
for _sub in ("model", "problems", "dynamics", "cli"):
    sys.modules["oscim." + _sub] = importlib.import_module("paper_2505_22631_b200." + _sub)

# The brute-force oracles (exact_maxcut / exact_min_conflicts) are test ground truth only and out of
# this build's scope: the reference's own module is loaded on top of OUR model
# types when it is there (it only imports `.model`).
_bf = Path("/root/reference/pkg/src/oscim/bruteforce.py")
if _bf.exists():
    import importlib.util
    _spec = importlib.util.spec_from_file_location("oscim.bruteforce", _bf)
    _mod = importlib.util.module_from_spec(_spec)
    sys.modules["oscim.bruteforce"] = _mod
    _spec.loader.exec_module(_mod)
