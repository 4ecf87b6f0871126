"""Device-side CSR build (`oscb_csr_from_edges`, csrc/oscb_csr_build.cu) against the host build of
CouplingMatrix.from_edges, which the reference's own test_model.py pins (reference model.py:151-200).

Integer / index work: the bar is bit-exact -- indptr, indices and data `array_equal`, the reference's ValueErrors with the
reference's messages in the reference's order.  Every row-length regime of the kernels is hit: rows of <= 32 entries (a warp
per row), longer rows ranked by counting, rows placed through the column bitmap, n beyond the bitmap's shared memory."""
import numpy as np
import pytest

import paper_2505_22631_b200 as pkg
from paper_2505_22631_b200 import model


def _random_pairs(n, m, rng, weights=None):
    """m distinct unordered pairs of [0, n), in random order and random orientation."""
    keys = set()
    while len(keys) < m:
        a = rng.integers(0, n, size=2 * (m - len(keys)) + 8)
        b = rng.integers(0, n, size=a.size)
        for p, q in zip(a.tolist(), b.tolist()):
            if p != q and len(keys) < m:
                keys.add((min(p, q), max(p, q)))
    lo, hi = np.array(sorted(keys), dtype=np.int64).T
    order = rng.permutation(m)
    lo, hi = lo[order], hi[order]
    flip = rng.random(m) < 0.5
    i, j = np.where(flip, hi, lo), np.where(flip, lo, hi)
    x = rng.standard_normal(m) if weights is None else rng.choice(np.asarray(weights, dtype=np.float64), size=m)
    return i, j, x


def _same(n, entries, storage=None):
    host = pkg.CouplingMatrix.from_edges(n, entries, storage=storage, build="host")
    dev = pkg.CouplingMatrix.from_edges(n, entries, storage=storage, build="device")
    assert dev.n == host.n and dev.storage_kind == host.storage_kind
    assert np.array_equal(dev.indptr, host.indptr)
    assert np.array_equal(dev.indices, host.indices)
    assert np.array_equal(dev.data.view(np.uint64), host.data.view(np.uint64))        # bit for bit, NaN payloads and -0.0 included
    if host.storage_kind == "dense":
        assert np.array_equal(dev.to_dense().view(np.uint64), host.to_dense().view(np.uint64))
    return dev


@pytest.mark.gpu
@pytest.mark.parametrize("n,m", [(1, 0), (2, 1), (5, 0), (64, 200), (2000, 19990), (20000, 40000), (300, 20000)])
def test_random_graphs_bit_exact(n, m):
    rng = np.random.default_rng(n * 7919 + m)
    _same(n, _random_pairs(n, m, rng) if m else (np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0)))


@pytest.mark.gpu
def test_every_row_regime():
    rng = np.random.default_rng(5)
    # a star (one row of n - 1 entries: the bitmap), a few hubs of 33..400 entries (rank by counting), a sparse rest (warps)
    n = 6000
    pairs = {(0, k) for k in range(1, n)}
    for hub, deg in ((10, 33), (11, 64), (12, 150), (13, 400), (14, 32), (15, 31)):
        for k in rng.choice(np.arange(100, n), size=deg, replace=False).tolist():
            pairs.add((hub, k))
    a, b, _ = _random_pairs(n, 9000, rng)
    pairs.update((min(p, q), max(p, q)) for p, q in zip(a.tolist(), b.tolist()))
    lo, hi = np.array(sorted(pairs), dtype=np.int64).T
    order = rng.permutation(lo.size)
    J = _same(n, (hi[order], lo[order], rng.standard_normal(lo.size)))
    deg = np.diff(J.indptr)
    assert deg[0] == n - 1 and deg.max() == n - 1 and (deg <= 32).sum() > n // 2


@pytest.mark.gpu
def test_complete_graph_and_dense_storage():
    n = 700
    iu, ju = np.triu_indices(n, 1)
    rng = np.random.default_rng(2)
    order = rng.permutation(iu.size)
    J = _same(n, (iu[order].astype(np.int64), ju[order].astype(np.int64), rng.choice([-1.0, 1.0], size=iu.size)))
    assert J.storage_kind == "dense" and J.nnz == n * (n - 1)


@pytest.mark.gpu
def test_n_beyond_the_bitmap():
    # 2.5 M oscillators: the column bitmap no longer fits in shared memory, the long row ranks by counting
    n = 2_500_000
    rng = np.random.default_rng(9)
    hub = np.unique(rng.integers(1, n, size=3000))
    chain = np.arange(1, n - 1, 7, dtype=np.int64)
    i = np.concatenate([np.zeros(hub.size, np.int64), chain + 1])
    j = np.concatenate([hub, chain])
    _same(n, (i, j, rng.standard_normal(i.size)))


@pytest.mark.gpu
def test_zero_valued_entries_are_dropped_after_validation():
    rng = np.random.default_rng(3)
    i, j, x = _random_pairs(500, 6000, rng, weights=(0.0, 1.0, -2.0, -0.0))
    J = _same(500, (i, j, x))
    assert J.nnz == 2 * int(np.count_nonzero(x))
    x[:] = 0.0
    assert _same(500, (i, j, x)).nnz == 0
    # a pair listed twice is an error even when one of the two entries is zero (the reference validates before it filters)
    i2, j2, x2 = np.append(i, j[17]), np.append(j, i[17]), np.append(x, 1.0)
    for build in ("host", "device"):
        with pytest.raises(ValueError, match="duplicate coupling entry on an unordered pair"):
            pkg.CouplingMatrix.from_edges(500, (i2, j2, x2), build=build)


@pytest.mark.gpu
def test_non_finite_values_travel():
    i = np.array([0, 1, 2], dtype=np.int64)
    j = np.array([1, 2, 3], dtype=np.int64)
    _same(4, (i, j, np.array([np.nan, np.inf, -np.inf])))


@pytest.mark.gpu
def test_errors_in_the_reference_order():
    def both(n, i, j, x, msg):
        for build in ("host", "device"):
            with pytest.raises(ValueError) as err:
                pkg.CouplingMatrix.from_edges(n, (np.array(i, np.int64), np.array(j, np.int64), np.array(x, np.float64)), build=build)
            assert str(err.value) == msg, build

    both(4, [0, 4], [1, 2], [1.0, 1.0], "coupling index out of range")
    both(4, [0, -1], [1, 2], [1.0, 1.0], "coupling index out of range")
    both(4, [0, 2], [1, 2], [1.0, 1.0], "diagonal entries must be zero (no self-coupling)")
    both(4, [0, 1], [1, 0], [1.0, 2.0], "duplicate coupling entry on an unordered pair")
    # precedence: range before diagonal before duplicate
    both(4, [0, 0, 3, 9], [1, 1, 3, 0], [1.0] * 4, "coupling index out of range")
    both(4, [0, 0, 3], [1, 1, 3], [1.0] * 3, "diagonal entries must be zero (no self-coupling)")
    # duplicates in a long row (the bitmap and the counting path) and in a short one
    n = 3000
    star_i, star_j = np.zeros(n - 1, np.int64), np.arange(1, n, dtype=np.int64)
    both(n, np.append(star_i, 5), np.append(star_j, 0), np.ones(n), "duplicate coupling entry on an unordered pair")
    both(n, np.append(star_i[:100], 5), np.append(star_j[:100], 0), np.ones(101), "duplicate coupling entry on an unordered pair")
    both(n, np.append(star_i[:35], 5), np.append(star_j[:35], 0), np.ones(36), "duplicate coupling entry on an unordered pair")
    both(n, np.append(star_i[:9], 5), np.append(star_j[:9], 0), np.ones(10), "duplicate coupling entry on an unordered pair")
    with pytest.raises(ValueError, match="n must be >= 1"):
        pkg.CouplingMatrix.from_edges(0, [], build="device")


@pytest.mark.gpu
def test_a_device_built_graph_solves_like_a_host_built_one():
    rng = np.random.default_rng(11)
    i, j, x = _random_pairs(256, 1500, rng, weights=(1.0, -1.0))
    params = pkg.SolverParams(K=0.3, ks_max=1.0, ks_period=2.0, kn=0.05, h=0.01, t_stop=2.0, seed=4)
    runs = [pkg.run_batch(pkg.CouplingMatrix.from_edges(256, (i, j, x), build=b), params, "maxcut", [1, 2, 3], precision="f64")
            for b in ("host", "device")]
    assert np.array_equal(runs[0].final_phases, runs[1].final_phases)
    assert np.array_equal(runs[0].best_objective, runs[1].best_objective)


@pytest.mark.gpu
def test_large_graph_and_auto_route(monkeypatch):
    # 2 M edges on 10^6 oscillators: past the auto threshold, so the default route is the device build
    n, m = 1_000_000, 2_000_000
    rng = np.random.default_rng(1)
    i = rng.integers(0, n, size=m)
    j = (i + 1 + rng.integers(0, n - 1, size=m)) % n
    keys = np.minimum(i, j) * n + np.maximum(i, j)
    _, first = np.unique(keys, return_index=True)
    i, j = i[first], j[first]
    x = rng.choice([-1.0, 1.0], size=i.size)
    assert i.size >= model.CSR_DEVICE_MIN_ENTRIES and model._csr_build_on_device(None, i.size)
    timing = {}
    indptr, cols, vals = model._device_csr(n, i, j, x, timing=timing)
    host = pkg.CouplingMatrix.from_edges(n, (i, j, x), build="host")
    assert np.array_equal(indptr, host.indptr) and np.array_equal(cols, host.indices) and np.array_equal(vals, host.data)
    assert timing["device_ms"] > 0.0
    monkeypatch.setenv(model.CSR_BUILD_ENV_VAR, "host")
    assert not model._csr_build_on_device(None, i.size)


def test_build_argument_is_validated():
    with pytest.raises(ValueError, match="build must be"):
        pkg.CouplingMatrix.from_edges(3, [(0, 1, 1.0)], build="gpu")
    # small lists stay on the host in auto mode: no device, no library call
    assert not model._csr_build_on_device(None, 10)
    J = pkg.CouplingMatrix.from_edges(3, [(0, 1, 1.0), (1, 2, -1.0)])
    assert J.nnz == 4


def test_device_build_fails_loudly_without_a_gpu():
    # explicit build="device" never falls back to the host build (no CPU path behind the C ABI)
    from paper_2505_22631_b200 import _native
    if _native.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(RuntimeError, match="oscb_csr_from_edges"):
        pkg.CouplingMatrix.from_edges(3, [(0, 1, 1.0), (1, 2, -1.0)], build="device")
