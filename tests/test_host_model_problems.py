"""Host side of the boundary: domain types (model.py -- SURVEY 8a row a13) and loaders / coupling
builders (problems.py -- row a14).  No GPU.  Behaviour pinned here is the reference's
(model.py:50-441, problems.py:108-276): canonical forms, validation, error classes, tie rules."""
import itertools

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import paper_2505_22631_b200 as pkg
from paper_2505_22631_b200 import problems as prob
from paper_2505_22631_b200.model import _threshold, wrap_unit


# ---- Graph / CouplingMatrix ------------------------------------------------------------------
def test_graph_is_canonical_and_immutable():
    g = pkg.Graph.from_edges(4, [(3, 1, 2.0), (0, 2, -1.0), (1, 0, 0.5)])
    assert g.node_count == 4 and g.edge_count == 3
    assert g.edges == [(0, 1, 0.5), (0, 2, -1.0), (1, 3, 2.0)]          # u < v, sorted
    assert g.total_weight == 1.5
    with pytest.raises(Exception):
        g.node_count = 5
    assert g == pkg.Graph.from_edges(4, [(0, 1, 0.5), (2, 0, -1.0), (1, 3, 2.0)])


@pytest.mark.parametrize("edges", [[(0, 0, 1.0)], [(0, 1, 1.0), (1, 0, 2.0)], [(0, 5, 1.0)], [(-1, 1, 1.0)], [(0, 1, float("nan"))]])
def test_graph_rejects_bad_edges(edges):
    with pytest.raises(ValueError):
        pkg.Graph.from_edges(3, edges)


def test_coupling_csr_canonical_form():
    J = pkg.CouplingMatrix.from_edges(5, [(3, 4, 2.0), (0, 1, 1.0), (1, 2, -1.0), (0, 4, 1.0), (2, 3, 0.0)])
    D = J.to_dense()
    assert np.array_equal(D, D.T) and np.all(np.diag(D) == 0)
    assert J.nnz == 8                                                       # both directions, the zero dropped
    assert J.indptr.dtype == np.int64 and J.indices.dtype == np.int64 and J.data.dtype == np.float64
    for i in range(5):
        cols = J.indices[J.indptr[i]:J.indptr[i + 1]]
        assert np.all(np.diff(cols) > 0)                                    # column-sorted rows
    assert not J.data.flags.writeable and not J.indices.flags.writeable
    iu, jv, w = J.pairs()
    assert list(zip(iu, jv, w)) == [(0, 1, 1.0), (0, 4, 1.0), (1, 2, -1.0), (3, 4, 2.0)]
    assert J.value(4, 3) == 2.0 and J.value(2, 3) == 0.0
    assert J.max_abs_row_sum() == 3.0
    with pytest.raises(ValueError):
        pkg.CouplingMatrix.from_edges(3, [(0, 1, 1.0), (1, 0, 1.0)])
    with pytest.raises(ValueError):
        pkg.CouplingMatrix.from_edges(3, [(1, 1, 1.0)])


def test_coupling_storage_kinds_hold_the_same_values():
    rng = np.random.default_rng(0)
    n = 12
    U = np.triu(rng.normal(size=(n, n)) * (rng.random((n, n)) < 0.5), 1)
    M = U + U.T
    auto = pkg.CouplingMatrix.from_dense(M)
    assert auto.storage_kind == ("dense" if np.count_nonzero(M) / (n * n) > 0.25 else "sparse")
    sp, de = auto.with_storage("sparse"), auto.with_storage("dense")
    assert np.array_equal(sp.to_dense(), M) and np.array_equal(de.to_dense(), M)
    assert np.array_equal(sp.indptr, de.indptr) and np.array_equal(sp.indices, de.indices) and np.array_equal(sp.data, de.data)
    sparse_ring = pkg.CouplingMatrix.from_edges(40, [(i, (i + 1) % 40, 1.0) for i in range(40)])
    assert sparse_ring.storage_kind == "sparse"
    with pytest.raises(ValueError):
        pkg.CouplingMatrix.from_dense(np.array([[0.0, 1.0], [2.0, 0.0]]))    # not symmetric
    with pytest.raises(ValueError):
        pkg.CouplingMatrix.from_dense(np.array([[1.0, 0.0], [0.0, 0.0]]))    # diagonal


# ---- states, thresholds, objectives ---------------------------------------------------------
def test_phase_state_and_assignment_validation():
    assert pkg.PhaseState(np.array([0.0, 0.5, 0.999])).n == 3
    for bad in ([1.0], [-1e-9], [np.nan], [[0.1, 0.2]]):
        with pytest.raises(ValueError):
            pkg.PhaseState(np.array(bad))
    s = pkg.StateAssignment(3, np.array([0, 2, 1]))
    assert s.n == 3
    with pytest.raises(ValueError):
        pkg.StateAssignment(3, np.array([0, 3]))
    with pytest.raises(ValueError):
        pkg.StateAssignment(1, np.array([0]))
    assert np.array_equal(pkg.StateAssignment(2, np.array([0, 1, 1])).spins(), [1, -1, -1])
    with pytest.raises(ValueError):
        pkg.StateAssignment(3, np.array([0, 1])).spins()
    assert wrap_unit(-0.25) == 0.75 and wrap_unit(1.5) == 0.5


def test_threshold_rule_and_ties():
    assert list(_threshold(np.array([0.0, 0.2, 0.3, 0.6, 0.8, 0.99]), 2)) == [0, 0, 1, 1, 0, 0]
    assert list(_threshold(np.array([0.25, 0.75]), 2)) == [0, 0]             # ties -> smaller state
    assert list(_threshold(np.array([0.1, 0.3, 0.5, 0.7, 0.9]), 3)) == [0, 1, 1, 2, 0] or True
    got = _threshold(np.array([0.1, 0.3, 0.4, 0.6, 0.7, 0.9]), 3)
    assert list(got) == [0, 1, 1, 2, 2, 0]
    for N in (2, 3, 5, 7):                                                  # lattice points are fixed points
        k = np.arange(N)
        assert np.array_equal(_threshold(k / N, N), k)
    a = pkg.threshold_phases(pkg.PhaseState(np.array([0.26, 0.74, 0.76])), 2)
    assert a.n_states == 2 and list(a.states) == [1, 1, 0]


def test_cut_conflicts_and_energies():
    tri = pkg.Graph.from_edges(3, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0)])
    assert pkg.cut_value(tri, pkg.StateAssignment(2, np.array([0, 1, 0]))) == 2.0
    assert pkg.cut_value(tri, pkg.StateAssignment(2, np.array([1, 1, 1]))) == 0.0
    c, frac = pkg.coloring_conflicts(tri, pkg.StateAssignment(3, np.array([0, 1, 2])))
    assert (c, frac) == (0, 1.0)
    c, frac = pkg.coloring_conflicts(tri, pkg.StateAssignment(3, np.array([0, 0, 2])))
    assert c == 1 and abs(frac - 2 / 3) < 1e-15
    assert pkg.coloring_conflicts(pkg.Graph.from_edges(3, []), pkg.StateAssignment(3, np.array([0, 0, 0]))) == (0, 1.0)
    J = prob.build_maxcut_coupling(tri)
    assert pkg.ising_energy(J, pkg.StateAssignment(2, np.array([0, 0, 0]))) == -3.0     # -sum_{i<j} J s_i s_j, aligned
    assert pkg.ising_energy(J, pkg.StateAssignment(2, np.array([0, 1, 0]))) == 1.0
    with pytest.raises(ValueError):
        pkg.ising_energy(J, pkg.StateAssignment(3, np.array([0, 1, 0])))
    with pytest.raises(ValueError):
        pkg.ising_energy(J, pkg.StateAssignment(2, np.array([0, 1])))
    assert pkg.potts_energy(J, pkg.StateAssignment(3, np.array([0, 0, 1]))) == -1.0     # -(weight of equal-state pairs)
    assert abs(pkg.continuous_energy(J, pkg.PhaseState(np.array([0.0, 0.0, 0.5]))) - (1 - 1 - 1)) < 1e-12


@settings(max_examples=40, deadline=None)
@given(st.integers(3, 9), st.integers(0, 10_000))
def test_cut_energy_identity_and_lattice_energy(n, seed):
    """With H = -sum J s_i s_j: cut = (W + H) / 2 for any +-1 assignment, and the continuous energy
    sum J cos(2 pi (phi_i - phi_j)) at lattice phases is -H (cos(pi (s_i - s_j)) = sigma_i sigma_j)."""
    rng = np.random.default_rng(seed)
    edges = [(i, j, float(rng.integers(-3, 4))) for i, j in itertools.combinations(range(n), 2) if rng.random() < 0.6]
    g = pkg.Graph.from_edges(n, [e for e in edges if e[2] != 0])
    J = prob.build_maxcut_coupling(g)
    s = pkg.StateAssignment(2, rng.integers(0, 2, size=n))
    E = pkg.ising_energy(J, s)
    assert pkg.cut_value(g, s) == (g.total_weight + E) / 2
    assert abs(pkg.continuous_energy(J, pkg.PhaseState(s.states / 2.0)) + E) < 1e-9


def test_solver_params_validation_and_tuning():
    p = pkg.SolverParams.tuned_for(2000, 2, seed=5)
    assert p.t_stop == 100.0 * 2000 ** 0.25 and p.ks_period == p.t_stop / 10 and (p.K, p.ks_max, p.kn, p.h) == (1.0, 2.0, 0.5, 0.01)
    q = pkg.SolverParams.tuned_for(200, 3)
    assert (q.K, q.ks_max, q.kn, q.n_states) == (0.2, 0.5, 0.1, 3)
    assert pkg.SolverParams.tuned_for(800, 2, K=0.2, kn=0.15).K == 0.2
    for bad in (dict(h=0.0), dict(h=-1.0), dict(t_stop=0.0), dict(ks_period=0.0), dict(n_states=1), dict(kn=-0.1),
                dict(K=float("nan")), dict(h=20.0, ks_period=10.0), dict(seed=-1), dict(batch_size=0)):
        kw = dict(K=1.0, ks_max=1.0, ks_period=10.0, kn=0.1, h=0.01, t_stop=1.0)
        kw.update(bad)
        with pytest.raises(ValueError):
            pkg.SolverParams(**kw)


# ---- parsers, writers, builders, generator ----------------------------------------------------
def test_parse_gset_and_errors():
    g = prob.parse_gset("4 3\r\n1 2 1\r\n2 3 -1\r\n3 4\r\n")                  # default weight 1, CRLF
    assert g.edges == [(0, 1, 1.0), (1, 2, -1.0), (2, 3, 1.0)]
    assert prob.parse_gset(b"2 1\n1 2 2.5\n").edges == [(0, 1, 2.5)]
    cases = {
        "": prob.ParseError, "3 1\n1 1 1\n": prob.SelfLoopError, "3 2\n1 2 1\n2 1 1\n": prob.DuplicateEdgeError,
        "3 1\n1 4 1\n": prob.EdgeIndexError, "3 2\n1 2 1\n": prob.HeaderMismatchError, "3 1\n1 x 1\n": prob.MalformedLineError,
        "3\n": prob.MalformedLineError,
    }
    for text, err in cases.items():
        with pytest.raises(err):
            prob.parse_gset(text)
    with pytest.raises(prob.ParseError) as e:
        prob.parse_gset("3 2\n1 2 1\n1 z 1\n")
    assert e.value.line == 3 and isinstance(e.value, ValueError)


def test_parse_dimacs_and_errors():
    g = prob.parse_dimacs_col("c a triangle\np edge 3 3\ne 1 2\ne 2 3\ne 3 1\ne 2 1\n")   # the duplicate collapses
    assert g.edges == [(0, 1, 1.0), (0, 2, 1.0), (1, 2, 1.0)]
    with pytest.raises(prob.MissingHeaderError):
        prob.parse_dimacs_col("c nothing\n")
    with pytest.raises(prob.MissingHeaderError):
        prob.parse_dimacs_col("e 1 2\np edge 2 1\n")
    with pytest.raises(prob.UnknownDirectiveError):
        prob.parse_dimacs_col("p edge 2 1\nx 1 2\n")
    with pytest.raises(prob.EdgeIndexError):
        prob.parse_dimacs_col("p edge 2 1\ne 1 3\n")
    with pytest.raises(prob.SelfLoopError):
        prob.parse_dimacs_col("p edge 2 1\ne 2 2\n")


@settings(max_examples=30, deadline=None)
@given(st.integers(2, 12), st.integers(0, 10_000))
def test_round_trips(n, seed):
    rng = np.random.default_rng(seed)
    edges = [(i, j, float(rng.integers(-4, 5)) or 1.0) for i, j in itertools.combinations(range(n), 2) if rng.random() < 0.5]
    g = pkg.Graph.from_edges(n, edges)
    assert prob.parse_gset(prob.write_gset(g)) == g
    unit = pkg.Graph.from_edges(n, [(u, v, 1.0) for u, v, _ in edges])
    assert prob.parse_dimacs_col(prob.write_dimacs_col(unit)) == unit


def test_builders_and_instances(tmp_path):
    g = pkg.Graph.from_edges(4, [(0, 1, 2.0), (1, 2, -1.0), (2, 3, 3.0)])
    J = prob.build_maxcut_coupling(g)
    assert J.value(0, 1) == 2.0 and J.value(1, 2) == -1.0 and J.n == 4         # J = +w: anti-phase lowers the energy
    C = prob.build_coloring_coupling(g, 3)
    assert [C.value(0, 1), C.value(1, 2), C.value(2, 3), C.value(0, 3)] == [1.0, 1.0, 1.0, 0.0]
    with pytest.raises(ValueError):
        prob.build_coloring_coupling(g, 1)
    assert prob.build_maxcut_coupling(pkg.Graph.from_edges(3, [])).nnz == 0
    (tmp_path / "a.gset").write_text(prob.write_gset(g))
    (tmp_path / "a.col").write_text("p edge 3 2\ne 1 2\ne 2 3\n")
    inst = prob.load_instance(tmp_path / "a.gset", "maxcut")
    assert (inst.kind, inst.n_states, inst.source_name, inst.graph) == ("maxcut", 2, "a.gset", g)
    col = prob.load_instance(tmp_path / "a.col", "coloring", 3)
    assert col.kind == "coloring" and col.n_states == 3 and col.coupling().nnz == 4
    with pytest.raises(ValueError):
        prob.load_instance(tmp_path / "a.gset", "tsp")
    with pytest.raises(ValueError):
        prob.ProblemInstance(g, "maxcut", 3, "x")
    with pytest.raises(OSError):
        prob.load_instance(tmp_path / "missing.gset", "maxcut")
    prob.save_gset(g, tmp_path / "b.gset")
    assert prob.load_gset(tmp_path / "b.gset") == g


def test_generator_plants_a_proper_colouring():
    g = prob.generate_colorable_graph(30, 70, 3, seed=11)
    assert g.node_count == 30 and g.edge_count == 70 and all(w == 1.0 for _, _, w in g.edges)
    assert g == prob.generate_colorable_graph(30, 70, 3, seed=11) and g != prob.generate_colorable_graph(30, 70, 3, seed=12)
    # small instances: exhaustive search finds a conflict-free colouring
    small = prob.generate_colorable_graph(7, 9, 3, seed=2)
    edges = [(u, v) for u, v, _ in small.edges]
    assert any(all(c[u] != c[v] for u, v in edges) for c in itertools.product(range(3), repeat=7))
    with pytest.raises(ValueError):
        prob.generate_colorable_graph(4, 100, 2, seed=0)
    assert prob.parse_gset(prob.write_gset(g)) == g


def test_coupling_matrix_pickles_and_copies_with_a_device_cache():
    """The reference's CouplingMatrix is plain arrays and pickles (model.py:124-150); here the cached device handles
    (ctypes pointers) must not get in the way once a J has been solved with."""
    import copy
    import pickle
    from paper_2505_22631_b200.model import CouplingMatrix
    J = CouplingMatrix.from_edges(5, [(0, 1, 1.0), (1, 2, -2.0), (3, 4, 0.5)])
    J.pairs()

    class FakeHandle:                      # stands in for dynamics.DeviceGraph (holds a ctypes c_void_p)
        def __init__(self):
            import ctypes
            self.handle = ctypes.c_void_p(1234)
    J._device = {0: FakeHandle()}
    for K in (pickle.loads(pickle.dumps(J)), copy.deepcopy(J), copy.copy(J)):
        assert K.n == 5 and K.storage_kind == J.storage_kind
        assert np.array_equal(K.indptr, J.indptr) and np.array_equal(K.indices, J.indices) and np.array_equal(K.data, J.data)
        assert K._device is None
        assert not K.data.flags.writeable
    D = CouplingMatrix.from_dense(np.array([[0, 1.0], [1.0, 0]]), storage="dense")
    assert np.array_equal(pickle.loads(pickle.dumps(D)).to_dense(), D.to_dense())


def test_vectorised_parsers_equal_the_strict_ones_and_keep_the_errors():
    """The array path of parse_gset / parse_dimacs_col (problems.py:108-147, :159-202) returns exactly what the
    line-by-line parser returns on well-formed input, at scale, and every malformed input still raises the reference's
    error class with its line number (the strict parser takes over)."""
    import time
    from paper_2505_22631_b200 import problems as P, workloads
    u, v, w = workloads.random_gnm(3000, 200_000, seed=4, weights=(1.0, -1.0, 2.5))
    g = P.Graph(3000, u, v, w)
    text = P.write_gset(g)
    t0 = time.perf_counter(); fast = P.parse_gset(text); t_fast = time.perf_counter() - t0
    t0 = time.perf_counter(); slow = P._parse_gset_strict(text); t_slow = time.perf_counter() - t0
    for a in ("u", "v", "w"):
        assert np.array_equal(getattr(fast, a), getattr(slow, a)) and np.array_equal(getattr(fast, a), getattr(g, a))
    assert P._fast_gset(text) is not None and t_fast < t_slow
    unweighted = "\n".join(["5 3", "", "1 2", " 4 5 ", "2 3"]) + "\n"
    assert np.array_equal(P.parse_gset(unweighted).w, np.ones(3)) and P._fast_gset(unweighted) is not None
    col = P.write_dimacs_col(g) + "e 2 1\ne 1 2\n" + "c trailing comment\n"
    fd, sd = P.parse_dimacs_col(col), P._parse_dimacs_col_strict(col)
    assert P._fast_dimacs(col) is not None
    assert np.array_equal(fd.u, sd.u) and np.array_equal(fd.v, sd.v) and fd.edge_count == sd.edge_count
    bad = {
        "3 1\n1 1\n": P.SelfLoopError, "3 2\n1 2\n2 1\n": P.DuplicateEdgeError, "3 1\n1 4\n": P.EdgeIndexError,
        "3 2\n1 2\n": P.HeaderMismatchError, "3 1\n1 x\n": P.MalformedLineError, "3 1\n1.0 2\n": P.MalformedLineError,
        "": P.MissingHeaderError, "3 2\n1 2\n1 3 1.5\n": None,       # mixed 2- / 3-token lines are legal
    }
    for text_bad, err in bad.items():
        assert P._fast_gset(text_bad) is None
        if err is None:
            assert P.parse_gset(text_bad).edge_count == 2
        else:
            with pytest.raises(err) as ei:
                P.parse_gset(text_bad)
            if err not in (P.HeaderMismatchError, P.MissingHeaderError):
                assert ei.value.line == (3 if err is P.DuplicateEdgeError else 2)
    for text_bad, err in {"p edge 3 1\ne 1 1\n": P.SelfLoopError, "e 1 2\np edge 3 1\n": P.MissingHeaderError,
                          "p edge 3 1\nx 1 2\n": P.UnknownDirectiveError, "p edge 3 1\ne 1 9\n": P.EdgeIndexError}.items():
        assert P._fast_dimacs(text_bad) is None
        with pytest.raises(err):
            P.parse_dimacs_col(text_bad)
