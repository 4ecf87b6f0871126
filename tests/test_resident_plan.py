"""Host logic of the persistent kernel's graph compiler (no GPU): the sliced-ELL stream must
present every CSR row exactly once, with exactly its neighbours (CSR order), a warp-uniform
group count per row position, and balanced slots.  The walk below is the kernel's own loop
nest (oscb_resident.cuh pass A) done in Python."""
import ctypes as C

import numpy as np
import pytest

from conftest import random_graph_arrays


@pytest.fixture(scope="module")
def nat():
    from paper_2505_22631_b200 import _native
    _native.build()
    return _native


def compile_plan(nat, J, RT, max_threads=1024):
    W, T, GR = C.c_int32(), C.c_int32(), C.c_int64()
    ip = np.ascontiguousarray(J.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(J.indices, dtype=np.int64)
    rc = nat.lib().oscb_resident_plan_host(J.n, nat.ptr(ip), nat.ptr(ix), RT, max_threads, C.byref(W), C.byref(T),
                                           C.byref(GR), None, None, None, None)
    assert rc == 0, nat.last_error()
    Cs = 32 // RT
    warp_start = np.zeros(W.value, np.int32)
    quad_of = np.zeros(W.value * T.value * Cs, np.int32)
    ginfo = np.zeros(W.value * T.value, np.uint32)
    ids = np.zeros(4 * GR.value * Cs, np.uint16)
    rc = nat.lib().oscb_resident_plan_host(J.n, nat.ptr(ip), nat.ptr(ix), RT, max_threads, C.byref(W), C.byref(T),
                                           C.byref(GR), nat.ptr(warp_start), nat.ptr(quad_of), nat.ptr(ginfo), nat.ptr(ids))
    assert rc == 0, nat.last_error()
    return W.value, T.value, GR.value, warp_start, quad_of, ginfo, ids.reshape(GR.value, Cs, 4)


def walk(J, RT, plan):
    """Replay pass A's loop nest; returns {row: [neighbour ids in visiting order]} and slot loads."""
    W, T, GR, warp_start, quad_of, ginfo, ids = plan
    Cs, n = 32 // RT, J.n
    seen, loads = {}, np.zeros((W, Cs), dtype=np.int64)
    for w in range(W):
        gp = int(warp_start[w])
        for t in range(T):
            g4 = int(ginfo[w * T + t])
            for kk in range(4):
                G = (g4 >> (8 * kk)) & 0xFF
                for c in range(Cs):
                    qw = int(quad_of[(w * T + t) * Cs + c])
                    if qw < 0:
                        assert np.all(ids[gp:gp + G, c] == n)      # an empty slot only sees padding
                        continue
                    quad, order = qw & 0xFFFFF, (qw >> 20) & 0xFF
                    i = 4 * quad + ((order >> (2 * kk)) & 3)
                    got = ids[gp:gp + G, c].reshape(-1)
                    if i >= n:
                        assert np.all(got == n)
                        continue
                    assert i not in seen, f"row {i} visited twice"
                    real = got[got != n]
                    assert np.all(got[len(real):] == n), "padding must trail the real neighbours"
                    seen[i] = real.astype(np.int64)
                    loads[w, c] += G
                gp += G
        end = int(warp_start[w + 1]) if w + 1 < W else GR
        assert gp == end
    return seen, loads


@pytest.mark.parametrize("n,density,RT", [(203, 0.05, 8), (203, 0.05, 1), (64, 0.5, 32), (1, 0.0, 1), (5, 1.0, 4),
                                          (2000, 0.01, 8), (2000, 0.01, 16), (801, 0.06, 2)])
def test_stream_covers_csr_exactly(nat, n, density, RT):
    import paper_2505_22631_b200 as pkg
    iu, iv, w = random_graph_arrays(n, density, seed=n + RT)
    J = pkg.CouplingMatrix.from_edges(n, (iu, iv, w))
    plan = compile_plan(nat, J, RT)
    seen, loads = walk(J, RT, plan)
    assert sorted(seen) == list(range(n))
    for i in range(n):
        assert np.array_equal(seen[i], J.indices[J.indptr[i]:J.indptr[i + 1]]), f"row {i}"
    W, T, GR = plan[:3]
    assert W * 32 <= 1024 and W >= 1 and T >= 1
    assert W * (32 // RT) * T * 4 >= n


def test_g22_shape_padding_and_balance(nat):
    """The headline shape: padding stays small and slot loads are balanced."""
    import paper_2505_22631_b200 as pkg
    from paper_2505_22631_b200 import workloads
    n, (u, v, w), _, _ = workloads.shape_graph("G22")
    J = pkg.CouplingMatrix.from_edges(n, (u, v, w))
    plan = compile_plan(nat, J, 8)
    seen, loads = walk(J, 8, plan)
    W, T, GR = plan[:3]
    entries = GR * 4 * 4
    fill = J.nnz / entries
    assert fill > 0.80, fill
    per_warp = loads.max(axis=1)
    assert per_warp.max() / per_warp.mean() < 1.10


def test_plan_argument_errors(nat):
    ip = np.zeros(3, np.int64)
    W, T, GR = C.c_int32(), C.c_int32(), C.c_int64()
    for RT in (0, 3, 64):
        rc = nat.lib().oscb_resident_plan_host(2, nat.ptr(ip), None, RT, 1024, C.byref(W), C.byref(T), C.byref(GR),
                                               None, None, None, None)
        assert rc == nat.EINVAL
