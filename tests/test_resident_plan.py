"""Host logic of the persistent kernel's graph compiler (no GPU): the sliced-ELL stream must
present every CSR row exactly once, with exactly its neighbours, a warp-uniform group count per
row position, balanced slots and (throughput mode) bank-conflict-free wavefronts.  The walk
below is the kernel's own loop nest (oscb_resident.cuh pass A) done in Python."""
import ctypes as C

import numpy as np
import pytest

from conftest import random_graph_arrays


@pytest.fixture(scope="module")
def nat():
    from paper_2505_22631_b200 import _native
    _native.build()
    return _native


def compile_plan(nat, J, RT, max_threads=1024, pair_bytes=8, keep_order=False, rpl=1):
    W, T, GR, BC = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64()
    ip = np.ascontiguousarray(J.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(J.indices, dtype=np.int64)
    args = (J.n, nat.ptr(ip), nat.ptr(ix), RT, rpl, max_threads, pair_bytes, int(keep_order), C.byref(W), C.byref(T),
            C.byref(GR), C.byref(BC))
    rc = nat.lib().oscb_resident_plan_host(*args, None, None, None, None)
    assert rc == 0, nat.last_error()
    Cs = 32 // (RT // rpl)
    warp_start = np.zeros(W.value, np.int32)
    rows = np.zeros(W.value * T.value * 4 * Cs, np.uint16)
    ginfo = np.zeros(W.value * T.value, np.uint32)
    ids = np.zeros(4 * (GR.value + 1) * Cs, np.uint16)
    rc = nat.lib().oscb_resident_plan_host(*args, nat.ptr(warp_start), nat.ptr(rows), nat.ptr(ginfo), nat.ptr(ids))
    assert rc == 0, nat.last_error()
    return dict(Cs=Cs, W=W.value, T=T.value, GR=GR.value, conflicts=BC.value, warp_start=warp_start,
                rows=rows.reshape(W.value, T.value, 4, Cs), ginfo=ginfo, ids=ids.reshape(GR.value + 1, Cs, 4))


def walk(J, RT, plan):
    """Replay pass A's loop nest; returns {row: neighbour ids in visiting order} and warp loads."""
    W, T, GR, ids = plan["W"], plan["T"], plan["GR"], plan["ids"]
    Cs, n = plan["Cs"], J.n
    nRT = n * RT
    seen, loads = {}, np.zeros(W, dtype=np.int64)
    for w in range(W):
        gp = int(plan["warp_start"][w])
        for t in range(T):
            g4 = int(plan["ginfo"][w * T + t])
            for kk in range(4):
                G = (g4 >> (8 * kk)) & 0xFF
                for c in range(Cs):
                    iRT = int(plan["rows"][w, t, kk, c])
                    got = ids[gp:gp + G, c].reshape(-1).astype(np.int64)
                    assert np.all(got % RT == 0) and np.all(got < (n + 16) * RT)
                    if iRT >= nRT:
                        assert np.all(got >= nRT)                  # an empty slot only sees padding
                        continue
                    i = iRT // RT
                    assert iRT % RT == 0 and i not in seen, f"row {i} visited twice"
                    seen[i] = got[got < nRT] // RT
                loads[w] += G
                gp += G
        end = int(plan["warp_start"][w + 1]) if w + 1 < W else GR
        assert gp == end
    assert np.all(ids[GR] >= nRT)                                   # the prefetch pad row
    return seen, loads


def wavefront_conflicts(RT, plan, pair_bytes):
    """Count stream positions where two slots of one shared-memory wavefront share a bank class."""
    Cs = plan["Cs"]
    H = max(1, min(Cs, (128 // pair_bytes) // RT))
    ids = plan["ids"][:plan["GR"]].astype(np.int64) // RT          # [GR, Cs, 4] row numbers (incl. padding rows)
    bad = 0
    for c0 in range(0, Cs, H):
        cls = ids[:, c0:c0 + H, :] % H                             # [GR, H, 4]
        for h in range(H):
            bad += int(((cls == h).sum(axis=1) > 1).sum())
    return bad, plan["GR"] * 4 * (Cs // H)


@pytest.mark.parametrize("keep_order", [True, False])
@pytest.mark.parametrize("n,density,RT,pair_bytes,rpl", [(203, 0.05, 8, 8, 1), (203, 0.05, 1, 8, 1), (64, 0.5, 32, 8, 1),
                                                         (1, 0.0, 1, 8, 1), (5, 1.0, 4, 16, 1), (2000, 0.01, 8, 8, 1),
                                                         (2000, 0.01, 4, 16, 1), (801, 0.06, 2, 8, 1), (203, 0.05, 8, 8, 2),
                                                         (2000, 0.01, 8, 8, 2), (64, 0.5, 32, 8, 2), (801, 0.06, 2, 8, 2)])
def test_stream_covers_csr_exactly(nat, n, density, RT, pair_bytes, rpl, keep_order):
    import paper_2505_22631_b200 as pkg
    iu, iv, w = random_graph_arrays(n, density, seed=n + RT)
    J = pkg.CouplingMatrix.from_edges(n, (iu, iv, w))
    plan = compile_plan(nat, J, RT, pair_bytes=pair_bytes, keep_order=keep_order, rpl=rpl)
    seen, loads = walk(J, RT, plan)
    assert sorted(seen) == list(range(n))
    for i in range(n):
        want = J.indices[J.indptr[i]:J.indptr[i + 1]]
        if keep_order:
            assert np.array_equal(seen[i], want), f"row {i}"        # parity mode: CSR order
        else:
            assert np.array_equal(np.sort(seen[i]), want), f"row {i}"
    assert plan["W"] * 32 <= 1024 and plan["W"] >= 1 and plan["T"] >= 1
    assert plan["W"] * plan["Cs"] * plan["T"] * 4 >= n
    bad, total = wavefront_conflicts(RT, plan, pair_bytes)
    assert bad >= 0 and total >= 0


def test_g22_shape_padding_balance_and_banks(nat):
    """The headline shape: small padding, balanced warps, and the reordering removes most of the
    bank conflicts the CSR order has."""
    import paper_2505_22631_b200 as pkg
    from paper_2505_22631_b200 import workloads
    n, (u, v, w), _, _ = workloads.shape_graph("G22")
    J = pkg.CouplingMatrix.from_edges(n, (u, v, w))
    for rpl in (1, 2):
        fast = compile_plan(nat, J, 8, rpl=rpl)
        strict = compile_plan(nat, J, 8, keep_order=True, rpl=rpl)
        seen, loads = walk(J, 8, fast)
        fill = J.nnz / (fast["GR"] * 4 * fast["Cs"])
        assert fill > 0.78, (rpl, fill)
        assert loads.max() / loads.mean() < 1.10
        bad_fast, total = wavefront_conflicts(8, fast, 8)
        bad_strict, _ = wavefront_conflicts(8, strict, 8)
        assert bad_fast < 0.15 * total, (bad_fast, total)
        assert bad_fast < 0.4 * bad_strict, (bad_fast, bad_strict)


def test_plan_argument_errors(nat):
    ip = np.zeros(3, np.int64)
    W, T, GR = C.c_int32(), C.c_int32(), C.c_int64()
    for RT in (0, 3, 64):
        rc = nat.lib().oscb_resident_plan_host(2, nat.ptr(ip), None, RT, 1, 1024, 8, 0, C.byref(W), C.byref(T), C.byref(GR),
                                               None, None, None, None, None)
        assert rc == nat.EINVAL
