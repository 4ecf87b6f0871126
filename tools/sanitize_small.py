"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2505_22631_b200 as pkg
from paper_2505_22631_b200 import dynamics, workloads

which = sys.argv[1:] or ["resident", "cluster", "stream", "dense-tc", "lowdeg", "lowdeg-pair", "dense-splitk"]
u, v, w = workloads.random_gnm(128, 700, seed=1, weights=(1.0,))
J = pkg.CouplingMatrix.from_edges(128, (u, v, w))
p = pkg.SolverParams.tuned_for(128, 2, seed=0, t_stop=0.6)
if "resident" in which:
    b = pkg.run_batch(J, p, "maxcut", list(range(20)), kernel="resident")
    print("resident", b.best_objective.max())
    c3 = pkg.run_batch(J, pkg.SolverParams.tuned_for(128, 3, seed=0, t_stop=0.6), "coloring", list(range(20)), kernel="resident")
    print("resident N=3", c3.best_objective.min())
if "cluster" in which:
    b = pkg.run_batch(J, p, "maxcut", [0, 1], kernel="cluster")
    print("cluster", b.best_objective.max())
if "stream" in which:
    b = pkg.run_batch(J, p, "maxcut", [0, 1, 2], kernel="stream", precision="f64")
    print("stream", b.best_objective.max())
if "dense-tc" in which:
    rng = np.random.default_rng(3)
    U = np.triu(rng.choice(np.array([-1.0, 1.0]), size=(300, 300)), 1)
    g = dynamics.DeviceGraph.from_dense(0, U + U.T)
    b = pkg.run_batch(None, pkg.SolverParams(K=0.02, ks_max=1.0, ks_period=0.5, kn=0.1, h=0.01, t_stop=0.3, seed=0), "maxcut", [0, 1, 2], graph=g)
    print("dense-tc", b.kernel, b.best_objective.max())
    g.close()
if "lowdeg" in which:
    # straight-line stream (torus, one and several replicas per CTA), looped stream (N = 3; N = 2 = the two-replica-per-lane kernel)
    ut, vt, wt = workloads.torus_pm1(10, 20, seed=2)
    Jt = pkg.CouplingMatrix.from_edges(200, (ut, vt, wt))
    pt = pkg.SolverParams.tuned_for(200, 2, seed=0, t_stop=0.4)
    for rt in (1, 8):
        b = pkg.run_batch(Jt, pt, "maxcut", list(range(11)), kernel="lowdeg", replicas_per_cta=rt)
        print("lowdeg uniform rt", rt, b.kernel, b.best_objective.max())
    us, vs, ws = workloads.random_gnm(203, 520, seed=5, weights=(1.0, -1.0, 2.0))
    Js = pkg.CouplingMatrix.from_edges(203, (us, vs, ws))
    for rt in (1, 4):
        b = pkg.run_batch(Js, pkg.SolverParams.tuned_for(203, 2, seed=0, t_stop=0.4), "maxcut", list(range(9)), kernel="lowdeg", replicas_per_cta=rt)
        print("lowdeg looped N=2 rt", rt, b.kernel, b.best_objective.max())
    uc, vc, wc = workloads.random_gnm(203, 480, seed=6)
    Jc = pkg.CouplingMatrix.from_edges(203, (uc, vc, wc))
    b = pkg.run_batch(Jc, pkg.SolverParams.tuned_for(203, 3, seed=0, t_stop=0.4), "coloring", list(range(37)), kernel="lowdeg")
    print("lowdeg looped N=3", b.kernel, b.replicas_per_cta, b.best_objective.min())
if "lowdeg" in which:
    # the mixed-tile schedule of the one-replica-per-lane kernel (flat200 x 4096: tiles of 32 and of 16), windows of 3 steps
    import os, bench
    os.environ["OSCB_LOWDEG_MIXED_MIN_WINDOW"] = "1"
    _, Jf, pf, kindf, Rf = bench.load_workload("flat200x4096")
    b = pkg.run_batch(Jf, pf, kindf, list(range(Rf)), steps=96, want_phases=False)
    print("lowdeg mixed-tile schedule N=3", b.kernel, b.kernel_launches, b.best_objective.min())
    del os.environ["OSCB_LOWDEG_MIXED_MIN_WINDOW"]
if "lowdeg-pair" in which:
    # k_lowdeg_pair pinned: weighted and unit couplings (slot stream in shared memory), and the headline route (G22 shape,
    # enough 8-replica tiles to fill the GPU) for a few steps
    import os
    os.environ["OSCB_LOWDEG_RPL"] = "2"
    us, vs, ws = workloads.random_gnm(203, 520, seed=5, weights=(1.0, -1.0, 2.0))
    Js = pkg.CouplingMatrix.from_edges(203, (us, vs, ws))
    uu, vu, wu = workloads.random_gnm(301, 1500, seed=7)
    Ju = pkg.CouplingMatrix.from_edges(301, (uu, vu, wu))
    for name, Jp in (("weighted", Js), ("unit", Ju)):
        for rt in (2, 8):
            b = pkg.run_batch(Jp, pkg.SolverParams.tuned_for(Jp.n, 2, seed=0, t_stop=0.4), "maxcut", list(range(2 * rt + 1)), kernel="lowdeg", replicas_per_cta=rt)
            print("lowdeg pair", name, "rt", rt, b.kernel, b.replicas_per_cta, b.best_objective.max())
    del os.environ["OSCB_LOWDEG_RPL"]
    import bench
    _, J22, p22, kind, _ = bench.load_workload("G22x1024")
    b = pkg.run_batch(J22, p22, kind, list(range(896)), steps=3, want_phases=False)
    print("lowdeg pair headline route", b.kernel, b.replicas_per_cta, b.best_objective.max())
    os.environ["OSCB_LOWDEG_MIXED_MIN_WINDOW"] = "1"                     # the mixed-tile schedule with windows of a few steps
    b = pkg.run_batch(J22, p22, kind, list(range(1024)), steps=64, want_phases=False)
    print("lowdeg pair mixed-tile schedule", b.kernel, b.kernel_launches, b.best_objective.max())
    del os.environ["OSCB_LOWDEG_MIXED_MIN_WINDOW"]
    b = pkg.run_batch(J22, p22, kind, list(range(500)), steps=3, want_phases=False)
    print("lowdeg pair tiles of 4", b.kernel, b.replicas_per_cta, b.best_objective.max())
if "dense-splitk" in which:
    import os
    os.environ["OSCB_UMMA_SPLITK"] = "4"
    rng = np.random.default_rng(4)
    U = np.triu(rng.choice(np.array([-1.0, 1.0]), size=(512, 512)), 1)
    g = dynamics.DeviceGraph.from_dense(0, U + U.T)
    b = pkg.run_batch(None, pkg.SolverParams(K=0.02, ks_max=1.0, ks_period=0.5, kn=0.1, h=0.01, t_stop=0.3, seed=0), "maxcut", [0, 1, 2], graph=g)
    print("dense-tc split-K", b.kernel, b.best_objective.max())
    g.close()
