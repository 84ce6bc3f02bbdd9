"""CPU (gloo): the distributed solve_stokes of paper_2306_06795_b200.dsolve over
the rank-local partition of paper_2306_06795_b200.partition reproduces the
reference's single-process solve (preconditioner.cpp:229-259): FGMRES
iteration count within +-1, final relative residual <= tol, same solution.
The rank-local kernels are the C restatement here (tests/dist_checker.py); on
B200 the same DistSolver drives libsag kernels over NCCL (test_gpu_dist.py)."""
import os
import socket

import numpy as np
import pytest
from conftest import collect_results

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def golden_system(name):
    import oracle as O
    g = dict(np.load(os.path.join(GOLD, name + ".npz")))
    k0 = O.Csr(*[int(v) for v in g["k0_shape"]], g["k0_rp"], g["k0_ci"], g["k0_v"])
    levels = []
    for l in range(int(g["nlevels"])):
        k = O.Csr(*[int(v) for v in g[f"L{l}_k_shape"]], g[f"L{l}_k_rp"], g[f"L{l}_k_ci"],
                  g[f"L{l}_k_v"])
        p = None
        if f"L{l}_p_shape" in g:
            p = O.Csr(*[int(v) for v in g[f"L{l}_p_shape"]], g[f"L{l}_p_rp"], g[f"L{l}_p_ci"],
                      g[f"L{l}_p_v"])
        levels.append((k, p, tuple(int(v) for v in g[f"L{l}_nxyz"])))
    nxyz0 = tuple(int(v) for v in g["nxyz0"])
    return g, k0, levels, nxyz0


def reference_system(n, variant=0, gamma=1):
    """A deeper hierarchy straight from the reference build (oracle/_ref), and
    the reference's solve with preconditioner `variant` (DC-all / DC-LO /
    DC-HO) and gamma V-cycles."""
    from conftest import ref_case
    c, d, k0, levels, conf = ref_case(n, cfg=dict(variant=variant, gamma=gamma))
    xs, rep = d.solve(c.rhs())
    g = {"rhs": c.rhs(), "solve_x": xs, "solve_iterations": np.array(rep["iterations"]),
         "config": np.array([1, 1, 30, 500]), "config_f": np.array([1e-8, 1.0, 1.0, 1.0]),
         "enclosed": np.array(int(c.enclosed)), "variant": variant, "gamma": gamma}
    return g, k0, levels, (c.n_x0, c.n_y0, c.n_p0)


def unstructured_system(n):
    """BASELINE config 4's recipe (jittered Delaunay, zero velocity, forced)
    at n x n points, built and solved by the reference (oracle/_ref)."""
    import tempfile
    import oracle as O
    from paper_2306_06795_b200 import meshgen
    path = os.path.join(tempfile.gettempdir(), f"sag_test_mesh_{n}_{os.getpid()}.json")
    meshgen.write_mesh(path, n, seed=7, jitter=0.3)
    k1, k2 = meshgen.force_wavenumbers()
    c = O.RefCase.mesh_forced(path, k1, k2)
    conf = dict(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500, enclosed_flow=c.enclosed)
    d = O.RefDC(c, conf)
    xs, rep = d.solve(c.rhs())
    g = {"rhs": c.rhs(), "solve_x": xs, "solve_iterations": np.array(rep["iterations"]),
         "config": np.array([1, 1, 30, 500]), "config_f": np.array([1e-8, 1.0, 1.0, 1.0]),
         "enclosed": np.array(int(c.enclosed))}
    return g, d.k0().csr(), d.levels_csr(), (c.n_x0, c.n_y0, c.n_p0)


def _system(source):
    if isinstance(source, str):
        return golden_system(source)
    if source[0] == "mesh":
        return unstructured_system(source[1])
    return reference_system(*source)


def _worker(rank, world, port, source, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    import paper_2306_06795_b200 as S
    from dist_checker import CheckerBackend
    from paper_2306_06795_b200.dsolve import Comm, DistSolver
    from paper_2306_06795_b200.partition import build_rank_systems

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, k0, levels, nxyz0 = _system(source)
        nu1, nu2, restart, max_iters = (int(v) for v in g["config"])
        tol = float(g["config_f"][0])
        cfg = S.SolverConfig(nu1=nu1, nu2=nu2, restart=restart, tol=tol, max_iters=max_iters,
                             enclosed_flow=bool(int(g["enclosed"])),
                             variant=int(g.get("variant", 0)), gamma=int(g.get("gamma", 1)))
        l0, p0, nxyz_l0 = levels[0]
        rs = build_rank_systems(world, k0, l0, p0, nxyz0, nxyz_l0, ranks=[rank])[0]
        be = CheckerBackend()
        solver = DistSolver(rs, levels, cfg, be, Comm(dist, torch))
        rhs = torch.from_numpy(g["rhs"][rs.l2g].copy())
        x = be.vec(rs.nl)
        rep = solver.solve(rhs, x)
        own = np.nonzero(rs.owned)[0]
        q.put((rank, rs.l2g[own], x.numpy()[own], rep.iterations, rep.final_relative_residual,
               rep.converged, rs.ghost_count()))
    finally:
        dist.destroy_process_group()


def _run(world, source):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, source, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = collect_results(q, procs, world)  # before join: a full pipe blocks the sender
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("world,source", [(1, "th_cavity_8"), (2, "th_cavity_8"),
                                          (1, "th_cavity_16"), (2, "th_cavity_16"),
                                          (1, (32,)), (2, (32,)), (3, (32,)),
                                          (2, (32, 1)), (2, (32, 2)), (2, (32, 0, 2)),
                                          (3, ("mesh", 24))])
def test_distributed_solve_matches_reference(world, source):
    """source: a golden case, or (n, variant, gamma) of a reference-built one
    (DC-all / DC-LO / DC-HO, gamma V-cycles)."""
    pytest.importorskip("torch")
    g = _system(source)[0]
    out = _run(world, source)
    n = len(g["rhs"])
    x = np.full(n, np.nan)
    its = set()
    for rank, gids, xo, it, rel, conv, ghosts in out:
        assert np.isnan(x[gids]).all()          # ownership is a partition
        x[gids] = xo
        its.add(it)
        assert conv and rel <= float(g["config_f"][0])
        if world > 1:
            assert ghosts > 0
    assert len(its) == 1                        # every rank ran the same iterations
    it = its.pop()
    assert abs(it - int(g["solve_iterations"])) <= 1, (it, int(g["solve_iterations"]))
    xr = g["solve_x"]
    assert np.abs(x - xr).max() <= 1e-5 * np.abs(xr).max()


def test_rank_plans_are_consistent():
    """Host planning: local numbering monotone, ownership a partition, local
    rows and patches are the global ones renumbered, halo plans pair up."""
    from paper_2306_06795_b200.partition import build_rank_systems, th_patches
    g, k0, levels, nxyz0 = golden_system("th_cavity_16")
    l0, p0, nl0 = levels[0]
    n = k0.nrows
    pk = th_patches(k0.rp, k0.ci, *nxyz0)
    # build_patches restated on the host equals the reference's lists
    for a, b in zip(pk, ("pptr", "pidx", "vptr", "vidx", "nx")):
        assert np.array_equal(a, g["patch_" + b])
    for world in (1, 2, 3):
        rss = build_rank_systems(world, k0, l0, p0, nxyz0, nl0)
        seen = np.zeros(n, dtype=int)
        for rs in rss:
            assert np.all(np.diff(rs.l2g) > 0)
            seen[rs.l2g[rs.owned.astype(bool)]] += 1
            assert rs.n_u_loc == np.searchsorted(rs.l2g, nxyz0[0] + nxyz0[1])
            ll = rs.levels["K0"]
            for li in np.nonzero(rs.owned)[0][:50]:
                gr = rs.l2g[li]
                a = slice(k0.rp[gr], k0.rp[gr + 1])
                b = slice(ll.rows_rp[li], ll.rows_rp[li + 1])
                assert np.array_equal(rs.l2g[ll.rows_ci[b]], k0.ci[a])
                assert np.array_equal(ll.rows_v[b], k0.v[a])
            pptr, pidx, vptr, vidx, nx = ll.patches
            lo, hi = rs.patch_lo, rs.patch_hi
            assert np.array_equal(rs.l2g[vidx], pk[3][pk[2][lo]:pk[2][hi]])
            assert np.array_equal(rs.l2g[pidx], pk[1][pk[0][lo]:pk[0][hi]])
            for q_, idx in rs.fwd_recv.items():
                assert np.array_equal(rs.l2g[idx], rss[q_].l2g[rss[q_].fwd_send[rs.rank]])
                assert not rs.owned[idx].any() and rss[q_].owned[rss[q_].fwd_send[rs.rank]].all()
            for q_, idx in rs.rev_send.items():
                assert np.array_equal(rs.l2g[idx], rss[q_].l2g[rss[q_].rev_recv[rs.rank]])
            # interior / boundary split: a partition of the patches and rows
            pi, pb = ll.patches_int, ll.patches_bnd
            assert len(pi[0]) - 1 + len(pb[0]) - 1 == len(pptr) - 1
            assert rs.owned[pi[3]].all() and rs.owned[pi[1]].all()
            ri, rb = ll.rows_int, ll.rows_bnd
            assert np.array_equal(np.diff(ri[0]) + np.diff(rb[0]), np.diff(ll.rows_rp))
            assert rs.owned[ri[1]].all()
            if world == 1:
                assert rs.ghost_count() == 0
                assert len(pb[0]) == 1 and len(rb[1]) == 0
        assert (seen == 1).all()
