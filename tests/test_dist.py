"""CPU (gloo, world size 2 and 3): the partitioned hot step of
paper_2306_06795_b200.dsolve.DistStep -- rank-local numbering
(paper_2306_06795_b200.partition), forward halo of x, rank-local Vanka + SpMV,
reverse halo of the Vanka partial sums -- reproduces the single-process
result. The rank-local kernels are the C restatement (oracle/) here, as the
checker (tests/dist_checker.py); on B200 the same DistStep drives libsag
kernels over NCCL (bench.py --gpus N)."""
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


def _worker(rank, world, port, name, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    from dist_checker import CheckerBackend
    from paper_2306_06795_b200.dsolve import Comm, DistStep
    from paper_2306_06795_b200.partition import build_rank_systems
    from test_dist_solve import golden_system

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, k0, levels, nxyz0 = golden_system(name)
        l0, p0, nxyz_l0 = levels[0]
        rs = build_rank_systems(world, k0, l0, p0, nxyz0, nxyz_l0, ranks=[rank])[0]
        be = CheckerBackend()
        step = DistStep(rs, be, Comm(dist, torch))
        x = torch.full((rs.nl,), float("nan"), dtype=torch.float64)
        own = np.nonzero(rs.owned)[0]
        x[own] = torch.from_numpy(g["x"][rs.l2g[own]])   # ghosts come from the halo
        delta, y = be.vec(rs.nl), be.vec(rs.nl)
        step.step(x, delta, y)
        q.put((rank, rs.l2g[own], delta.numpy()[own], y.numpy()[own], rs.ghost_count()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("th_cavity_8", 2), ("th_cavity_16", 2),
                                        ("th_cavity_16", 3)])
def test_partitioned_step_matches_single_process(name, world):
    pytest.importorskip("torch")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = collect_results(q, procs, world)
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    g = dict(np.load(os.path.join(GOLD, name + ".npz")))
    seen = np.zeros(len(g["x"]), dtype=bool)
    for rank, gids, delta, y, ghosts in out:
        assert ghosts > 0                       # a real halo exists
        assert not seen[gids].any()             # ownership is a partition
        seen[gids] = True
        assert np.allclose(delta, g["apply_vanka"][gids], rtol=1e-13, atol=1e-15)
        assert np.array_equal(y, g["spmv"][gids])  # same rows, same order
    assert seen.all()
