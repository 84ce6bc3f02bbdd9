"""GPU: the distributed solve (paper_2306_06795_b200.dsolve) with libsag's
sm_100a kernels as the rank-local kernels (dsolve.LibsagBackend) against the
reference's single-process solve (oracle/_ref): FGMRES iterations within +-1,
final relative residual <= tol, same solution.

* world 1 over NCCL (every collective degenerate, the device path itself);
* world 2 as two processes sharing the one GPU of the test box, exchanging
  over gloo staged through host memory -- the ranks' kernels never wait on
  one another (every exchange is a host-synchronised copy), so this is the
  multi-rank host logic (halos, masked reductions, all-reduces, agglomerated
  coarse levels) driving the real device kernels; with "gloo-peer" the
  reverse halo of every sweep goes over peer memory (each rank writes its
  partial sums into the neighbour's buffer mapped by CUDA IPC). NCCL across
  GPUs is the bench's --gpus N path."""
import os
import socket

import numpy as np
import pytest
from conftest import collect_results

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, backend, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    import paper_2306_06795_b200 as S
    from paper_2306_06795_b200.dsolve import Comm, DistSolver, LibsagBackend
    from paper_2306_06795_b200.partition import build_rank_systems
    from test_dist_solve import reference_system

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    peer = backend == "gloo-peer"   # reverse halo over peer memory (CUDA IPC)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, k0, levels, nxyz0 = reference_system(n)
        cfg = S.SolverConfig(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500,
                             enclosed_flow=True)
        l0, p0, nxyz_l0 = levels[0]
        rs = build_rank_systems(world, k0, l0, p0, nxyz0, nxyz_l0, ranks=[rank])[0]
        stream = torch.cuda.Stream(device=dev)
        ctx = S.Context(0, stream=stream.cuda_stream)
        with torch.cuda.stream(stream):
            be = LibsagBackend(ctx, dev, torch, stream)
            solver = DistSolver(rs, levels, cfg, be, Comm(dist, torch, stage=backend != "nccl"),
                                peer=peer)
            assert (solver.peer is not None) == peer
            rhs = be.from_host(g["rhs"][rs.l2g])
            x = be.vec(rs.nl)
            l0n = ctx.launch_count()
            rep = solver.solve(rhs, x)
            torch.cuda.synchronize(dev)
            launches = ctx.launch_count() - l0n
        own = np.nonzero(rs.owned)[0]
        # the preconditioner runs as a CUDA graph whenever the communicator allows
        assert (solver.graph is not None) == (backend == "nccl"), solver.graph_error
        if peer:
            # a rank with ghost partial sums sent them from its boundary gathers
            # (fused path; the lowest rank owns every dof its patches touch)
            assert solver.peer.fused > 0 or not rs.rev_send
        # fence, unmap the neighbours' buffers, barrier, free ours
        solver.close()
        assert solver.peer is None
        q.put((rank, rs.l2g[own], x.cpu().numpy()[own], rep.iterations,
               rep.final_relative_residual, rep.converged, launches))
    finally:
        dist.destroy_process_group()


def _run(world, n, backend):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, backend, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = collect_results(q, procs, world)
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("world,n,backend", [(1, 32, "nccl"), (1, 64, "nccl"),
                                             (2, 32, "gloo"), (2, 64, "gloo"),
                                             (2, 32, "gloo-peer"), (2, 64, "gloo-peer"),
                                             (4, 32, "gloo"), (4, 32, "gloo-peer")])
def test_gpu_distributed_solve_matches_reference(world, n, backend):
    from test_dist_solve import reference_system
    g = reference_system(n)[0]
    out = _run(world, n, backend)
    x = np.full(len(g["rhs"]), np.nan)
    its = set()
    for rank, gids, xo, it, rel, conv, launches in out:
        assert launches > 0                     # libsag kernels ran
        assert np.isnan(x[gids]).all()
        x[gids] = xo
        its.add(it)
        assert conv and rel <= 1e-8
    assert len(its) == 1
    it = its.pop()
    assert abs(it - int(g["solve_iterations"])) <= 1, (it, int(g["solve_iterations"]))
    xr = g["solve_x"]
    assert np.abs(x - xr).max() <= 1e-5 * np.abs(xr).max()
