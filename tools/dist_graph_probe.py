#!/usr/bin/env python
"""Probe: the distributed solve at world size 1 (NCCL) with the
preconditioner captured into a CUDA graph, with progress on stderr. Run under
`timeout` on a GPU box:  timeout 300 python tools/dist_graph_probe.py [n]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, file=sys.stderr, flush=True)


def main():
    import torch
    import torch.distributed as dist

    import paper_2306_06795_b200 as S
    from paper_2306_06795_b200.dsolve import Comm, DistSolver, LibsagBackend
    from paper_2306_06795_b200.partition import build_rank_systems
    from test_dist_solve import reference_system

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    backend = sys.argv[2] if len(sys.argv) > 2 else "nccl"
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29571")
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    log("init", backend)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=0, world_size=1)
    g, k0, levels, nxyz0 = reference_system(n)
    log("case", k0.nrows, "levels", len(levels), "ref its", int(g["solve_iterations"]))
    cfg = S.SolverConfig(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500, enclosed_flow=True)
    l0, p0, nxyz_l0 = levels[0]
    rs = build_rank_systems(1, k0, l0, p0, nxyz0, nxyz_l0, ranks=[0])[0]
    stream = torch.cuda.Stream(device=dev)
    ctx = S.Context(0, stream=stream.cuda_stream)
    with torch.cuda.stream(stream):
        be = LibsagBackend(ctx, dev, torch, stream)
        solver = DistSolver(rs, levels, cfg, be, Comm(dist, torch))
        solver.use_graph = os.environ.get("PROBE_GRAPH", "1") == "1"
        log("solver ready, use_graph", solver.use_graph)
        rhs = be.from_host(g["rhs"][rs.l2g])
        x = be.vec(rs.nl)
        v, z = be.vec(rs.nl), be.vec(rs.nl)
        v.copy_(rhs)
        log("apply 1 (eager)")
        try:
            solver.apply_prec(v, z)
        finally:
            log("graph", solver.graph is not None, solver.graph_error)
        torch.cuda.synchronize()
        log("apply 1 done")
        solver.apply_prec(v, z)
        torch.cuda.synchronize()
        log("apply 2 done")
        t = time.perf_counter()
        rep = solver.solve(rhs, x)
        torch.cuda.synchronize()
        log("solve", rep.iterations, rep.final_relative_residual, time.perf_counter() - t)
    dist.destroy_process_group()
    log("done")


if __name__ == "__main__":
    main()
