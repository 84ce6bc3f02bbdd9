#!/usr/bin/env python
"""Solve time of every preconditioner variant (preconditioner.hpp:14: DC-all,
DC-LO, DC-HO, HO-AMG, Uzawa) on one bench config, GPU (CUDA events around
solve_stokes, after a warm-up solve) and optionally the reference on one host
core (oracle/_ref, experiments.cpp's make_preconditioner + solve_stokes).

    python tools/variants_bench.py [--config 1] [--ref] [--variants 0,3,4]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_06795_b200 as S  # noqa: E402

NAMES = {0: "DC-all", 1: "DC-LO", 2: "DC-HO", 3: "HO-AMG", 4: "Uzawa"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--ref", action="store_true")
    ap.add_argument("--variants", default="0,3,4")
    args = ap.parse_args()
    conf = bench.CONFIGS[args.config]
    t0 = time.perf_counter()
    case = bench.host_case(conf)
    setup = time.perf_counter() - t0
    stream = torch.cuda.Stream(device=torch.device("cuda", 0))
    ctx = S.Context(0, stream=stream.cuda_stream)
    rhs = case.rhs()
    print(json.dumps({"config": conf["workload"], "n0": case.n0, "host_setup_s": setup}),
          flush=True)
    for v in (int(s) for s in args.variants.split(",")):
        cfg = S.SolverConfig(variant=v, nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500,
                             enclosed_flow=case.enclosed, eta_u=conf.get("eta_u", 1.0),
                             eta_p=conf.get("eta_p", 1.0), omega0=conf.get("omega0", 1.0))
        rec = {"variant": NAMES[v]}
        try:
            ts = time.perf_counter()
            if v == 3:
                K0, prec = case.hoamg_device(cfg, ctx)
            elif v == 4:
                K0, prec = case.uzawa_device(cfg, ctx)
            else:
                K0, prec, _ = case.device(cfg, ctx)
            ctx.synchronize()
            rec["setup_s"] = time.perf_counter() - ts  # host hierarchy + device factors
            S.solve_stokes(K0, rhs, prec, cfg)  # warm-up (graph capture)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            x, rep = S.solve_stokes(K0, rhs, prec, cfg)
            e1.record(stream)
            e1.synchronize()
            rec.update(gpu_solve_s=e0.elapsed_time(e1) / 1e3, iterations=rep.iterations,
                       converged=rep.converged, final_rel=rep.final_relative_residual)
        except S.Error as e:
            rec["error"] = str(e)
        if args.ref:
            import oracle as O
            c = bench.ref_case(conf)
            rconf = dict(variant=v, nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500,
                         enclosed_flow=c.enclosed, eta_u=conf.get("eta_u", 1.0),
                         eta_p=conf.get("eta_p", 1.0), omega0=conf.get("omega0", 1.0))
            try:
                p = O.RefPrec(c, rconf)
                ts = time.perf_counter()
                _, rr = p.solve(c.rhs())
                rec.update(ref_cpu_solve_s_1core=time.perf_counter() - ts,
                           ref_iterations=rr["iterations"])
            except O.OracleError as e:
                rec["ref_error"] = str(e)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
