#!/usr/bin/env python
"""FGMRES iteration counts of the full DC-all solve under launch-shape
variants (env strings read at device setup), one host case built once.
A variant that changes the count changes the numerics, not only the speed.

    python tools/iters_check.py [n=512] ["ENV=V,ENV=V;ENV=V"]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2306_06795_b200 as S  # noqa: E402
from paper_2306_06795_b200.cases import HostCase  # noqa: E402


def main():
    n_mesh = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    variants = sys.argv[2].split(";") if len(sys.argv) > 2 else [""]
    case = HostCase("cavity", False, "structured", n_mesh)
    ctx = S.Context(0)
    cfg = S.SolverConfig(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500, enclosed_flow=True)
    rhs = case.rhs()
    for var in variants:
        env = dict(kv.split("=") for kv in var.split(",") if kv)
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        K0, dc, _ = case.device(cfg, ctx)
        t0 = time.perf_counter()
        x, rep = S.solve_stokes(K0, rhs, dc, cfg)
        ctx.synchronize()
        print(json.dumps({"variant": var, "iterations": rep.iterations,
                          "final_rel": rep.final_relative_residual,
                          "solve_s": time.perf_counter() - t0}), flush=True)
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        del dc, K0


if __name__ == "__main__":
    main()
