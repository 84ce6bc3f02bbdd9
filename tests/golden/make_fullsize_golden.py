#!/usr/bin/env python
"""Full-size goldens of the BASELINE configs, produced by the UNMODIFIED
reference (oracle/_ref/libstokesamg_ref.so, built from /root/reference by
oracle/Makefile) on exactly the inputs bench.py uses:

  config 1  TH cavity 64x64            (experiments.cpp:215-235)
  config 2  TH cavity 512x512
  config 3  SV cavity 256x256 barycentric, (omega0, eta_u, eta_p) = (0.78, 1, 2.68)
  config 4  TH on meshgen.write_mesh(500, seed=7, jitter=0.3), zero velocity,
            f = (sin k1 x, cos k2 y) with k1, k2 = meshgen.force_wavenumbers()
            (splitmix64; SURVEY 8(d) asks for a portable generator)

Vectors of this size are not committed; the fixture holds what a GPU test
needs to pin parity without /root/reference:
  * sha256 of K0's and ISO0's (low-order level 0) CSR arrays, so the GPU box
    proves it rebuilt the very same operators,
  * the reference's solve_stokes report (iterations, final relative residual,
    the residual history) with DC-all V(1,1), FGMRES(30), rtol 1e-8,
  * norms of spmv / apply_vanka on K0 and ISO0 with the splitmix64 input,
  * the wall time of that solve on one core of this container.

    python tests/golden/make_fullsize_golden.py [config ...]   (one file per config, fullsize_config<N>.json; ~5 min each for 2-4)
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

def out_path(config: int) -> str:
    return os.path.join(HERE, f"fullsize_config{config}.json")


def csr_sha(m) -> str:
    h = hashlib.sha256()
    for a in (np.asarray(m.rp, np.int32), np.asarray(m.ci, np.int32), np.asarray(m.v, np.float64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def vec_stats(v):
    v = np.asarray(v)
    return {"l2": float(np.linalg.norm(v)), "linf": float(np.abs(v).max()),
            "sum": float(v.sum()), "sha256": hashlib.sha256(v.tobytes()).hexdigest()}


def make(config: int) -> dict:
    import bench
    cfg = bench.CONFIGS[config]
    t0 = time.perf_counter()
    case = bench.ref_case(cfg)
    conf = dict(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500, enclosed_flow=case.enclosed,
                eta_u=cfg.get("eta_u", 1.0), eta_p=cfg.get("eta_p", 1.0),
                omega0=cfg.get("omega0", 1.0))
    d = O.RefDC(case, conf)
    setup_s = time.perf_counter() - t0
    k0r = d.k0()
    k0 = k0r.csr()
    iso0, p0, nxyz1 = d.level(0)
    iso0c = iso0.csr()
    out = {"workload": cfg["workload"], "nxyz0": [case.n_x0, case.n_y0, case.n_p0],
           "nxyz_iso0": list(nxyz1), "sv": bool(case.sv), "solver": conf,
           "k0": {"nrows": k0.nrows, "nnz": k0.nnz, "sha256": csr_sha(k0)},
           "iso0": {"nrows": iso0c.nrows, "nnz": iso0c.nnz, "sha256": csr_sha(iso0c)},
           "rhs": vec_stats(case.rhs())}
    x = O.splitmix64_uniform(k0.nrows)
    out["k0"]["spmv"] = vec_stats(k0r.spmv(x))
    rv = O.RefVanka.build(k0r, case.n_x0, case.n_y0, case.n_p0, sv_triples=case.sv)
    out["k0"]["apply_vanka"] = vec_stats(rv.apply(x))
    del rv
    xi = O.splitmix64_uniform(iso0c.nrows)
    out["iso0"]["spmv"] = vec_stats(iso0.spmv(xi))
    out["iso0"]["apply_vanka"] = vec_stats(d.level_vanka(0).apply(xi))
    t1 = time.perf_counter()
    xs, rep = d.solve(case.rhs())
    solve_s = time.perf_counter() - t1
    out["solve"] = {"converged": rep["converged"], "iterations": rep["iterations"],
                    "final_relative_residual": rep["final_relative_residual"],
                    "residual_history": [float(v) for v in rep["residual_history"]],
                    "x": vec_stats(xs), "cpu_s_1core": solve_s,
                    "cpu": "this container's host, 1 thread"}
    out["setup_s"] = setup_s
    return out


def main():
    for c in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4]:
        t = time.perf_counter()
        d = make(c)
        print(f"config {c}: {d['solve']['iterations']} its, "
              f"{d['solve']['final_relative_residual']:.6e}, {time.perf_counter() - t:.0f} s",
              flush=True)
        with open(out_path(c), "w") as f:
            json.dump(d, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
