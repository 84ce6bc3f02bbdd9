#!/usr/bin/env python
"""Generates the golden fixtures under tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/libstokesamg_ref.so, built from /root/reference by
oracle/Makefile). Run in the build container:

    python tests/golden/make_golden.py

Each .npz holds the reference's inputs (K0, low-order hierarchy, patch lists)
and outputs (spmv, factor payload, apply_vanka, vanka_relax, DC apply, solve)
for one small case, so the CPU suite can pin the C restatement and the GPU
suite can check the device path without /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402


def csr_dict(prefix, m):
    return {f"{prefix}_shape": np.array([m.nrows, m.ncols]), f"{prefix}_rp": m.rp,
            f"{prefix}_ci": m.ci, f"{prefix}_v": m.v}


def make_case(name, problem, sv, n, cfg):
    c = O.RefCase.build(problem, sv, "structured", n)
    conf = dict(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500, enclosed_flow=c.enclosed)
    conf.update(cfg)
    out = {"nxyz0": np.array([c.n_x0, c.n_y0, c.n_p0]), "enclosed": np.array(int(c.enclosed)),
           "config": np.array([conf["nu1"], conf["nu2"], conf["restart"], conf["max_iters"]]),
           "config_f": np.array([conf["tol"], conf.get("eta_u", 1.0), conf.get("eta_p", 1.0),
                                 conf.get("omega0", 1.0)])}
    rhs = c.rhs()
    out["rhs"] = rhs
    k0r = c.k0()
    k0 = k0r.csr()
    out.update(csr_dict("k0", k0))
    x = O.splitmix64_uniform(k0.nrows)
    out["x"] = x
    out["spmv"] = k0r.spmv(x)
    v = O.RefVanka.build(k0r, c.n_x0, c.n_y0, c.n_p0, sv_triples=sv)
    p = v.patches()
    for a in ("pptr", "pidx", "vptr", "vidx", "nx"):
        out[f"patch_{a}"] = getattr(p, a)
    fac = v.factors()
    for a in ("uhat", "bhat", "sinv", "weights"):
        out[f"factor_{a}"] = fac[a]
    out["storage"] = np.array([fac["a_factor_bytes"], fac["aux_bytes"],
                               fac["dense_inverse_bytes"]])
    out["apply_vanka"] = v.apply(x)
    x0 = np.sin(0.1 * np.arange(k0.nrows))
    out["relax_kw1"] = v.relax(x0, x, 0, 1, 1.0)
    out["relax_kw2"] = v.relax(x0, x, 0, 2, 1.0)
    out["relax_st3"] = v.relax(x0, x, 1, 3, 0.78)
    if not sv:
        d = O.RefDC(c, conf)
        levels = d.levels_csr()
        out["nlevels"] = np.array(len(levels))
        for l, (k, pm, nxyz) in enumerate(levels):
            out.update(csr_dict(f"L{l}_k", k))
            out[f"L{l}_nxyz"] = np.array(nxyz)
            if pm is not None:
                out.update(csr_dict(f"L{l}_p", pm))
        out["dc_apply"] = d.apply(x)
        out["vcycle"] = d.vcycle(x[:levels[0][0].nrows])
        xs, rep = d.solve(rhs)
        out["solve_x"] = xs
        out["solve_iterations"] = np.array(rep["iterations"])
        out["solve_final_rel"] = np.array(rep["final_relative_residual"])
        out["solve_history"] = rep["residual_history"]
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, {k: v.shape for k, v in out.items() if k in ("k0_v", "x")},
          "solve its", out.get("solve_iterations"))


def make_kats():
    """Known-answer tests of the reference suite, as reference outputs."""
    out = {}
    # tests/test_sparse.cpp:37-45
    m = O.RefMat.from_triplets(3, 3, [0, 0, 1, 1, 2, 2], [0, 1, 1, 2, 0, 2], [1, 2, 3, 4, 5, 6])
    out["hand_spmv"] = m.spmv(np.array([1.0, 2.0, 3.0]))
    # tests/test_vanka.cpp:98-113
    k = O.RefMat.from_triplets(3, 3, [0, 0, 1, 2], [0, 2, 1, 0], [1, 1, 1, 1])
    pt = O.Patches(np.array([0, 1], np.int32), np.array([2], np.int32),
                   np.array([0, 2], np.int32), np.array([0, 1], np.int32),
                   np.array([1], np.int32))
    v = O.RefVanka.from_patches(k, pt, 2)
    out["hand_patch_sinv"] = v.factors()["sinv"]
    out["hand_patch_apply"] = v.apply(np.array([1.0, 0.0, 1.0]))
    # tests/test_vanka.cpp:196-212 / :244-262 single-patch system
    k1 = O.RefMat.from_triplets(3, 3, [0, 0, 1, 1, 2, 2], [0, 2, 1, 2, 0, 1],
                                [2, 1, 3, -1, 1, -1])
    v1 = O.RefVanka.from_patches(k1, pt, 2)
    out["onepatch_apply"] = v1.apply(np.array([1.0, 2.0, 3.0]))
    xref = np.array([1.0, -2.0, 0.5])
    b = k1.spmv(xref)
    out["onepatch_stationary"] = v1.relax(np.zeros(3), b, 1, 4, 0.78)
    out["onepatch_kw"] = v1.relax(np.zeros(3), np.array([1.0, -2.0, 0.5]), 0, 1, 1.0)
    # tests/test_sparse.cpp:85-107 dense LU known system
    a = np.array([[2, 1, 0], [1, 3, 1], [0, 1, 4]], dtype=float)
    out["lu_known"] = O.Oracle.lu_solve_dense(a, [4.0, 10.0, 14.0])
    # tests/test_krylov.cpp:83-95: poisson1d(32), b = 1, identity prec, tol 1e-9
    nn = 32
    rows, cols, vals = [], [], []
    for i in range(nn):
        rows.append(i), cols.append(i), vals.append(2.0)
        if i > 0:
            rows.append(i), cols.append(i - 1), vals.append(-1.0)
        if i + 1 < nn:
            rows.append(i), cols.append(i + 1), vals.append(-1.0)
    pm = O.RefMat.from_triplets(nn, nn, rows, cols, vals)
    xk, rep = O.ref_fgmres(pm, np.ones(nn), np.zeros(nn), 0, None, tol=1e-9, max_iters=500,
                           restart=20)
    out["poisson_csr_rp"], out["poisson_csr_ci"], out["poisson_csr_v"] = (
        pm.csr().rp, pm.csr().ci, pm.csr().v)
    out["poisson_fgmres_x"] = xk
    out["poisson_fgmres_hist"] = rep["residual_history"]
    out["poisson_fgmres_its"] = np.array(rep["iterations"])
    np.savez_compressed(os.path.join(HERE, "kats.npz"), **out)
    print("kats", sorted(out))


if __name__ == "__main__":
    make_case("th_cavity_8", "cavity", False, 8, {})
    make_case("th_cavity_16", "cavity", False, 16, dict(coarse_size=0))
    make_case("sv_cavity_4", "cavity", True, 4, dict(omega0=0.78, eta_p=2.68))
    make_kats()
