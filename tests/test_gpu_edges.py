"""GPU edge cases and size-independent properties of the sm_100a path, against
the reference (oracle/_ref) where it defines the answer:

* CSR upload validation and degenerate shapes (empty, empty rows, 1x1,
  rectangular) -- sparse.cpp:11-76 semantics, errors.hpp exception classes;
* FGMRES (krylov.cpp:17-121) with every preconditioner kind, forced restarts,
  the iteration cap, a zero right-hand side and an exact first step;
* DC variants (DC-LO / DC-HO, gamma = 2, nu = 2) against the reference's
  DCPreconditioner (preconditioner.cpp:114-153);
* full-size config 2 (K0 of the 512x512 TH cavity): SpMV and Vanka sweep
  against the reference at 1e-12, linearity of both operators, and the full
  FGMRES solve's iteration count / true residual (38, 9.957e-9).
"""
import numpy as np
import pytest

import oracle as O
from conftest import ref_case

pytestmark = pytest.mark.gpu

TOL = 1e-12


def rel_inf(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    s = np.abs(b).max()
    return np.abs(a - b).max() / (s if s > 0 else 1.0)


@pytest.fixture(scope="module")
def S():
    import paper_2306_06795_b200 as S
    return S


# ------------------------------------------------------------------ CSR --
def test_csr_degenerate_shapes(S):
    # 0 x 0, all-empty rows, 1 x 1, rectangular with empty rows
    e = S.SparseMatrix(0, 0, [0], [], [])
    assert S.spmv(e, np.zeros(0)).size == 0
    z = S.SparseMatrix(3, 4, [0, 0, 0, 0], [], [])
    assert np.array_equal(S.spmv(z, np.ones(4)), np.zeros(3))
    one = S.SparseMatrix(1, 1, [0, 1], [0], [2.5])
    assert np.array_equal(S.spmv(one, np.array([4.0])), [10.0])
    r = O.RefMat.from_triplets(4, 2, [0, 0, 3], [0, 1, 1], [1.0, -2.0, 3.0]).csr()
    x = np.array([0.5, 0.25])
    assert np.array_equal(S.spmv(S.SparseMatrix.from_csr(r), x), O.RefMat.from_csr(r).spmv(x))


def test_csr_validation_errors(S):
    with pytest.raises(S.DimensionMismatch):  # row offsets not monotone
        S.SparseMatrix(2, 2, [0, 2, 1], [0, 1], [1.0, 1.0])
    with pytest.raises(S.DimensionMismatch):  # column out of range
        S.SparseMatrix(2, 2, [0, 1, 2], [0, 2], [1.0, 1.0])
    with pytest.raises(S.Error):  # non-canonical row (unsorted columns)
        S.SparseMatrix(1, 3, [0, 2], [2, 0], [1.0, 1.0])
    m = S.SparseMatrix(2, 2, [0, 1, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(S.DimensionMismatch):  # x of the wrong length
        S.spmv(m, np.ones(3))


# --------------------------------------------------------------- FGMRES --
def _fgmres_pair(S, k, prec_kind, tol=1e-8, max_iters=200, restart=20, b=None):
    rk = O.RefMat.from_csr(k)
    b = O.splitmix64_uniform(k.nrows) if b is None else b
    K = S.SparseMatrix.from_csr(k)
    if prec_kind == 1:
        nxyz = ref_case(16)[1].nxyz0
        rp = O.RefVanka.build(rk, *nxyz)
        gp = S.factor_patches(K, S.build_patches(K, *nxyz), nxyz[0] + nxyz[1])
    elif prec_kind == 2:
        rp, gp = rk, K
    else:
        rp, gp = None, None
    xr, rep_r = O.ref_fgmres(rk, b, np.zeros(k.nrows), prec_kind, rp, tol, max_iters, restart)
    xg = np.zeros(k.nrows)
    rep_g = S.fgmres(K, b, xg, gp, S.FgmresOptions(tol=tol, max_iters=max_iters,
                                                   restart=restart))
    return xr, rep_r, xg, rep_g


def _leading_block(k, n):
    """K[0:n, 0:n] of a Csr (the x-velocity block: SPD, nonzero diagonal)."""
    rows, cols, vals = [], [], []
    for i in range(n):
        sl = slice(k.rp[i], k.rp[i + 1])
        c = k.ci[sl]
        keep = c < n
        rows += [i] * int(keep.sum())
        cols += list(c[keep])
        vals += list(k.v[sl][keep])
    return O.RefMat.from_triplets(n, n, rows, cols, vals).csr()


@pytest.mark.parametrize("prec_kind,restart", [(0, 20), (1, 20), (1, 5), (2, 7)])
def test_fgmres_matches_reference(S, prec_kind, restart):
    # identity / Vanka / Jacobi preconditioners; restarts 5 and 7 force several
    # restart cycles (the true-residual restart at krylov.cpp:44-46). Jacobi
    # runs on the x-velocity block (the saddle-point K0 has a zero diagonal)
    c, d, k0, levels, _ = ref_case(16)
    k = _leading_block(k0, d.nxyz0[0]) if prec_kind == 2 else k0
    xr, rr, xg, rg = _fgmres_pair(S, k, prec_kind, restart=restart)
    assert rg.converged == rr["converged"]
    assert abs(rg.iterations - rr["iterations"]) <= 1
    n = min(len(rg.residual_history), len(rr["residual_history"]))
    h_g, h_r = rg.residual_history[:n], rr["residual_history"][:n]
    assert np.all(np.abs(h_g - h_r) <= 1e-6 * np.maximum(h_r, 1e-300) + 1e-14)
    if rr["converged"]:
        assert rg.final_relative_residual <= 1e-8


def test_jacobi_zero_diagonal_raises(S):
    # inv_diagonal on the saddle-point K0 (zero pressure diagonal) -> ZeroDiagonal
    c, d, k0, levels, _ = ref_case(8)
    K = S.SparseMatrix.from_csr(k0)
    with pytest.raises(O.OracleError):
        O.ref_fgmres(O.RefMat.from_csr(k0), np.ones(k0.nrows), np.zeros(k0.nrows), 2,
                     O.RefMat.from_csr(k0))
    with pytest.raises(S.ZeroDiagonal):
        S.fgmres(K, np.ones(k0.nrows), np.zeros(k0.nrows), K)


def test_fgmres_iteration_cap(S):
    c, d, k0, levels, _ = ref_case(16)
    xr, rr, xg, rg = _fgmres_pair(S, k0, 0, tol=1e-14, max_iters=7, restart=4)
    assert not rr["converged"] and not rg.converged
    assert rg.iterations == rr["iterations"] == 7
    assert abs(rg.final_relative_residual - rr["final_relative_residual"]) <= \
        1e-6 * rr["final_relative_residual"]


def test_fgmres_zero_rhs(S):
    c, d, k0, levels, _ = ref_case(8)
    xr, rr, xg, rg = _fgmres_pair(S, k0, 0, b=np.zeros(k0.nrows))
    assert rg.converged == rr["converged"]
    assert rg.iterations == rr["iterations"]
    assert np.array_equal(xg, xr)


def test_fgmres_exact_preconditioner_one_step(S):
    # one Vanka patch covering the whole system inverts K exactly: FGMRES
    # converges in one step (tests/test_krylov.cpp semantics, happy breakdown)
    a = np.array([[4.0, 1.0, 0.0, 1.0], [1.0, 3.0, 0.0, -1.0], [0.0, 0.0, 5.0, 2.0],
                  [1.0, -1.0, 2.0, 0.0]])
    r, cc = np.nonzero(a)
    k = O.RefMat.from_triplets(4, 4, r, cc, a[r, cc]).csr()
    K = S.SparseMatrix.from_csr(k)
    p = S.Patches.from_lists([0, 1], [3], [0, 3], [0, 1, 2], [2])
    f = S.factor_patches(K, p, 3)
    b = np.array([1.0, 2.0, 3.0, 4.0])
    x = np.zeros(4)
    rep = S.fgmres(K, b, x, f, S.FgmresOptions(tol=1e-12, max_iters=10, restart=5))
    rk = O.RefMat.from_csr(k)
    pp = O.Patches(*[np.asarray(v, dtype=np.int32) for v in ([0, 1], [3], [0, 3], [0, 1, 2], [2])])
    xr, rr = O.ref_fgmres(rk, b, np.zeros(4), 1, O.RefVanka.from_patches(rk, pp, 3), 1e-12, 10, 5)
    assert rep.converged and rr["converged"]
    assert rep.iterations == rr["iterations"] <= 2
    assert np.allclose(x, np.linalg.solve(a, b), rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------ DC variants --
def _device_dc(S, k0, nxyz0, levels, conf):
    K0 = S.SparseMatrix.from_csr(k0)
    lv = [(S.SparseMatrix.from_csr(k), S.SparseMatrix.from_csr(p) if p is not None else None,
           nxyz) for k, p, nxyz in levels]
    cfg = S.SolverConfig(variant=conf.get("variant", 0), nu1=conf["nu1"], nu2=conf["nu2"],
                         gamma=conf.get("gamma", 1), restart=conf["restart"], tol=conf["tol"],
                         max_iters=conf["max_iters"], enclosed_flow=conf["enclosed_flow"])
    return K0, S.DCPreconditioner(K0, nxyz0, lv, cfg), cfg


@pytest.mark.parametrize("extra", [dict(variant=1), dict(variant=2), dict(gamma=2),
                                   dict(nu1=2, nu2=2)])
def test_dc_variants_match_reference(S, extra):
    c, d, k0, levels, conf = ref_case(32, cfg=extra)
    K0, dc, cfg = _device_dc(S, k0, d.nxyz0, levels, conf)
    r = O.splitmix64_uniform(k0.nrows)
    assert rel_inf(dc.apply(r), d.apply(r)) <= 1e-9
    x_ref, rep_ref = d.solve(c.rhs())
    x, rep = S.solve_stokes(K0, c.rhs(), dc, cfg)
    assert rep.converged == rep_ref["converged"]
    assert abs(rep.iterations - rep_ref["iterations"]) <= 1
    if rep_ref["converged"]:
        assert rep.final_relative_residual <= cfg.tol


# ------------------------------------------------- full size (config 2) --
@pytest.fixture(scope="module")
def config2():
    from paper_2306_06795_b200.cases import HostCase
    h = HostCase("cavity", False, "structured", 512)
    return h, h.k0()


@pytest.mark.slow
def test_config2_k0_spmv_vanka_fullsize(S, config2):
    h, k0 = config2
    rk = O.RefMat.from_csr(k0)
    K = S.SparseMatrix.from_csr(k0)
    x = O.splitmix64_uniform(k0.nrows)
    y = S.spmv(K, x)
    assert rel_inf(y, rk.spmv(x)) <= TOL
    rv = O.RefVanka.build(rk, *h.nxyz0)
    f = S.factor_patches(K, S.build_patches(K, *h.nxyz0), h.n_x0 + h.n_y0)
    d = S.apply_vanka(f, x)
    assert rel_inf(d, rv.apply(x)) <= TOL
    # linearity at full size: A(a x + b z) = a A x + b A z
    z = O.splitmix64_uniform(k0.nrows, seed=99)
    comb = 0.75 * x - 1.5 * z
    assert rel_inf(S.spmv(K, comb), 0.75 * y - 1.5 * S.spmv(K, z)) <= 1e-13
    assert rel_inf(S.apply_vanka(f, comb), 0.75 * d - 1.5 * S.apply_vanka(f, z)) <= 1e-12
    # run-to-run reproducibility (fixed-order, atomic-free scatter)
    assert np.array_equal(S.apply_vanka(f, x), d)
    assert np.array_equal(S.spmv(K, x), y)


@pytest.mark.slow
def test_config2_solve_fullsize(S, config2):
    h, k0 = config2
    cfg = S.SolverConfig(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500, enclosed_flow=True)
    K0, dc, _ = h.device(cfg)
    rhs = h.rhs()
    x, rep = S.solve_stokes(K0, rhs, dc, cfg)
    assert rep.converged and abs(rep.iterations - 38) <= 1
    assert rep.final_relative_residual <= 1e-8
    # the true residual, recomputed by the reference's own spmv
    res = rhs - O.RefMat.from_csr(k0).spmv(x)
    assert np.linalg.norm(res) / np.linalg.norm(rhs) <= 1.01e-8


# --------------------------------------- HO-AMG and Uzawa --
def _prec_pair(S, n, variant, sv=False, extra=None):
    from paper_2306_06795_b200.cases import HostCase
    conf = dict(variant=variant, nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500)
    conf.update(extra or {})
    c = O.RefCase.build("cavity", sv, "structured", n)
    conf["enclosed_flow"] = c.enclosed
    ref = O.RefPrec(c, conf)
    h = HostCase("cavity", sv, "structured", n)
    cfg = S.SolverConfig(variant=variant, nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500,
                         enclosed_flow=c.enclosed, **{k: v for k, v in (extra or {}).items()
                                                     if k in ("eta_u", "eta_p", "omega0")})
    if variant == 3:
        K0, prec = h.hoamg_device(cfg)
    else:
        K0, prec = h.uzawa_device(cfg)
    return c, ref, h, K0, prec, cfg


@pytest.mark.parametrize("variant,n,sv", [(3, 16, False), (3, 32, False), (4, 16, False),
                                          (4, 32, False), (4, 8, True)])
def test_hoamg_uzawa_match_reference(S, variant, n, sv):
    # HoAmgPreconditioner / UzawaPreconditioner (preconditioner.cpp:155-218)
    c, ref, h, K0, prec, cfg = _prec_pair(S, n, variant, sv)
    r = O.splitmix64_uniform(c.n0)
    assert rel_inf(prec.apply(r), ref.apply(r)) <= 1e-9
    x_ref, rep_ref = ref.solve(c.rhs())
    x, rep = S.solve_stokes(K0, c.rhs(), prec, cfg)
    assert rep.converged == rep_ref["converged"]
    assert abs(rep.iterations - rep_ref["iterations"]) <= 1
    if rep_ref["converged"]:
        assert rep.final_relative_residual <= cfg.tol
        assert rel_inf(x, x_ref) <= 1e-6
    # the C++ drop-in (gpu::HoAmgPreconditioner / gpu::UzawaPreconditioner)
    xd, repd = h.solve_dropin(variant=variant, nu=1, restart=30, tol=1e-8, max_iters=500)
    assert abs(repd["iterations"] - rep_ref["iterations"]) <= 1


def test_hoamg_refused_on_sv(S):
    from paper_2306_06795_b200.cases import HostCase
    c = O.RefCase.build("cavity", True, "structured", 8)
    with pytest.raises(O.OracleError):
        O.RefPrec(c, dict(variant=3, enclosed_flow=True))
    h = HostCase("cavity", True, "structured", 8)
    with pytest.raises(S.UnsupportedDiscretization):
        h.hoamg_device(S.SolverConfig(variant=3, enclosed_flow=True))
    K0, prec = h.hoamg_device(S.SolverConfig(variant=3, enclosed_flow=True, allow_sv_hoamg=True))
    assert prec.apply(np.ones(h.n0)).shape == (h.n0,)


def test_uzawa_scalar_tail(S, monkeypatch):
    # Uzawa's scalar V(2,2) cycles (A_x: three levels at n = 64) with the
    # cluster tail off, from level 1 on, and over the whole cycle: same
    # operator as the reference, fewer launches as the tail grows
    ctx = S.default_context()
    launches = {}
    for tail in ("0", "from1", "all"):
        monkeypatch.setenv("SAG_SCALAR_TAIL", "0" if tail == "0" else "1")
        monkeypatch.setenv("SAG_TAIL_ROWS", "5000" if tail == "from1" else "65536")
        c, ref, h, K0, prec, cfg = _prec_pair(S, 64, 4)
        r = O.splitmix64_uniform(c.n0)
        z = prec.apply(r)
        assert rel_inf(z, ref.apply(r)) <= 1e-9, tail
        l0 = ctx.launch_count()
        assert np.array_equal(z, prec.apply(r))
        launches[tail] = ctx.launch_count() - l0
    assert launches["all"] < launches["from1"] < launches["0"], launches


# ------------------------------------------ parameter scan --
def test_set_parameters_recaptures_solve_graph(S):
    # parameter_scan (preconditioner.cpp:261-277): one preconditioner, its
    # (eta_u, eta_p, omega0) changed between solves. Every scan point must
    # solve with its own parameters -- the whole-solve CUDA graph captured for
    # the previous point bakes them into kernel arguments and must be dropped.
    c, d, k0, levels, conf = ref_case(16)
    K0, dc, cfg = _device_dc(S, k0, d.nxyz0, levels, conf)
    rhs = c.rhs()
    x1, rep1 = S.solve_stokes(K0, rhs, dc, cfg)
    points = [(0.5, 0.5, 0.8), (0.75, 0.75, 1.0), (1.0, 1.0, 1.0)]
    for eu, ep, om in points:
        dc.set_parameters(eu, ep, om)
        x, rep = S.solve_stokes(K0, rhs, dc, cfg)
        K0f, fresh, _ = _device_dc(S, k0, d.nxyz0, levels, conf)
        fresh.set_parameters(eu, ep, om)
        xf, repf = S.solve_stokes(K0f, rhs, fresh, cfg)
        assert rep.iterations == repf.iterations, (eu, ep, om)
        assert np.array_equal(x, xf), (eu, ep, om)
        d.set_parameters(eu, ep, om)
        _, rr = d.solve(rhs)
        assert abs(rep.iterations - rr["iterations"]) <= 1, (eu, ep, om, rr["iterations"])
    # back at the first point: the first solve exactly
    assert np.array_equal(x, x1) and rep.iterations == rep1.iterations
