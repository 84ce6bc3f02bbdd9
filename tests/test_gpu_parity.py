"""GPU parity of the sm_100a path against the reference (oracle/_ref) and the
C restatement (oracle/), through the C-ABI (include/sag.h).

Tolerances (north_star): Vanka apply and SpMV agree to 1e-12 relative,
measured normwise ||y_gpu - y_ref||_inf / ||y_ref||_inf; FGMRES iteration
counts agree within +-1 and both final relative residuals are <= rtol.
Integer work (patch sets) and the stored factor payload (u_hat, b_hat, s_inv,
weights: same elimination order, explicit round-to-nearest ops) are bitwise.
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


@pytest.mark.parametrize("n", [8, 64])
def test_spmv_all_levels(S, n):
    c, d, k0, levels, _ = ref_case(n)
    mats = [k0] + [l[0] for l in levels] + [l[1] for l in levels if l[1] is not None]
    for m in mats:
        x = O.splitmix64_uniform(m.ncols)
        ref = O.RefMat.from_csr(m).spmv(x)
        got = S.spmv(S.SparseMatrix.from_csr(m), x)
        assert rel_inf(got, ref) <= TOL
        # restatement is bitwise the reference
        assert np.array_equal(O.Oracle.spmv(m, x), ref)


def test_spmv_hand_product(S):
    # tests/test_sparse.cpp:37-45
    m = O.RefMat.from_triplets(3, 3, [0, 0, 1, 1, 2, 2], [0, 1, 1, 2, 0, 2],
                               [1, 2, 3, 4, 5, 6]).csr()
    y = S.spmv(S.SparseMatrix.from_csr(m), np.array([1.0, 2.0, 3.0]))
    assert np.array_equal(y, [5.0, 18.0, 23.0])


@pytest.mark.parametrize("n", [8, 64])
def test_build_patches_exact(S, n):
    c, d, k0, levels, _ = ref_case(n)
    for k, nxyz in [(k0, d.nxyz0)] + [(l[0], l[2]) for l in levels[:-1]]:
        ref = O.ref_build_patches(O.RefMat.from_csr(k), *nxyz)
        got = S.build_patches(S.SparseMatrix.from_csr(k), *nxyz).export()
        assert np.array_equal(got.pressure_ptr, ref.pptr)
        assert np.array_equal(got.pressure, ref.pidx)
        assert np.array_equal(got.velocity_ptr, ref.vptr)
        assert np.array_equal(got.velocity, ref.vidx)
        assert np.array_equal(got.nx, ref.nx)


def test_build_patches_sv_triples(S):
    c, d, k0, levels, _ = ref_case(4, sv=True, cfg=dict(omega0=0.78, eta_p=2.68))
    ref = O.ref_build_patches(O.RefMat.from_csr(k0), *d.nxyz0, sv_triples=True)
    got = S.build_patches(S.SparseMatrix.from_csr(k0), *d.nxyz0, sv_triples=True).export()
    assert np.array_equal(got.velocity_ptr, ref.vptr)
    assert np.array_equal(got.velocity, ref.vidx)
    assert np.array_equal(got.pressure, ref.pidx)
    assert np.array_equal(got.nx, ref.nx)
    assert int(np.diff(ref.vptr).max() + 3) == 15  # tests/test_vanka.cpp:81-96


@pytest.mark.parametrize("n", [8, 64])
def test_factor_payload_bitwise(S, n):
    c, d, k0, levels, _ = ref_case(n)
    for k, nxyz in [(k0, d.nxyz0)] + [(l[0], l[2]) for l in levels[:-1]]:
        rk = O.RefMat.from_csr(k)
        rv = O.RefVanka.build(rk, *nxyz)
        want = rv.factors()
        K = S.SparseMatrix.from_csr(k)
        p = S.build_patches(K, *nxyz)
        f = S.factor_patches(K, p, nxyz[0] + nxyz[1])
        got = f.export(p.export())
        for key in ("uhat", "bhat", "sinv", "weights"):
            assert np.array_equal(got[key], want[key]), key
        assert f.a_factor_bytes == want["a_factor_bytes"]
        assert f.aux_bytes == want["aux_bytes"]
        assert f.dense_inverse_bytes == want["dense_inverse_bytes"]


@pytest.mark.parametrize("n", [8, 64])
def test_apply_vanka_parity(S, n):
    c, d, k0, levels, _ = ref_case(n)
    for k, nxyz in [(k0, d.nxyz0)] + [(l[0], l[2]) for l in levels[:-1]]:
        rv = O.RefVanka.build(O.RefMat.from_csr(k), *nxyz)
        K = S.SparseMatrix.from_csr(k)
        f = S.factor_patches(K, S.build_patches(K, *nxyz), nxyz[0] + nxyz[1])
        r = O.splitmix64_uniform(k.nrows)
        assert rel_inf(S.apply_vanka(f, r), rv.apply(r)) <= TOL
        z = S.apply_vanka(f, np.zeros(k.nrows))
        assert np.all(z == 0.0)  # tests/test_vanka.cpp:264-271


@pytest.mark.parametrize("mode,sv,stages", [("device", False, 0), ("pinned", False, 0),
                                             ("pinned", False, 1), ("pinned", False, 3),
                                             ("pinned", False, 40), ("pageable", False, 0),
                                             ("pinned", True, 0), ("pinned", True, 5)])
def test_vanka_spmv_step(S, monkeypatch, mode, sv, stages):
    """sag_vanka_spmv equals spmv + apply_vanka of the reference with device
    buffers (x read once), pageable host buffers (staged, y copied back under
    the sweep) and pinned host buffers -- the pipelined step: x arrives in
    stages, row ranges of y, patch windows and dof ranges of delta run and
    leave as their inputs arrive -- bitwise the unpipelined results, for any
    stage count, one-class (TH) and multi-class (SV: fixed-shape + sub-warp +
    32-lane) levels."""
    import torch
    if stages:
        monkeypatch.setenv("SAG_STEP_STAGES", str(stages))
    if sv:
        c = O.RefCase.build("cavity", True, "structured", 64)  # sub-warp classes
        k0 = c.k0().csr()
        nxyz = (c.n_x0, c.n_y0, c.n_p0)
    else:
        c, d, k0, levels, _ = ref_case(64)
        nxyz = d.nxyz0
    rv = O.RefVanka.build(O.RefMat.from_csr(k0), *nxyz, sv_triples=sv)
    K = S.SparseMatrix.from_csr(k0)
    f = S.factor_patches(K, S.build_patches(K, *nxyz, sv_triples=sv), nxyz[0] + nxyz[1])
    x = O.splitmix64_uniform(k0.nrows)
    if mode == "device":
        xt = torch.from_numpy(x).cuda()
        dt, yt = S.vanka_spmv_step(f, K, xt)
        dl, y = dt.cpu().numpy(), yt.cpu().numpy()
    elif mode == "pageable":
        dl, y = S.vanka_spmv_step(f, K, x.copy())
    else:
        xh = torch.from_numpy(x).pin_memory().numpy()
        dh = torch.empty(k0.nrows, dtype=torch.float64).pin_memory().numpy()
        yh = torch.empty(k0.nrows, dtype=torch.float64).pin_memory().numpy()
        dh[:] = np.nan
        yh[:] = np.nan
        dl, y = S.vanka_spmv_step(f, K, xh, dh, yh)
        assert dl is dh and y is yh
        plan = S.vanka_step_plan(f)
        want = stages if stages else 8
        assert plan["stages"] == (want if want >= 2 else 0), plan
        if want >= 2:  # a strip-ordered numbering: a handful of ranges per stage
            assert 0 < plan["ranges"] <= 64 * want and plan["patch_windows"] >= 1, plan
            # forced by SAG_STEP_STAGES; by default timed against the plain step
            # at the first call (either may win on a case this small)
            if not stages:
                assert plan["choice"] in ("pipelined", "plain"), plan
                assert plan["plain_ms"] > 0 and plan["pipelined_ms"] > 0
            dl2, y2 = S.vanka_spmv_step(f, K, xh, dh, yh)  # the cached plan again
            assert np.array_equal(dl2, dl) and np.array_equal(y2, y)
    assert rel_inf(y, O.RefMat.from_csr(k0).spmv(x)) <= TOL
    assert rel_inf(dl, rv.apply(x)) <= TOL
    assert np.array_equal(dl, S.apply_vanka(f, x)) and np.array_equal(y, S.spmv(K, x))


def test_apply_vanka_sv(S):
    c, d, k0, levels, _ = ref_case(8, sv=True, cfg=dict(omega0=0.78, eta_p=2.68))
    rv = O.RefVanka.build(O.RefMat.from_csr(k0), *d.nxyz0, sv_triples=True)
    K = S.SparseMatrix.from_csr(k0)
    f = S.factor_patches(K, S.build_patches(K, *d.nxyz0, sv_triples=True),
                         d.nxyz0[0] + d.nxyz0[1])
    r = O.splitmix64_uniform(k0.nrows)
    assert rel_inf(S.apply_vanka(f, r), rv.apply(r)) <= TOL


def test_hand_factored_patch(S):
    # tests/test_vanka.cpp:98-113
    k = O.RefMat.from_triplets(3, 3, [0, 0, 1, 2], [0, 2, 1, 0], [1, 1, 1, 1]).csr()
    K = S.SparseMatrix.from_csr(k)
    p = S.Patches.from_lists([0, 1], [2], [0, 2], [0, 1], [1])
    f = S.factor_patches(K, p, 2)
    assert f.export(p.export())["sinv"][0] == -1.0
    assert np.allclose(S.apply_vanka(f, np.array([1.0, 0.0, 1.0])), [1.0, 0.0, 0.0])


def test_block_lu_random_patches(S):
    # tests/test_vanka.cpp:115-155: block-LU patch solve == dense solve, 200 trials
    rng = np.random.default_rng(42)
    worst = 0.0
    for _ in range(200):
        ax = 0.3 * rng.uniform(-1, 1, (5, 5))
        ay = 0.3 * rng.uniform(-1, 1, (5, 5))
        A = np.zeros((12, 12))
        A[:5, :5] = 0.5 * (ax + ax.T) + 4 * np.eye(5)
        A[5:10, 5:10] = 0.5 * (ay + ay.T) + 4 * np.eye(5)
        B = rng.uniform(-1, 1, (2, 10))
        A[10:, :10] = B
        A[:10, 10:] = B.T
        r, cc = np.nonzero(A)
        k = O.RefMat.from_triplets(12, 12, r, cc, A[r, cc]).csr()
        K = S.SparseMatrix.from_csr(k)
        p = S.Patches.from_lists([0, 2], [10, 11], [0, 10], list(range(10)), [5])
        f = S.factor_patches(K, p, 10)
        b = rng.uniform(-1, 1, 12)
        x = S.apply_vanka(f, b)
        ref = np.linalg.solve(A, b)
        worst = max(worst, float(np.max(np.abs(x - ref) / np.maximum(1.0, np.abs(ref)))))
    assert worst <= 1e-10


def _saddle_blocks(rng, sizes):
    """Independent symmetric saddle-point blocks, dofs ordered [x | y | p]
    over all blocks; one Vanka patch per block (its own dofs)."""
    nxs = [a for a, _ in sizes]
    nys = [b for _, b in sizes]
    ox = np.concatenate([[0], np.cumsum(nxs)])
    oy = ox[-1] + np.concatenate([[0], np.cumsum(nys)])
    n_u = int(oy[-1])
    n = n_u + len(sizes)
    rr, cc, vv = [], [], []
    vidx, vptr = [], [0]
    for b, (mx, my) in enumerate(sizes):
        xs = np.arange(ox[b], ox[b] + mx)
        ys = np.arange(oy[b], oy[b] + my)
        pr = n_u + b
        for dofs in (xs, ys):
            m = len(dofs)
            a = 0.3 * rng.uniform(-1, 1, (m, m))
            a = 0.5 * (a + a.T) + 4 * np.eye(m)
            i, j = np.meshgrid(dofs, dofs, indexing="ij")
            rr += list(i.ravel()); cc += list(j.ravel()); vv += list(a.ravel())
        bu = rng.uniform(-1, 1, mx + my)
        vel = np.concatenate([xs, ys])
        rr += [pr] * len(vel) + list(vel); cc += list(vel) + [pr] * len(vel)
        vv += list(bu) + list(bu)
        vidx += list(vel)
        vptr.append(len(vidx))
    k = O.RefMat.from_triplets(n, n, rr, cc, vv)
    pptr = list(range(len(sizes) + 1))
    pidx = [n_u + b for b in range(len(sizes))]
    return k, n_u, (pptr, pidx, vptr, vidx, nxs)


@pytest.mark.parametrize("big", [False, True])
def test_apply_vanka_many_patches_per_warp(S, big):
    # thousands of patches (several per warp: ring reuse, the paired
    # (A_x, A_y) layout, zero-padded when nx != ny), plus m = 31 / 32
    # patches; with `big` one 40-dof component puts the level on the
    # two-rows-per-lane paired kernel (m + np <= 64)
    rng = np.random.default_rng(7)
    sizes = [(m, m) for m in rng.integers(2, 32, 6000)] + [(5, 7), (9, 4), (32, 32), (31, 31)]
    if big:
        sizes.append((40, 40))
    rng.shuffle(sizes)
    k, n_u, lists = _saddle_blocks(rng, sizes)
    pp = O.Patches(*[np.asarray(a, dtype=np.int32) for a in lists])
    rv = O.RefVanka.from_patches(k, pp, n_u)
    K = S.SparseMatrix.from_csr(k.csr())
    f = S.factor_patches(K, S.Patches.from_lists(*lists), n_u)
    want = rv.factors()
    got = f.export(S.Patches.from_lists(*lists).export())
    for key in ("uhat", "bhat", "sinv"):
        assert np.array_equal(got[key], want[key]), key
    r = O.splitmix64_uniform(k.csr_shape()[0])
    assert rel_inf(S.apply_vanka(f, r), rv.apply(r)) <= TOL


@pytest.mark.parametrize("lo,hi", [(2, 8), (8, 16)])
def test_apply_vanka_subwarp_classes(S, lo, hi):
    # >= 4096 small paired patches form their own class and run on the
    # sub-warp kernel (m + np <= 8: four patches per warp; <= 16: two)
    rng = np.random.default_rng(11)
    sizes = [(int(m), int(m)) for m in rng.integers(lo - 1, hi, 9000)]
    sizes += [(int(a), int(b)) for a, b in rng.integers(max(lo - 2, 1), hi - 1, (500, 2))]
    rng.shuffle(sizes)
    k, n_u, lists = _saddle_blocks(rng, sizes)
    pp = O.Patches(*[np.asarray(a, dtype=np.int32) for a in lists])
    rv = O.RefVanka.from_patches(k, pp, n_u)
    K = S.SparseMatrix.from_csr(k.csr())
    f = S.factor_patches(K, S.Patches.from_lists(*lists), n_u)
    r = O.splitmix64_uniform(k.csr_shape()[0])
    assert rel_inf(S.apply_vanka(f, r), rv.apply(r)) <= TOL


def test_apply_vanka_sv_subwarp(S):
    # SV fine level (element triples, m + np = 9): 6144 patches at n = 32 run
    # on the two-patches-per-warp kernel
    c, d, k0, levels, _ = ref_case(32, sv=True, cfg=dict(omega0=0.78, eta_p=2.68))
    rv = O.RefVanka.build(O.RefMat.from_csr(k0), *d.nxyz0, sv_triples=True)
    K = S.SparseMatrix.from_csr(k0)
    f = S.factor_patches(K, S.build_patches(K, *d.nxyz0, sv_triples=True),
                         d.nxyz0[0] + d.nxyz0[1])
    r = O.splitmix64_uniform(k0.nrows)
    assert rel_inf(S.apply_vanka(f, r), rv.apply(r)) <= TOL
    x0 = np.sin(0.1 * np.arange(k0.nrows))
    want = rv.relax(x0, r, 1, 2, 0.78)
    got = S.vanka_relax(K, f, x0.copy(), r, 1, 2, 0.78)
    assert rel_inf(got, want) <= 1e-11


def test_apply_vanka_sv_fixed_shape(S, monkeypatch):
    # the interior element triples (nx = ny = 6, np = 3) run on the
    # fixed-shape kernel: x_p = S^-1 (b_p + U_hat^T b_u) instead of the
    # stored b_hat, so the sweep is within rounding (1e-14) of the one with
    # that class switched off and within 1e-12 of the reference; the factor
    # payload (b_hat rebuilt by the export) is bitwise the reference's
    c, d, k0, levels, _ = ref_case(32, sv=True, cfg=dict(omega0=0.78, eta_p=2.68))
    rv = O.RefVanka.build(O.RefMat.from_csr(k0), *d.nxyz0, sv_triples=True)
    K = S.SparseMatrix.from_csr(k0)
    p = S.build_patches(K, *d.nxyz0, sv_triples=True)
    f = S.factor_patches(K, p, d.nxyz0[0] + d.nxyz0[1])
    kinds = [k[0] for k in f.classes()]
    assert any(k.startswith("vanka_fixed_kernel") for k in kinds), kinds
    r = O.splitmix64_uniform(k0.nrows)
    z = S.apply_vanka(f, r)
    assert rel_inf(z, rv.apply(r)) <= TOL
    monkeypatch.setenv("SAG_VANKA_FIXED", "0")
    f0 = S.factor_patches(K, p, d.nxyz0[0] + d.nxyz0[1])
    assert not any(k[0].startswith("vanka_fixed_kernel") for k in f0.classes())
    assert rel_inf(z, S.apply_vanka(f0, r)) <= 1e-14
    got, want = f.export(p.export()), rv.factors()
    for key in ("uhat", "bhat", "sinv", "weights"):
        assert np.array_equal(got[key], want[key]), key


def test_singular_patch_raises(S):
    k = O.RefMat.from_triplets(3, 3, [0, 1, 2], [2, 1, 0], [1.0, 1.0, 1.0]).csr()
    K = S.SparseMatrix.from_csr(k)
    p = S.Patches.from_lists([0, 1], [2], [0, 2], [0, 1], [1])
    with pytest.raises(S.SingularPatch):
        S.factor_patches(K, p, 2)


@pytest.mark.parametrize("mode,sweeps,omega", [(0, 1, 1.0), (0, 2, 1.0), (1, 3, 0.78)])
def test_vanka_relax_parity(S, mode, sweeps, omega):
    c, d, k0, levels, _ = ref_case(32)
    rk = O.RefMat.from_csr(k0)
    rv = O.RefVanka.build(rk, *d.nxyz0)
    K = S.SparseMatrix.from_csr(k0)
    f = S.factor_patches(K, S.build_patches(K, *d.nxyz0), d.nxyz0[0] + d.nxyz0[1])
    x0 = np.sin(0.1 * np.arange(k0.nrows))
    b = O.splitmix64_uniform(k0.nrows)
    want = rv.relax(x0, b, mode, sweeps, omega)
    got = S.vanka_relax(K, f, x0.copy(), b, mode, sweeps, omega)
    assert rel_inf(got, want) <= 1e-11


def test_relax_fixed_point(S):
    # tests/test_vanka.cpp:214-233: b = K x => relaxation leaves x unchanged
    c, d, k0, levels, _ = ref_case(8)
    K = S.SparseMatrix.from_csr(k0)
    f = S.factor_patches(K, S.build_patches(K, *d.nxyz0), d.nxyz0[0] + d.nxyz0[1])
    x = np.sin(0.1 * np.arange(k0.nrows))
    b = O.RefMat.from_csr(k0).spmv(x)
    x1 = S.vanka_relax(K, f, x.copy(), b, 0, 2)
    assert np.allclose(x1, x, rtol=1e-12, atol=1e-12)
    x2 = S.vanka_relax(K, f, x.copy(), b, 1, 3, 0.0)
    assert np.array_equal(x2, x)


def _device_dc(S, k0, nxyz0, levels, conf, sv=False):
    K0 = S.SparseMatrix.from_csr(k0)
    lv = [(S.SparseMatrix.from_csr(k), S.SparseMatrix.from_csr(p) if p is not None else None,
           nxyz) for k, p, nxyz in levels]
    cfg = S.SolverConfig(nu1=conf["nu1"], nu2=conf["nu2"], restart=conf["restart"],
                         tol=conf["tol"], max_iters=conf["max_iters"],
                         enclosed_flow=conf["enclosed_flow"], eta_u=conf.get("eta_u", 1.0),
                         eta_p=conf.get("eta_p", 1.0), omega0=conf.get("omega0", 1.0))
    return K0, S.DCPreconditioner(K0, nxyz0, lv, cfg, sv=sv), cfg


@pytest.mark.parametrize("n", [8, 32, 64])
def test_dc_apply_parity(S, n):
    c, d, k0, levels, conf = ref_case(n)
    K0, dc, cfg = _device_dc(S, k0, d.nxyz0, levels, conf)
    r = O.splitmix64_uniform(k0.nrows)
    want = d.apply(r)
    got = dc.apply(r)
    assert rel_inf(got, want) <= 1e-9


@pytest.mark.parametrize("n,its", [(32, 20), (64, 24)])
def test_solve_stokes_cavity(S, n, its):
    c, d, k0, levels, conf = ref_case(n)
    K0, dc, cfg = _device_dc(S, k0, d.nxyz0, levels, conf)
    rhs = c.rhs()
    x_ref, rep_ref = d.solve(rhs)
    assert rep_ref["iterations"] == its
    x, rep = S.solve_stokes(K0, rhs, dc, cfg)
    assert rep.converged
    assert abs(rep.iterations - rep_ref["iterations"]) <= 1
    assert rep.final_relative_residual <= cfg.tol
    assert len(rep.residual_history) == rep.iterations + 1
    assert rel_inf(x, x_ref) <= 1e-6


# ----------------------------------------------------- SV (config 3 family)
def _host_device(S, case_kw, conf):
    from paper_2306_06795_b200.cases import HostCase
    h = HostCase(**case_kw)
    cfg = S.SolverConfig(nu1=conf["nu1"], nu2=conf["nu2"], restart=conf["restart"],
                         tol=conf["tol"], max_iters=conf["max_iters"],
                         enclosed_flow=conf["enclosed_flow"], eta_u=conf.get("eta_u", 1.0),
                         eta_p=conf.get("eta_p", 1.0), omega0=conf.get("omega0", 1.0))
    K0, dc, _ = h.device(cfg)
    return h, K0, dc, cfg


@pytest.mark.parametrize("n", [4, 8])
def test_sv_dc_apply_and_solve(S, n):
    # Scott-Vogelius: 3-seed element patches, stationary fine relaxation,
    # pressure duplication / mass-projection transfer (transfer.cpp:18-53)
    conf = dict(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500, enclosed_flow=True,
                omega0=0.78, eta_u=1.0, eta_p=2.68)
    c, d, k0, levels, _ = ref_case(n, sv=True, cfg=conf)
    h, K0, dc, cfg = _host_device(S, dict(problem="cavity", sv=True, n=n), conf)
    assert h.n0 == c.n0
    r = O.splitmix64_uniform(c.n0)
    assert rel_inf(dc.apply(r), d.apply(r)) <= 1e-8
    x_ref, rep_ref = d.solve(c.rhs())
    x, rep = S.solve_stokes(K0, c.rhs(), dc, cfg)
    assert rep.converged and rep.final_relative_residual <= cfg.tol
    assert abs(rep.iterations - rep_ref["iterations"]) <= 1


def test_unstructured_forced_solve(S, tmp_path):
    # BASELINE config 4 family: jittered Delaunay mesh, zero velocity, body force
    from paper_2306_06795_b200 import meshgen
    path = meshgen.write_mesh(str(tmp_path / "m.json"), 24, seed=7, jitter=0.3)
    k1, k2 = meshgen.force_wavenumbers()
    c = O.RefCase.mesh_forced(path, k1, k2)
    conf = dict(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500, enclosed_flow=True)
    d = O.RefDC(c, conf)
    h, K0, dc, cfg = _host_device(S, dict(problem="cavity", mesh_kind="file_forced",
                                          mesh_path=path, k1=k1, k2=k2), conf)
    assert h.n0 == c.n0 and np.array_equal(h.rhs(), c.rhs())
    r = O.splitmix64_uniform(c.n0)
    assert rel_inf(dc.apply(r), d.apply(r)) <= 1e-9
    x_ref, rep_ref = d.solve(c.rhs())
    x, rep = S.solve_stokes(K0, c.rhs(), dc, cfg)
    assert rep.converged and rep.final_relative_residual <= cfg.tol
    assert abs(rep.iterations - rep_ref["iterations"]) <= 1


def test_dropin_cpp_adapter_solve(S):
    # the C++ drop-in (stokesamg::gpu::DCPreconditioner + gpu::solve_stokes)
    # against the reference's own DCPreconditioner + solve_stokes (config 1)
    from paper_2306_06795_b200.cases import HostCase
    c, d, k0, levels, conf = ref_case(64)
    h = HostCase("cavity", False, "structured", 64)
    x, rep = h.solve_dropin(nu=1, restart=30, tol=1e-8, max_iters=500)
    x_ref, rep_ref = d.solve(c.rhs())
    assert rep["converged"] and abs(rep["iterations"] - rep_ref["iterations"]) <= 1
    assert rep["final_relative_residual"] <= 1e-8
    assert rel_inf(x, x_ref) <= 1e-6


@pytest.mark.parametrize("tail", ["0", "1"])
def test_sv_scalar_tail(S, monkeypatch, tail):
    # the mass projection's scalar V(2,2) cycles with their small levels as one
    # cluster launch (here the whole two-level cycle) against the per-kernel
    # path and the reference
    conf = dict(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500, enclosed_flow=True,
                omega0=0.78, eta_u=1.0, eta_p=2.68)
    c, d, k0, levels, _ = ref_case(64, sv=True, cfg=conf)
    monkeypatch.setenv("SAG_SCALAR_TAIL", tail)
    h, K0, dc, cfg = _host_device(S, dict(problem="cavity", sv=True, n=64), conf)
    r = O.splitmix64_uniform(c.n0)
    z = dc.apply(r)
    assert rel_inf(z, d.apply(r)) <= 1e-8
    assert np.array_equal(z, dc.apply(r))          # deterministic
    x, rep = S.solve_stokes(K0, c.rhs(), dc, cfg)
    assert rep.converged and rep.final_relative_residual <= cfg.tol
    assert abs(rep.iterations - d.solve(c.rhs())[1]["iterations"]) <= 1


@pytest.mark.parametrize("n,tail_rows,ngl", [(32, None, 1), (64, None, 1), (64, "300", 2)])
def test_sv_projection_one_launch(S, monkeypatch, n, tail_rows, ngl):
    # transfer.cpp:18-37 (FGMRES(20) to 1e-12 on Mcg, scalar V(2,2) cycle) as one
    # persistent launch (sv_project_kernel: grid levels in global memory behind
    # grid barriers, the small levels in cluster 0) against the multi-launch
    # path and the reference; tail_rows forces two grid levels
    conf = dict(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500, enclosed_flow=True,
                omega0=0.78, eta_u=1.0, eta_p=2.68)
    c, d, k0, levels, _ = ref_case(n, sv=True, cfg=conf)
    r = O.splitmix64_uniform(c.n0)
    zref = d.apply(r)
    if tail_rows:
        monkeypatch.setenv("SAG_TAIL_ROWS", tail_rows)
    out = {}
    for fused in ("0", "1"):
        monkeypatch.setenv("SAG_PROJ_FUSED", fused)
        h, K0, dc, cfg = _host_device(S, dict(problem="cavity", sv=True, n=n), conf)
        info = dc.info()
        assert info["proj_fused"] == (fused == "1")
        if fused == "1":
            assert info["proj_grid_levels"] == ngl and info["proj_workers"] > 0
        z = dc.apply(r)
        assert rel_inf(z, zref) <= 1e-8
        assert np.array_equal(z, dc.apply(r))          # deterministic
        x, rep = S.solve_stokes(K0, c.rhs(), dc, cfg)
        assert rep.converged and rep.final_relative_residual <= cfg.tol
        out[fused] = (z, x, rep.iterations)
    assert rel_inf(out["1"][0], out["0"][0]) <= 1e-10
    assert abs(out["1"][2] - out["0"][2]) <= 1
    assert abs(out["1"][2] - d.solve(c.rhs())[1]["iterations"]) <= 1


def test_vanka_spmv_step_any_numbering(S):
    """The pipelined step's plan is derived from the operator alone: with the
    dofs of each block (x, y, p) randomly renumbered the stages fragment, the
    plan collapses to the plain step, and the results stay bitwise those of
    apply_vanka + spmv (and within 1e-12 of the reference on the permuted
    operator)."""
    import torch
    c, d, k0, levels, _ = ref_case(32)
    nx, ny, npp = d.nxyz0
    n = k0.nrows
    rng = np.random.default_rng(11)
    perm = np.concatenate([rng.permutation(nx), nx + rng.permutation(ny),
                           nx + ny + rng.permutation(npp)])      # new -> old
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    rp, ci, v = np.asarray(k0.rp), np.asarray(k0.ci), np.asarray(k0.v)
    rows_new, cols_new, vals = [], [], []
    for r_new in range(n):
        r_old = perm[r_new]
        cc = inv[ci[rp[r_old]:rp[r_old + 1]]]
        o = np.argsort(cc, kind="stable")
        rows_new.append(len(cc))
        cols_new.append(cc[o])
        vals.append(v[rp[r_old]:rp[r_old + 1]][o])
    rp2 = np.concatenate([[0], np.cumsum(rows_new)]).astype(np.int32)
    kp = O.Csr(n, n, rp2, np.concatenate(cols_new).astype(np.int32), np.concatenate(vals))
    K = S.SparseMatrix.from_csr(kp)
    f = S.factor_patches(K, S.build_patches(K, nx, ny, npp), nx + ny)
    rv = O.RefVanka.build(O.RefMat.from_csr(kp), nx, ny, npp)
    x = O.splitmix64_uniform(n)
    xh = torch.from_numpy(x).pin_memory().numpy()
    dh = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    yh = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    dl, y = S.vanka_spmv_step(f, K, xh, dh, yh)
    plan = S.vanka_step_plan(f)
    assert plan["stages"] in (0, 8) and plan["choice"] != "untimed" or plan["stages"] == 0, plan
    assert np.array_equal(dl, S.apply_vanka(f, x)) and np.array_equal(y, S.spmv(K, x))
    assert rel_inf(y, O.RefMat.from_csr(kp).spmv(x)) <= TOL
    assert rel_inf(dl, rv.apply(x)) <= TOL
