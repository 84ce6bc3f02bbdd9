"""GPU: the reference's hot-path known-answer tests (KAT table)
re-run through the C-ABI, with the reference's own oracles -- dense
restatements, exact invariants -- as the checkers:

* tests/test_vanka.cpp:157-185  PoU exact + assembled Vanka operator vs the
  dense sum_i V_i^T W (V_i K V_i^T)^-1 V_i
* tests/test_vanka.cpp:187-194  storage accounting
* tests/test_vanka.cpp:196-212  one patch covering the system = K^-1
* tests/test_vanka.cpp:244-262  stationary relaxation contracts by (1 - omega)^4
* tests/test_preconditioner.cpp:96-120  relaxation-unit counters per variant
* tests/test_preconditioner.cpp:122-138  DC-LO iteration counts independent of eta
* tests/test_preconditioner.cpp:220-238  enclosed flow: converges, mean p = 0
* tests/acceptance.cpp:69-116   jittered 14 x 14 TH patches (seed 99) vs dense
* tests/acceptance.cpp:153-205  PoU exact on every hierarchy level
"""
import numpy as np
import pytest

import oracle as O
from conftest import ref_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2306_06795_b200 as S
    return S


def dense_vanka(k, pl, n):
    """sum_i V_i^T W (V_i K V_i^T)^-1 V_i with W = 1 / multiplicity."""
    kd = k.to_scipy().toarray()
    mult = np.zeros(n)
    sets = []
    for i in range(len(pl.pressure_ptr) - 1):
        d = np.concatenate([pl.velocity[pl.velocity_ptr[i]:pl.velocity_ptr[i + 1]],
                            pl.pressure[pl.pressure_ptr[i]:pl.pressure_ptr[i + 1]]])
        sets.append(d)
        mult[d] += 1
    w = np.divide(1.0, mult, out=np.zeros(n), where=mult > 0)
    m = np.zeros((n, n))
    for d in sets:
        m[np.ix_(d, d)] += np.diag(w[d]) @ np.linalg.inv(kd[np.ix_(d, d)])
    return m, mult


def assembled(S, f, n):
    return np.column_stack([S.apply_vanka(f, np.eye(n)[:, j]) for j in range(n)])


def test_pou_and_assembled_operator_vs_dense(S):
    # tests/test_vanka.cpp:157-185 (4 x 4 TH)
    c, d, k0, levels, _ = ref_case(4)
    n = k0.nrows
    K = S.SparseMatrix.from_csr(k0)
    p = S.build_patches(K, *d.nxyz0)
    f = S.factor_patches(K, p, d.nxyz0[0] + d.nxyz0[1])
    pl = p.export()
    m_ref, mult = dense_vanka(k0, pl, n)
    w = f.export(pl)["weights"]
    touched = mult > 0
    assert np.all(w[touched] * mult[touched] == 1.0)        # exact PoU
    m = assembled(S, f, n)
    assert np.abs(m - m_ref).max() <= 1e-11 * np.abs(m_ref).max()


def test_storage_accounting(S):
    # tests/test_vanka.cpp:187-194, and the reference's own byte counts
    c, d, k0, levels, _ = ref_case(8)
    K = S.SparseMatrix.from_csr(k0)
    f = S.factor_patches(K, S.build_patches(K, *d.nxyz0), d.nxyz0[0] + d.nxyz0[1])
    assert 2 * f.a_factor_bytes <= f.dense_inverse_bytes
    assert f.a_factor_bytes + f.aux_bytes <= f.dense_inverse_bytes
    rv = O.RefVanka.build(O.RefMat.from_csr(k0), *d.nxyz0).factors()
    assert (f.a_factor_bytes, f.aux_bytes, f.dense_inverse_bytes) == (
        rv["a_factor_bytes"], rv["aux_bytes"], rv["dense_inverse_bytes"])


def _one_patch_system(S):
    # tests/test_vanka.cpp:196-212: a 2-velocity / 1-pressure saddle system
    m = O.RefMat.from_triplets(3, 3, [0, 0, 1, 1, 2, 2], [0, 2, 1, 2, 0, 1],
                               [2.0, 1.0, 3.0, -1.0, 1.0, -1.0]).csr()
    K = S.SparseMatrix.from_csr(m)
    p = S.Patches.from_lists([0, 1], [2], [0, 2], [0, 1], [1])
    return m, K, S.factor_patches(K, p, 2)


def test_one_patch_is_the_inverse(S):
    m, K, f = _one_patch_system(S)
    b = np.array([1.0, 2.0, 3.0])
    x = S.apply_vanka(f, b)
    assert np.allclose(m.to_scipy().toarray() @ x, b, rtol=0, atol=1e-13)


def test_stationary_contraction(S):
    # tests/test_vanka.cpp:244-262: e_k = (1 - omega)^k e_0 with one exact patch
    m, K, f = _one_patch_system(S)
    xref = np.array([1.0, -2.0, 0.5])
    b = m.to_scipy().toarray() @ xref
    x = np.zeros(3)
    S.vanka_relax(K, f, x, b, S.RelaxMode.Stationary, 4, 0.78)
    e = np.linalg.norm(x - xref) / np.linalg.norm(xref)
    assert abs(e - (1 - 0.78) ** 4) <= 1e-10


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_relaxation_unit_counters(S, variant):
    # tests/test_preconditioner.cpp:96-120: the units each variant spends
    conf = dict(variant=variant)
    c, d, k0, levels, cf = ref_case(16, cfg=conf)
    K0 = S.SparseMatrix.from_csr(k0)
    lv = [(S.SparseMatrix.from_csr(k), S.SparseMatrix.from_csr(p) if p is not None else None,
           nxyz) for k, p, nxyz in levels]
    cfg = S.SolverConfig(variant=variant, nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500,
                         enclosed_flow=True)
    dc = S.DCPreconditioner(K0, d.nxyz0, lv, cfg)
    r = O.splitmix64_uniform(k0.nrows)
    before = d.counters()
    dc.apply(r)
    d.apply(r)
    after = d.counters()
    assert (dc.fine_relax_units, dc.level1_relax_units) == (after[0] - before[0],
                                                            after[1] - before[1])


def test_dclo_iterations_independent_of_eta(S):
    # tests/test_preconditioner.cpp:122-138: DC-LO skips the fine relaxation, so
    # the eta weighting of the restricted residual only scales the correction
    from paper_2306_06795_b200.cases import HostCase
    h = HostCase("cavity", False, "structured", 16)
    its = []
    for eta in (1.0, 0.5):
        cfg = S.SolverConfig(variant=1, nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500,
                             enclosed_flow=True, eta_u=eta, eta_p=eta)
        K0, dc, _ = h.device(cfg)
        _, rep = S.solve_stokes(K0, h.rhs(), dc, cfg)
        assert rep.converged
        its.append(rep.iterations)
    assert its[0] == its[1]


def test_enclosed_flow_zero_mean_pressure(S):
    # tests/test_preconditioner.cpp:220-238
    from paper_2306_06795_b200.cases import HostCase
    h = HostCase("cavity", False, "structured", 16)
    cfg = S.SolverConfig(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500, enclosed_flow=True)
    K0, dc, _ = h.device(cfg)
    x, rep = S.solve_stokes(K0, h.rhs(), dc, cfg)
    assert rep.converged and rep.final_relative_residual <= 1e-8
    p = x[h.n_x0 + h.n_y0:]
    assert abs(p.mean()) <= 1e-8 * max(np.abs(p).max(), 1.0)


def test_acceptance_jittered_patches_vs_dense(S):
    # tests/acceptance.cpp:69-116: jittered 14 x 14 TH mesh; the Vanka operator
    # on probes against the dense oracle
    c = O.RefCase.custom_th(14, 0, 0.2 / 14, 0)   # displacement 0.2 h
    k0 = c.k0().csr()
    n = k0.nrows
    K = S.SparseMatrix.from_csr(k0)
    nxyz = (c.n_x0, c.n_y0, c.n_p0)
    p = S.build_patches(K, *nxyz)
    f = S.factor_patches(K, p, nxyz[0] + nxyz[1])
    m_ref, _ = dense_vanka(k0, p.export(), n)
    rng = np.random.default_rng(99)
    for _ in range(3):
        r = rng.uniform(-1, 1, n)
        ref = m_ref @ r
        assert np.abs(S.apply_vanka(f, r) - ref).max() <= 1e-10 * np.abs(ref).max()


def test_acceptance_pou_every_level(S):
    # tests/acceptance.cpp:153-205: w * multiplicity == 1 exactly on K0 and on
    # every non-coarsest level of the hierarchy
    c, d, k0, levels, _ = ref_case(32)
    for k, nxyz in [(k0, d.nxyz0)] + [(l[0], l[2]) for l in levels[:-1]]:
        K = S.SparseMatrix.from_csr(k)
        p = S.build_patches(K, *nxyz)
        f = S.factor_patches(K, p, nxyz[0] + nxyz[1])
        pl = p.export()
        mult = np.bincount(np.concatenate([pl.velocity, pl.pressure]), minlength=k.nrows)
        w = f.export(pl)["weights"]
        t = mult > 0
        assert t.all()
        assert np.all(w[t] * mult[t] == 1.0)
