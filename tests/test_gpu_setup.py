"""GPU: the SA hierarchy setup products on the device (sag_spgemm,
sag_galerkin, sag_smooth_prolongator) are BITWISE the
reference's. The low-order hierarchy of a case is built twice -- by the
reference's build_monolithic_hierarchy (amg.cpp:300-360) and by
gpu::build_monolithic_hierarchy, whose smoothed prolongators and Galerkin
products run on the device -- and every level's K and P must be identical
(patterns and values): the setup drops entries that cancel to exactly 0.0
(SURVEY H1), so anything but the reference's summation order would show."""
import numpy as np
import pytest

import oracle as O
from conftest import ref_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("problem,sv,n", [("cavity", False, 16), ("cavity", False, 64),
                                          ("cavity", True, 8), ("bfs", False, 16)])
def test_hierarchy_on_device_is_bitwise(problem, sv, n):
    from paper_2306_06795_b200.cases import HostCase
    case = HostCase(problem, sv, "structured", n)
    r = case.hierarchy_gpu(0)
    assert r["levels"] >= 2
    assert r["bitwise_equal"], r
    assert r["soc_device"] >= 3 and r["soc_host"] == 0, r   # every strength graph on the device


def test_hierarchy_on_device_is_bitwise_unstructured(tmp_path):
    """The same on a jittered Delaunay mesh (BASELINE config 4's recipe at
    40 x 40 points): irregular patterns and strength supports."""
    from paper_2306_06795_b200 import meshgen
    from paper_2306_06795_b200.cases import HostCase
    path = meshgen.write_mesh(str(tmp_path / "m.json"), 40, seed=7, jitter=0.3)
    k1, k2 = meshgen.force_wavenumbers()
    case = HostCase("cavity", False, "file_forced", 0, mesh_path=path, k1=k1, k2=k2)
    r = case.hierarchy_gpu(0)
    assert r["bitwise_equal"] and r["soc_host"] == 0, r
    s = case.scalar_hierarchies_gpu(0)
    assert s["bitwise_equal"], s


@pytest.mark.parametrize("sv,n", [(False, 16), (False, 64), (True, 8)])
def test_scalar_hierarchies_on_device_are_bitwise(sv, n):
    """gpu::build_scalar_hierarchy (Uzawa's A_x / Mp hierarchies, SV's pressure
    projection) equals build_scalar_hierarchy (amg.cpp:200-256) bit for bit:
    levels, prolongators, Jacobi diagonals and the coarse LU."""
    from paper_2306_06795_b200.cases import HostCase
    r = HostCase("cavity", sv, "structured", n).scalar_hierarchies_gpu(0)
    assert r["bitwise_equal"] and r["operators"] == 2 and r["soc_device"] >= 1, r


def test_evolution_soc_graph_matches_reference():
    """sag_evolution_soc vs the reference's evolution_soc through the
    aggregation it feeds: the hierarchy test checks the end result; here the
    graph of a level's velocity block against a CPU restatement of amg.cpp:45-110."""
    import paper_2306_06795_b200 as S
    c, d, k0, levels, _ = ref_case(16)
    k, p, (nx, ny, npp) = levels[0]
    a = k.to_scipy().tocsr()[:nx, :nx].tocsr()
    a.sort_indices()
    A = S.SparseMatrix(nx, nx, a.indptr, a.indices, a.data)
    dinv = 1.0 / a.diagonal()
    rho = 2.0  # any positive omega exercises the same arithmetic
    omega = 4.0 / (3.0 * rho)
    g = S.evolution_soc(A, omega, 0.5, 2)
    grp, gci, gv = g.to_csr()
    at = a.T.tocsr()
    at.sort_indices()
    adj = [dict() for _ in range(nx)]
    for j in range(nx):
        z, touched = {j: 1.0}, [j]
        for _ in range(2):
            az, azt = {}, []
            for idx in list(touched):
                v = z.get(idx, 0.0)
                if v == 0.0:
                    continue
                for q in range(at.indptr[idx], at.indptr[idx + 1]):
                    i = at.indices[q]
                    if i not in az:
                        az[i] = 0.0
                        azt.append(i)
                    az[i] += at.data[q] * v
            for i in azt:
                if i not in z:
                    z[i] = 0.0
                    touched.append(i)
                z[i] -= omega * dinv[i] * az[i]
        zj = abs(z[j])
        if zj > 0.0:
            smax = max([abs(z[i]) / zj for i in touched if i != j] + [0.0])
            if smax > 0.0:
                for i in touched:
                    s = abs(z[i]) / zj
                    if i != j and s > 0.0 and s >= 0.5 * smax:
                        adj[i][j] = max(adj[i].get(j, 0.0), s)
                        adj[j][i] = max(adj[j].get(i, 0.0), s)
    for i in range(nx):
        cols = sorted(adj[i])
        assert list(gci[grp[i]:grp[i + 1]]) == cols
        assert np.array_equal(gv[grp[i]:grp[i + 1]], [adj[i][c_] for c_ in cols])


def test_spgemm_transpose_match_reference():
    """spgemm / transpose / galerkin_triple on a reference level and its
    prolongator against the reference's next level (the hierarchy's own
    Galerkin product), through the Python mirror."""
    import paper_2306_06795_b200 as S
    c, d, k0, levels, _ = ref_case(32)
    k, p, _ = levels[0]
    K, P = S.SparseMatrix.from_csr(k), S.SparseMatrix.from_csr(p)
    kc = S.galerkin_triple(P, K)
    rp, ci, v = kc.to_csr()
    nxt = levels[1][0]
    assert np.array_equal(rp, nxt.rp) and np.array_equal(ci, nxt.ci)
    assert np.array_equal(v.view(np.int64), nxt.v.view(np.int64))
    pt = S.transpose(P).to_csr()
    ref_t = O.RefMat.from_csr(p)
    # transpose: rows of P^T list the rows of P in ascending order
    sp = p.to_scipy().T.tocsr()
    sp.sort_indices()
    assert np.array_equal(pt[0], sp.indptr) and np.array_equal(pt[1], sp.indices)
    assert np.array_equal(pt[2], sp.data)
    del ref_t
    kp = S.spgemm(K, P).to_csr()
    assert kp[0][-1] > 0 and (np.diff(kp[0]) >= 0).all()


def test_spgemm_drops_exact_cancellation_and_keeps_empty_rows():
    """sparse.cpp:140-146: an entry whose products cancel to exactly 0.0 is
    not stored; rows without products stay empty; columns ascend."""
    import paper_2306_06795_b200 as S
    # A = [[1, 1, 0], [0, 0, 0], [2, 0, 3]], B = [[1, 2], [-1, 5], [0, 1]]
    a = S.SparseMatrix(3, 3, [0, 2, 2, 4], [0, 1, 0, 2], [1.0, 1.0, 2.0, 3.0])
    b = S.SparseMatrix(3, 2, [0, 2, 4, 5], [0, 1, 0, 1, 1], [1.0, 2.0, -1.0, 5.0, 1.0])
    rp, ci, v = S.spgemm(a, b).to_csr()
    # row 0: (1 - 1, 2 + 5) -> col 0 cancels exactly; row 1 empty; row 2: (2, 4 + 3)
    assert list(rp) == [0, 1, 1, 3]
    assert list(ci) == [1, 0, 1] and list(v) == [7.0, 2.0, 7.0]
    # transpose of the result and a Galerkin product with an identity prolongator
    t = S.transpose(S.spgemm(a, b)).to_csr()
    assert list(t[0]) == [0, 1, 3] and list(t[1]) == [2, 0, 2]
    eye = S.SparseMatrix(3, 3, [0, 1, 2, 3], [0, 1, 2], [1.0, 1.0, 1.0])
    g = S.galerkin_triple(eye, a).to_csr()
    assert list(g[0]) == [0, 2, 2, 4] and list(g[2]) == [1.0, 1.0, 2.0, 3.0]


def test_tentative_prolongator_device():
    # amg.cpp:184-205: per-aggregate norms summed in node order, T = nullvec
    # / norm with exact zeros dropped (from_triplets), coarse nullvec = norms;
    # an aggregate with a zero norm (or no node) raises
    import math
    import paper_2306_06795_b200 as S
    rng = np.random.default_rng(5)
    n, nc = 5000, 700
    agg = rng.permutation(np.arange(n) % nc).astype(np.int32)
    nv = rng.standard_normal(n)
    nv[::97] = 0.0
    t, cn = S.tentative_prolongator(agg, nc, nv)
    want = np.zeros(nc)
    for i in range(n):                   # the reference's loop, in order
        want[agg[i]] += nv[i] * nv[i]
    want = np.array([math.sqrt(v) for v in want])
    assert cn.tobytes() == want.tobytes()
    rp, ci, v = t.to_csr()
    keep = nv != 0.0
    assert np.array_equal(np.diff(rp), keep.astype(np.int32))
    assert np.array_equal(ci, agg[keep])
    assert v.tobytes() == (nv[keep] / want[agg[keep]]).tobytes()
    with pytest.raises(S.Error):
        S.tentative_prolongator(np.zeros(4, np.int32), 2, np.ones(4))   # aggregate 1 empty
    with pytest.raises(S.Error):
        S.tentative_prolongator(np.array([0, 1], np.int32), 2, np.array([1.0, 0.0]))


def test_power_rho_device():
    # sparse.cpp:239-261 with the reference's start vector and sequential norms
    import paper_2306_06795_b200 as S
    c = O.RefCase.build("cavity", False, "structured", 16)
    k = c.k0().csr()
    a = O.Csr(k.nrows, k.nrows, k.rp, k.ci, k.v)
    n = k.nrows
    d = np.array([1.0 / a.v[a.rp[r]:a.rp[r + 1]][a.ci[a.rp[r]:a.rp[r + 1]] == r][0]
                  if (a.ci[a.rp[r]:a.rp[r + 1]] == r).any() else 1.0 for r in range(n)])
    x = np.random.default_rng(1).uniform(-1, 1, n)
    x = x / np.sqrt(np.sum(x * x))
    rho = S.power_rho(S.SparseMatrix.from_csr(k), d, x, 10)
    xr = x.copy()
    ref = 0.0
    for _ in range(10):                  # the reference loop with row-ordered sums
        y = np.empty(n)
        for r in range(n):
            s = 0.0
            for q in range(a.rp[r], a.rp[r + 1]):
                s += a.v[q] * xr[a.ci[q]]
            y[r] = s * d[r]
        s = 0.0
        for v in y:
            s += v * v
        ref = float(np.sqrt(s))
        xr = y / ref
    assert rho == ref
