"""GPU: the 3-component Vanka kernels (BASELINE config 5: 3D Taylor-Hood
P2/P1 on the unit cube, n^3 hexes x 6 tets, lid-driven cavity -- no
reference support) against oracle.c's 3-component restatement
(or_*3, itself pinned to dense patch inverses in tests/test_oracle3d.py):
apply within 1e-12, SpMV within 1e-12, linearity, run-to-run determinism,
patches of up to ~170 dofs (CTA per patch)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2306_06795_b200 as S
    return S


def rel_inf(a, b):
    return np.abs(np.asarray(a) - b).max() / np.abs(b).max()


@pytest.mark.parametrize("n", [2, 4, 6, 8])
def test_vanka3_matches_oracle(S, n):
    from paper_2306_06795_b200 import mesh3d
    N, rp, ci, v, nxyz, rhs = mesh3d.k0_csr(n)
    k = O.Csr(N, N, rp, ci, v)
    K = S.SparseMatrix.from_csr(k)
    f = S.VankaFactorization3(K, *nxyz)
    ref = O.OracleVanka3(k, *nxyz)
    r = O.splitmix64_uniform(N)
    d = f.apply(r)
    assert rel_inf(d, ref.apply(r)) <= 1e-12
    assert rel_inf(S.spmv(K, r), O.Oracle.spmv(k, r)) <= 1e-12
    z = O.splitmix64_uniform(N, seed=5)
    assert rel_inf(f.apply(0.5 * r - 2.0 * z), 0.5 * d - 2.0 * f.apply(z)) <= 1e-12
    assert np.array_equal(f.apply(r), d)
    if n >= 4:
        assert f.max_nv > 100   # the large 3D patches
