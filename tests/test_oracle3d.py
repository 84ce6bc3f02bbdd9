"""CPU: the 3-component Vanka restatement (oracle.c or_*3, BASELINE config 5;
the reference has no 3D path) pinned to a dense computation of
its definition on the 3D Taylor-Hood cavity (mesh3d): delta = sum_i V_i^T
W (K_i)^-1 V_i r over the pressure-seeded patches, K_i the patch's dense
saddle block, W the partition-of-unity weights (vanka.cpp:64-184) -- the
block-LU route (one LU per velocity component, Schur complement with the
symmetric-A b_hat formula) equals the dense inverse on every patch because
A = block_diag(A_x, A_y, A_z) and each A_c is symmetric."""
import numpy as np
import pytest

import oracle as O


def system(n):
    from paper_2306_06795_b200 import mesh3d
    N, rp, ci, v, nxyz, rhs = mesh3d.k0_csr(n)
    return O.Csr(N, N, rp, ci, v), nxyz


@pytest.mark.parametrize("n", [2, 3, 4])
def test_oracle3_equals_dense_patch_inverses(n):
    k, nxyz = system(n)
    f = O.OracleVanka3(k, *nxyz)
    r = O.splitmix64_uniform(k.nrows)
    got = f.apply(r)
    Kd = k.to_scipy().toarray()
    n_u = sum(nxyz[:3])
    mult = np.zeros(k.nrows)
    want = np.zeros(k.nrows)
    contrib = []
    for i in range(len(f.pptr) - 1):
        dofs = np.concatenate([f.vidx[f.vptr[i]:f.vptr[i + 1]], f.pidx[f.pptr[i]:f.pptr[i + 1]]])
        mult[dofs] += 1
        contrib.append((dofs, np.linalg.solve(Kd[np.ix_(dofs, dofs)], r[dofs])))
    for dofs, x in contrib:
        want[dofs] += x / mult[dofs]
    assert np.abs(got - want).max() <= 1e-9 * np.abs(want).max()
    # patch shapes: every velocity list split x | y | z in ascending order
    assert (f.cnt.sum(axis=1) == np.diff(f.vptr)).all()
    assert (f.vidx < n_u).all()


def test_mesh3d_counts_match_baseline_config5_formula():
    # BASELINE config 5 at 64^3: 3 x 129^3 velocity dofs before elimination
    # (~6.4M) and 65^3 = 274,625 pressure dofs; check the formula at small n
    from paper_2306_06795_b200 import mesh3d
    for n in (2, 4):
        K, (nx, ny, nz, np_), rhs = mesh3d.assemble(n)
        assert np_ == (n + 1) ** 3
        assert nx == ny == nz == (2 * n - 1) ** 3      # interior P2 nodes
        assert K.shape[0] == 3 * nx + np_
