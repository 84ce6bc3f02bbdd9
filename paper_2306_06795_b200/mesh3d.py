"""Input generator for BASELINE config 5 (3D Taylor-Hood P2/P1 on the unit
cube, n^3 hexes each split into 6 tetrahedra, lid-driven cavity), which the
reference does not support (2D only). It states the 3D analogue of
the reference's 2D assembly (fem.cpp:354-450: P2 vector Laplacian per
component, divergence against the P1 pressure with the sign convention
B_kj = -int psi_k d(phi_j)/dx_c, all-Dirichlet elimination, fem.cpp:207-252)
with numpy / scipy, so that the 3-component Vanka kernels have realistic
inputs: patches of ~100-250 DoFs seeded at the pressure vertices.

Layout of K0 (fem.cpp:290-305 generalised): rows/cols
[x-velocity | y-velocity | z-velocity | pressure], the velocity block
block_diag(A, A, A) of the reduced scalar P2 Laplacian A.
"""
from __future__ import annotations

import itertools

import numpy as np


def cube_mesh(n: int):
    """(vertices (V, 3), tets (T, 4)): n^3 cubes, each split into the 6
    Kuhn tetrahedra along its main diagonal (positively oriented)."""
    g = np.linspace(0.0, 1.0, n + 1)
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    verts = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    vid = lambda i, j, k: (i * (n + 1) + j) * (n + 1) + k  # noqa: E731
    tets = []
    unit = np.eye(3, dtype=int)
    for i, j, k in itertools.product(range(n), repeat=3):
        base = np.array([i, j, k])
        for perm in itertools.permutations(range(3)):
            p = [base.copy()]
            for ax in perm:
                p.append(p[-1] + unit[ax])
            tets.append([vid(*q) for q in p])
    tets = np.array(tets, dtype=np.int64)
    a, b, c, d = (verts[tets[:, q]] for q in range(4))
    vol = np.einsum("ij,ij->i", np.cross(b - a, c - a), d - a)
    neg = vol < 0
    tets[neg] = tets[neg][:, [0, 2, 1, 3]]
    return verts, tets


_EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def p2_dofs(verts, tets):
    """Scalar P2 dofs: vertices, then the edges in lexicographic (a < b) order
    (mesh.cpp:55-73 generalised). Returns (dofs (T, 10), edges (E, 2))."""
    nv = len(verts)
    e = np.concatenate([np.sort(tets[:, list(p)], axis=1) for p in _EDGES])
    edges, inv = np.unique(e, axis=0, return_inverse=True)
    inv = inv.reshape(len(_EDGES), len(tets)).T
    return np.concatenate([tets, nv + inv], axis=1), edges


# degree-2 exact rule on the reference tetrahedron (4 points, weights 1/4)
_QA, _QB = 0.5854101966249685, 0.1381966011250105
_QL = np.array([[_QA, _QB, _QB, _QB], [_QB, _QA, _QB, _QB], [_QB, _QB, _QA, _QB],
                [_QB, _QB, _QB, _QA]])


def assemble(n: int):
    """(K0 scipy CSR, (n_x, n_y, n_z, n_p), rhs) of the lid-driven cavity
    (u = (1, 0, 0) on z = 1, zero elsewhere), Dirichlet dofs eliminated."""
    import scipy.sparse as sp
    verts, tets = cube_mesh(n)
    dofs, edges = p2_dofs(verts, tets)
    nv, ne, nt = len(verts), len(edges), len(tets)
    ns = nv + ne
    P = verts[tets]                                   # (T, 4, 3)
    J = np.stack([P[:, 1] - P[:, 0], P[:, 2] - P[:, 0], P[:, 3] - P[:, 0]], axis=2)
    det = np.linalg.det(J)
    vol = det / 6.0
    Jinv = np.linalg.inv(J)                           # rows: grad of lambda_1..3
    gl = np.concatenate([-Jinv.sum(axis=1, keepdims=True), Jinv], axis=1)  # (T, 4, 3)
    rows_a, cols_a, vals_a = [], [], []
    rows_b, cols_b, vals_b = [], [], []
    for q in range(4):
        lam = _QL[q]
        w = vol / 4.0
        # grad of the P2 basis: vertex i: (4 lam_i - 1) grad lam_i;
        # edge (i, j): 4 (lam_i grad lam_j + lam_j grad lam_i)
        gphi = np.empty((nt, 10, 3))
        for i in range(4):
            gphi[:, i] = (4 * lam[i] - 1) * gl[:, i]
        for e, (i, j) in enumerate(_EDGES):
            gphi[:, 4 + e] = 4 * (lam[i] * gl[:, j] + lam[j] * gl[:, i])
        a = np.einsum("t,tic,tjc->tij", w, gphi, gphi)
        rows_a.append(np.repeat(dofs, 10, axis=1).ravel())
        cols_a.append(np.tile(dofs, (1, 10)).ravel())
        vals_a.append(a.ravel())
        for c in range(3):
            bq = -np.einsum("t,k,tj->tkj", w, lam, gphi[:, :, c])  # (T, 4, 10)
            rows_b.append(np.repeat(tets, 10, axis=1).ravel())
            cols_b.append((c * ns + np.tile(dofs, (1, 4))).ravel())
            vals_b.append(bq.ravel())
    A = sp.csr_matrix((np.concatenate(vals_a), (np.concatenate(rows_a),
                                                np.concatenate(cols_a))), shape=(ns, ns))
    B = sp.csr_matrix((np.concatenate(vals_b), (np.concatenate(rows_b),
                                                np.concatenate(cols_b))), shape=(nv, 3 * ns))
    A.sum_duplicates()
    B.sum_duplicates()
    # Dirichlet dofs: every vertex / edge midpoint on the boundary
    coords = np.concatenate([verts, 0.5 * (verts[edges[:, 0]] + verts[edges[:, 1]])])
    on_b = ((coords < 1e-12) | (coords > 1 - 1e-12)).any(axis=1)
    lid = coords[:, 2] > 1 - 1e-12
    g = np.zeros((ns, 3))
    g[lid, 0] = 1.0
    keep = np.nonzero(~on_b)[0]
    cons = np.nonzero(on_b)[0]
    A_ff = A[keep][:, keep]
    lift = A[keep][:, cons] @ g[cons]                 # (n_free, 3)
    Bk = sp.hstack([B[:, c * ns + keep] for c in range(3)]).tocsr()
    rhs_p = -sum(B[:, c * ns + cons] @ g[cons, c] for c in range(3))
    nf = len(keep)
    K = sp.bmat([[sp.block_diag([A_ff, A_ff, A_ff]), Bk.T], [Bk, None]], format="csr")
    K.sort_indices()
    K.eliminate_zeros()
    rhs = np.concatenate([-lift[:, 0], -lift[:, 1], -lift[:, 2], rhs_p])
    return K, (nf, nf, nf, nv), rhs


def k0_csr(n: int):
    """K0 of config 5 at n^3 as int32 / float64 CSR arrays plus the block sizes."""
    K, nxyz, rhs = assemble(n)
    return (K.shape[0], K.indptr.astype(np.int32), K.indices.astype(np.int32),
            K.data.astype(np.float64), nxyz, rhs)
