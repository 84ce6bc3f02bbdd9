#!/usr/bin/env python
"""Two sweeps of the 3-component Vanka apply on the config-5 operator, for
ncu captures (-k regex:apply3_kernel):   python tools/prof3d_once.py [n=24]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402  (Csr container only)
import paper_2306_06795_b200 as S  # noqa: E402
from paper_2306_06795_b200 import mesh3d  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
N, rp, ci, v, nxyz, rhs = mesh3d.k0_csr(n)
K = S.SparseMatrix.from_csr(O.Csr(N, N, rp, ci, v))
f = S.VankaFactorization3(K, *nxyz)
r = O.splitmix64_uniform(N)
for _ in range(2):
    f.apply(r)
print({"n": n, "rows": N})
