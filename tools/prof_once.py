#!/usr/bin/env python
"""One launch of each hot kernel of the bench step on config 2's K0 (after one
untimed warm-up round), for `ncu --set full` captures:

    ncu --set full --import-source on --clock-control none -s <warm-up launches> \
        -o gpurun_out/prof python tools/prof_once.py [n=512]

Order per round: spmv (Store), spmv (StoreDot), Vanka patch kernel, Vanka
gather kernel.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2306_06795_b200 as S  # noqa: E402
from paper_2306_06795_b200.cases import HostCase  # noqa: E402
from bench import splitmix64_uniform  # noqa: E402


def main():
    n_mesh = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    case = HostCase("cavity", False, "structured", n_mesh)
    k0 = case.k0()
    ctx = S.Context(0)
    dev = torch.device("cuda", 0)
    n = k0.nrows
    x = torch.from_numpy(splitmix64_uniform(n)).to(dev)
    y = torch.empty_like(x)
    aux = torch.from_numpy(splitmix64_uniform(n, 7)).to(dev)
    K = S.SparseMatrix.from_csr(k0, ctx)
    p = S.build_patches(K, *case.nxyz0)
    f = S.factor_patches(K, p, case.n_x0 + case.n_y0)
    lib = S.lib()
    xp, yp, ap = (S.C.c_void_p(t.data_ptr()) for t in (x, y, aux))
    for _ in range(2):
        S._check(lib.sag_spmv_fused(ctx.h, K.h, xp, yp, ap, 0))
        S._check(lib.sag_spmv_fused(ctx.h, K.h, xp, yp, ap, 3))
        S._check(lib.sag_apply_vanka_stage(ctx.h, f.h, xp, yp, 1))
        S._check(lib.sag_apply_vanka_stage(ctx.h, f.h, xp, yp, 2))
        ctx.synchronize()


if __name__ == "__main__":
    main()
