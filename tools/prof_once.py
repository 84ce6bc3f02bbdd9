#!/usr/bin/env python
"""Two rounds of the hot kernels of one level of a bench config (the first
round warms up; ncu_traffic.py keeps the second), for ncu captures:

    ncu --set full --import-source on --clock-control none \
        -k regex:"spmv_kernel|vanka_patch_kernel|vanka_subwarp_kernel|vanka_fixed_kernel|vanka_gather" \
        -o gpurun_out/prof python tools/prof_once.py --config 3 --level ISO0

Order per round: spmv (Store), Vanka patch stage (one launch per size class),
Vanka gather. --level K0 (default) or ISO0 (level 0 of the low-order
hierarchy).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2306_06795_b200 as S  # noqa: E402
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--level", default="K0", choices=["K0", "ISO0"])
    a = ap.parse_args()
    case = bench.host_case(bench.CONFIGS[a.config])
    if a.level == "K0":
        k, nxyz, sv = case.k0(), case.nxyz0, case.sv
    else:
        k, _, nxyz = case.level(0)
        sv = False
    ctx = S.Context(0)
    dev = torch.device("cuda", 0)
    n = k.nrows
    x = torch.from_numpy(bench.splitmix64_uniform(n)).to(dev)
    y = torch.empty_like(x)
    K = S.SparseMatrix.from_csr(k, ctx)
    f = S.factor_patches(K, S.build_patches(K, *nxyz, sv_triples=sv), nxyz[0] + nxyz[1])
    lib = S.lib()
    xp, yp = (S.C.c_void_p(t.data_ptr()) for t in (x, y))
    for _ in range(2):
        S._check(lib.sag_spmv_fused(ctx.h, K.h, xp, yp, None, 0))
        S._check(lib.sag_apply_vanka_stage(ctx.h, f.h, xp, yp, 1))
        S._check(lib.sag_apply_vanka_stage(ctx.h, f.h, xp, yp, 2))
        ctx.synchronize()
    print({"config": a.config, "level": a.level, "rows": n, "classes": f.classes(),
           "patch_bytes": bench.vanka_patch_bytes(f, n), "spmv_bytes": bench.spmv_bytes(n, n, k.nnz)})


if __name__ == "__main__":
    main()
