#!/usr/bin/env python
"""e2e time of the pipelined host-buffer step (sag_vanka_spmv, pinned host
buffers) against the stage count SAG_STEP_STAGES.

    python tools/e2e_stages.py [--config 2] [stages ...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_06795_b200 as S  # noqa: E402


def main():
    args = [a for a in sys.argv[1:]]
    ci = 2
    if "--config" in args:
        i = args.index("--config")
        ci = int(args[i + 1])
        del args[i:i + 2]
    stages = [int(a) for a in args] or [1, 2, 4, 6, 8, 12, 16, 24, 32]
    conf = bench.CONFIGS[ci]
    case = bench.host_case(conf)
    ctx = S.Context(0)
    k0, nxyz0 = case.k0(), case.nxyz0
    K0 = S.SparseMatrix.from_csr(k0, ctx)
    f = S.factor_patches(K0, S.build_patches(K0, *nxyz0, sv_triples=case.sv), nxyz0[0] + nxyz0[1])
    n = K0.nrows
    x = bench.splitmix64_uniform(n)
    xh = torch.from_numpy(x).pin_memory().numpy()
    dh = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    yh = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    ref_d, ref_y = None, None
    out = {"config": ci, "n": n, "runs": []}
    for st in stages:
        os.environ["SAG_STEP_STAGES"] = str(st)
        for _ in range(3):
            S.vanka_spmv_step(f, K0, xh, dh, yh)
        k = 20
        t0 = time.perf_counter()
        for _ in range(k):
            S.vanka_spmv_step(f, K0, xh, dh, yh)
        t = (time.perf_counter() - t0) / k
        if ref_d is None:
            ref_d, ref_y = dh.copy(), yh.copy()
        same = bool(np.array_equal(ref_d, dh) and np.array_equal(ref_y, yh))
        out["runs"].append({"stages": st, "ms": 1e3 * t, "gdofs": n / t / 1e9, "bitwise": same,
                            "plan": S.vanka_step_plan(f)})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
