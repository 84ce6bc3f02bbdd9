#!/usr/bin/env python
"""Host-link probe for the e2e step (pinned host buffers): DMA copies each
way and both ways at once, and sag_vanka_spmv with host buffers (x in, then
y and delta out in chunks under the compute).

    python tools/e2e_probe.py [--config 2]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_06795_b200 as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    a = ap.parse_args()
    case = bench.host_case(bench.CONFIGS[a.config])
    k0 = case.k0()
    n = k0.nrows
    ctx = S.Context(0)
    K = S.SparseMatrix.from_csr(k0, ctx)
    f = S.factor_patches(K, S.build_patches(K, *case.nxyz0, sv_triples=case.sv),
                         case.n_x0 + case.n_y0)
    out = {"n": n}
    xh = torch.from_numpy(bench.splitmix64_uniform(n)).pin_memory()
    dh = torch.empty(n, dtype=torch.float64).pin_memory()
    yh = torch.empty(n, dtype=torch.float64).pin_memory()
    xd = torch.empty(n, dtype=torch.float64, device="cuda")
    yd = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    y2h = torch.empty(2 * n, dtype=torch.float64).pin_memory()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def wall(fn, k=10):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / k

    out["h2d_8n_ms"] = 1e3 * wall(lambda: xd.copy_(xh, non_blocking=True))
    out["d2h_16n_ms"] = 1e3 * wall(lambda: y2h.copy_(yd, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            xd.copy_(xh, non_blocking=True)
        with torch.cuda.stream(s2):
            y2h.copy_(yd, non_blocking=True)
    out["h2d_8n_and_d2h_16n_ms"] = 1e3 * wall(both)
    xn, dn, yn = xh.numpy(), dh.numpy(), yh.numpy()
    t = wall(lambda: S.vanka_spmv_step(f, K, xn, dn, yn))
    out["step_ms"] = 1e3 * t
    out["step_gdofs"] = n / t / 1e9
    out["bound_ms"] = out["h2d_8n_ms"] + out["d2h_16n_ms"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
