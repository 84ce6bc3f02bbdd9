#!/usr/bin/env python
"""Launch-shape sweep for the Vanka apply and the SpMV on one config (GPU).
Prints one JSON line per variant: microseconds per launch (CUDA events over K
launches on libsag's stream) and GB/s of algorithmic / device bytes.

    python tools/sweep.py [n=512] ["ENV=V,ENV=V;ENV=V,..."]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2306_06795_b200 as S  # noqa: E402
from paper_2306_06795_b200.cases import HostCase  # noqa: E402
from bench import splitmix64_uniform, spmv_bytes, vanka_bytes  # noqa: E402

DEFAULT_VARIANTS = [
    "SAG_VANKA_TPP=0,SAG_VANKA_UNROLL=1,SAG_VANKA_STAGES=3,SAG_VANKA_CTA_SMEM=60000",
    "SAG_VANKA_TPP=0,SAG_VANKA_UNROLL=1,SAG_VANKA_STAGES=3,SAG_VANKA_CTA_SMEM=112000",
    "SAG_VANKA_TPP=0,SAG_VANKA_UNROLL=1,SAG_VANKA_STAGES=4,SAG_VANKA_CTA_SMEM=60000",
    "SAG_VANKA_TPP=0,SAG_VANKA_UNROLL=0,SAG_VANKA_STAGES=3,SAG_VANKA_CTA_SMEM=60000",
]


def main():
    n_mesh = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    variants = sys.argv[2].split(";") if len(sys.argv) > 2 else DEFAULT_VARIANTS
    t0 = time.time()
    case = HostCase("cavity", False, "structured", n_mesh)
    k0 = case.k0()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)  # torch-owned: libsag never destroys it
    ctx = S.Context(0, stream=stream.cuda_stream)
    n = k0.nrows
    x = torch.from_numpy(splitmix64_uniform(n)).to(dev)
    y = torch.empty_like(x)
    print(json.dumps({"setup_s": time.time() - t0, "n": n, "nnz": k0.nnz}), flush=True)

    def timed(fn, k=30):
        for _ in range(3):
            fn()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / k * 1e3  # us

    bs = spmv_bytes(n, n, k0.nnz)
    lib = S.lib()
    aux = torch.from_numpy(splitmix64_uniform(n, 7)).to(dev)
    xp_, yp_, ap_ = (S.C.c_void_p(t.data_ptr()) for t in (x, y, aux))
    spmv_variants = os.environ.get("SWEEP_SPMV", "").split(";")
    for sv in spmv_variants:
        env = dict(kv.split("=") for kv in sv.split(",") if kv)
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        K = S.SparseMatrix.from_csr(k0, ctx)  # launch shape is chosen at upload
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        us = timed(lambda: S.spmv(K, x, out=y))
        rec = {"kernel": "spmv", "variant": sv, "us": us, "gbs": bs / us / 1e3}
        for epi, name in ((0, "store"), (1, "resid"), (2, "add"), (3, "store_dot"),
                          (4, "resid_ssq")):
            rec[name] = timed(lambda: S._check(lib.sag_spmv_fused(ctx.h, K.h, xp_, yp_, ap_, epi)))
        print(json.dumps(rec), flush=True)
    K = S.SparseMatrix.from_csr(k0, ctx)
    built = {}
    for var in variants:
        env = dict(kv.split("=") for kv in var.split(",") if kv)
        os.environ.update(env)
        key = (env.get("SAG_VANKA_TPP", "0"), env.get("SAG_VANKA_SYM", "1"),
               env.get("SAG_VANKA_PAIRS", "1"))
        if key not in built:
            built.clear()
            p = S.build_patches(K, *case.nxyz0)
            f = S.factor_patches(K, p, case.n_x0 + case.n_y0)
            built[key] = (p, f)
        p, f = built[key]
        bv = vanka_bytes(f, p.total_velocity + p.total_pressure, n)
        xp, dp = S.C.c_void_p(x.data_ptr()), S.C.c_void_p(y.data_ptr())
        try:
            us_patch = timed(lambda: S._check(lib.sag_apply_vanka_stage(ctx.h, f.h, xp, dp, 1)))
            us_g = timed(lambda: S._check(lib.sag_apply_vanka_stage(ctx.h, f.h, xp, dp, 2)))
        except S.Error as e:
            print(json.dumps({"variant": var, "err": str(e)}), flush=True)
            continue
        print(json.dumps({"kernel": "vanka", "variant": var, "patch_us": us_patch,
                          "gather_us": us_g, "sweep_us": us_patch + us_g,
                          "device_bytes": f.device_bytes,
                          "patch_dev_gbs": f.device_bytes / us_patch / 1e3,
                          "sweep_alg_gbs": bv / (us_patch + us_g) / 1e3}), flush=True)


if __name__ == "__main__":
    main()
