#!/usr/bin/env python
"""Vanka patch-stage time on one level of a bench config under launch-shape
knobs (SAG_VANKA_STAGES / _WARPS / _CTA_SMEM / _MINB), CUDA events on the
context's stream, 20 launches per setting after 3 warm-ups:

    python tools/knob_sweep.py --config 3 --level K0 "STAGES=2,3" "WARPS=4,8"
"""
import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_06795_b200 as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--level", default="K0", choices=["K0", "ISO0"])
    ap.add_argument("knobs", nargs="*")
    a = ap.parse_args()
    case = bench.host_case(bench.CONFIGS[a.config])
    if a.level == "K0":
        k, nxyz, sv = case.k0(), case.nxyz0, case.sv
    else:
        k, _, nxyz = case.level(0)
        sv = False
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    ctx = S.Context(0, stream=stream.cuda_stream)
    n = k.nrows
    x = torch.from_numpy(bench.splitmix64_uniform(n)).to(dev)
    y = torch.empty_like(x)
    K = S.SparseMatrix.from_csr(k, ctx)
    f = S.factor_patches(K, S.build_patches(K, *nxyz, sv_triples=sv), nxyz[0] + nxyz[1])
    lib = S.lib()
    xp, yp = (S.C.c_void_p(t.data_ptr()) for t in (x, y))
    names, values = [], []
    for kv in a.knobs:
        nm, vs = kv.split("=")
        names.append(nm)
        values.append(vs.split(","))
    ref = None
    for combo in itertools.product(*values) if names else [()]:
        for nm, v in zip(names, combo):
            os.environ["SAG_VANKA_" + nm] = v
        for _ in range(3):
            S._check(lib.sag_apply_vanka_stage(ctx.h, f.h, xp, yp, 1))
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(20):
            S._check(lib.sag_apply_vanka_stage(ctx.h, f.h, xp, yp, 1))
        e1.record(stream)
        e1.synchronize()
        S._check(lib.sag_apply_vanka_stage(ctx.h, f.h, xp, yp, 2))
        ctx.synchronize()
        out = y.cpu()
        same = True if ref is None else bool(torch.equal(out, ref))
        ref = out if ref is None else ref
        print(json.dumps({"config": a.config, "level": a.level, **dict(zip(names, combo)),
                          "patch_us": 1e3 * e0.elapsed_time(e1) / 20, "same": same}), flush=True)


if __name__ == "__main__":
    main()
