#!/usr/bin/env python
"""Where the one-launch SV mass projection (sv_project_kernel) spends its
time: per-phase (tag) wait and work times of worker CTA 0 from the in-kernel
globaltimer trace (SAG_PROJ_TRACE=1), for one DC apply of a bench config.

    python tools/proj_trace.py [--config 3]
"""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SAG_PROJ_TRACE"] = "1"

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_06795_b200 as S  # noqa: E402

TAGS = {1: "smooth ssq/resid", 2: "smooth z0", 3: "smooth A z0 . v0", 4: "smooth |w|",
        5: "smooth z1", 6: "smooth A z1 . v0", 7: "smooth w . v1", 8: "smooth |w| (2)",
        9: "pre-smooth x", 10: "residual", 11: "restrict", 12: "tail", 13: "prolong",
        14: "post-smooth x", 15: "rhs = M_mix p", 16: "restart residual", 17: "A z_j . v0",
        18: "MGS", 19: "|w|", 20: "x update"}


def main():
    ci = int(sys.argv[sys.argv.index("--config") + 1]) if "--config" in sys.argv else 3
    conf = bench.CONFIGS[ci]
    case = bench.host_case(conf)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    ctx = S.Context(0, stream=stream.cuda_stream)
    cfg = S.SolverConfig(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500,
                         enclosed_flow=case.enclosed, eta_u=conf.get("eta_u", 1.0),
                         eta_p=conf.get("eta_p", 1.0), omega0=conf.get("omega0", 1.0))
    K0, dc, _ = case.device(cfg, ctx)
    n = K0.nrows
    r = torch.from_numpy(bench.splitmix64_uniform(n)).to(dev)
    z = torch.empty_like(r)
    for _ in range(3):
        dc.apply(r, out=z)
    ctx.synchronize()
    w, t = dc.proj_trace()
    out = {"info": dc.info()}
    for name, tr in (("worker0", w), ("tail0", t)):
        tags = tr[:, 0].astype(np.int64)
        ns = tr[:, 1].astype(np.int64)
        end = int(np.argmax(tags == 9999)) if (tags == 9999).any() else len(tags)
        tags, ns = tags[:end + 1], ns[:end + 1]
        if len(ns) < 2:
            continue
        # arrive (tag) -> release (tag + 1000) = wait; release -> next arrive = work
        wait = collections.defaultdict(float)
        work = collections.defaultdict(float)
        cnt = collections.Counter()
        for i in range(len(tags) - 1):
            d = (ns[i + 1] - ns[i]) * 1e-3
            a, b = int(tags[i]), int(tags[i + 1])
            if b == a + 1000:
                wait[a] += d
                cnt[a] += 1
            else:
                work[b if b < 1000 else b] += d  # work leading up to arrival at b
        tot = (ns[-1] - ns[0]) * 1e-3
        rows = []
        for k in sorted(set(wait) | set(work)):
            rows.append({"tag": k, "phase": TAGS.get(k, str(k)), "count": cnt.get(k, 0),
                         "wait_us": round(wait.get(k, 0.0), 1), "work_us": round(work.get(k, 0.0), 1)})
        out[name] = {"total_us": round(tot, 1), "entries": int(len(tags)), "phases": rows}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
