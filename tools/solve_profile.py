#!/usr/bin/env python
"""Time the pieces of a full DC-all FGMRES solve on the GPU (CUDA events on
libsag's stream): one DC preconditioner application (CUDA graph), the whole
solve, per-iteration cost. With --nvtx, a 2-iteration solve runs inside an
NVTX range "solve2" for `ncu --nvtx --nvtx-include solve2/` launch lists.

    python tools/solve_profile.py [n=512] [--config C] [--table] [--solve-table] [--nvtx]
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
from bench import splitmix64_uniform  # noqa: E402


def main():
    n_mesh = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 512
    nvtx = "--nvtx" in sys.argv
    t0 = time.time()
    conf = {}
    if "--config" in sys.argv:  # a bench.py config instead of the TH cavity n
        import bench
        conf = bench.CONFIGS[int(sys.argv[sys.argv.index("--config") + 1])]
        case = bench.host_case(conf)
    else:
        case = HostCase("cavity", False, "structured", n_mesh)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)  # torch-owned: libsag never destroys it
    ctx = S.Context(0, stream=stream.cuda_stream)
    cfg = S.SolverConfig(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500,
                         enclosed_flow=case.enclosed, eta_u=conf.get("eta_u", 1.0),
                         eta_p=conf.get("eta_p", 1.0), omega0=conf.get("omega0", 1.0))
    K0, dc, _ = case.device(cfg, ctx)
    out = {"setup_s": time.time() - t0, "info": dc.info()}
    rhs = case.rhs()
    x, rep = S.solve_stokes(K0, rhs, dc, cfg)  # warm + graph capture
    n = K0.nrows
    r = torch.from_numpy(splitmix64_uniform(n)).to(dev)
    z = torch.empty_like(r)

    def timed(fn, k):
        fn()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / k * 1e3

    out["dc_apply_us"] = timed(lambda: dc.apply(r, out=z), 10)
    out["spmv_k0_us"] = timed(lambda: S.spmv(K0, r, out=z), 20)
    ts = time.perf_counter()
    x, rep = S.solve_stokes(K0, rhs, dc, cfg)
    ctx.synchronize()
    out["solve_s"] = time.perf_counter() - ts
    out["iterations"] = rep.iterations
    out["per_iteration_ms"] = 1e3 * out["solve_s"] / max(rep.iterations, 1)
    out["final_rel"] = rep.final_relative_residual
    l0 = ctx.launch_count()
    S.solve_stokes(K0, rhs, dc, cfg)
    out["launches_per_solve"] = ctx.launch_count() - l0
    if nvtx:
        os.environ["SAG_NO_GRAPH"] = "1"  # individual launches for the profiler
        torch.cuda.nvtx.range_push("dcapply")
        dc.apply(r, out=z)
        ctx.synchronize()
        torch.cuda.nvtx.range_pop()
        cfg2 = S.SolverConfig(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=2, enclosed_flow=True)
        torch.cuda.nvtx.range_push("solve2")
        S.solve_stokes(K0, rhs, dc, cfg2)
        ctx.synchronize()
        torch.cuda.nvtx.range_pop()
    if "--table" in sys.argv:
        os.environ["SAG_NO_GRAPH"] = "1"
        tab = kernel_table(lambda: dc.apply(r, out=z), steps=3)
        out["dc_apply_kernels_us"] = [(k, c, round(t, 1)) for k, c, t in tab]
        os.environ.pop("SAG_NO_GRAPH")
    if "--solve-table" in sys.argv:
        tab = kernel_table(lambda: S.solve_stokes(K0, rhs, dc, cfg), steps=1)
        out["solve_kernels_us"] = [(k, c, round(t, 1)) for k, c, t in tab[:30]]
        out["solve_kernel_sum_us"] = round(sum(t for _, _, t in tab), 1)
    print(json.dumps(out))


def kernel_table(fn, steps=1):
    """Live (warm, concurrent-capable) per-kernel device times via CUPTI
    (torch.profiler), for kernels launched by libsag on its own stream."""
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            fn()
        torch.cuda.synchronize()
    rows = {}
    for e in prof.events():
        if e.device_type.name == "CUDA" or "cuda" in str(e.device_type).lower():
            name = e.name.replace("void ", "").replace("sag::", "")
            name = name.split(">(")[0] + ">" if ">(" in name else name.split("(")[0]
            d = rows.setdefault(name, [0, 0.0])
            d[0] += 1
            d[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    return sorted(((k, v[0], v[1] / steps) for k, v in rows.items()), key=lambda t: -t[2])


if __name__ == "__main__":
    main()
