#!/usr/bin/env python
"""Benchmark of the B200 solve-phase hot path (BASELINE.json metric:
"Vanka sweep + SpMV GDOF/s (frac. of HBM roofline); FGMRES solve s vs CPU").

A step = one additive Vanka sweep (apply_vanka, vanka.cpp:151-184) plus one
CSR SpMV (sparse.cpp:78-91) on the high-order operator K0 of BASELINE config 2
(TH P2/P1 lid-driven cavity, 512x512 structured mesh), input x_i ~ U[-1,1)
from splitmix64. value = total K0 DoFs processed per second
by all ranks (GDOF/s). Inputs (K0 0.48 GB + Vanka factors 1.4 GB) exceed the
126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2]
  python bench.py --impl reference      # the reference's CPU path, host cores

Multi-GPU (torchrun, N > 1; --dist at N = 1): K0's rows and Vanka patches are
partitioned across the ranks in rank-local numbering by libsag's planner with
NCCL halo exchanges, through the C-ABI (sag_dist_*; strong scaling); the line
also carries the distributed FGMRES + DC-all solve (one CUDA graph with the
collectives captured). Times are CUDA events on libsag's stream, max over
ranks.

roofline: the dominant kernel is the Vanka patch kernel; its algorithmic bytes
are those of the representation it streams (factor blobs incl. dof indices,
r once, the local results), `traffic` is ncu's DRAM bytes per launch from the
committed profile (profiles/*/ncu_traffic.json). The SURVEY 8(d) formula
bytes of the whole sweep (reference representation) are reported beside it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    1: dict(workload="th_cavity_64x64", problem="cavity", sv=False, n=64),
    2: dict(workload="th_cavity_512x512", problem="cavity", sv=False, n=512),
    3: dict(workload="sv_cavity_256x256_barycentric", problem="cavity", sv=True, n=256,
            omega0=0.78, eta_p=2.68),
    # jittered Delaunay of a 501x501 grid (251,001 points, jitter 0.3 h, seed 7),
    # zero velocity, f = (sin k1 x, cos k2 y) with k from splitmix64
    4: dict(workload="th_unstructured_251k_forced", problem="cavity", sv=False, n=500,
            mesh="file_forced"),
    # 3D Taylor-Hood cavity on n^3 hexes x 6 tets (no reference support: the
    # kernel-level 3-component Vanka sweep + SpMV, parity against oracle.c's
    # 3-component restatement); n from --n3d
    5: dict(workload="th3d_cavity", problem="cavity", sv=False, n=32, dim=3),
}


def _mesh_file(cfg):
    from paper_2306_06795_b200 import meshgen
    path = os.path.join("/tmp", f"sag_mesh_{cfg['n']}_7_0.3.json")
    if not os.path.exists(path):
        meshgen.write_mesh(path + f".{os.getpid()}", cfg["n"], seed=7, jitter=0.3)
        os.replace(path + f".{os.getpid()}", path)
    return path


def host_case(cfg):
    """The reference-built case of a config (host adapter)."""
    from paper_2306_06795_b200.cases import HostCase
    if cfg.get("mesh") == "file_forced":
        from paper_2306_06795_b200 import meshgen
        k1, k2 = meshgen.force_wavenumbers()
        return HostCase(cfg["problem"], False, "file_forced", 0, mesh_path=_mesh_file(cfg),
                        k1=k1, k2=k2)
    return HostCase(cfg["problem"], cfg["sv"], "structured", cfg["n"])


def ref_case(cfg):
    """The same case built by the reference library in oracle/_ref."""
    import oracle as O
    if cfg.get("mesh") == "file_forced":
        from paper_2306_06795_b200 import meshgen
        k1, k2 = meshgen.force_wavenumbers()
        return O.RefCase.mesh_forced(_mesh_file(cfg), k1, k2)
    return O.RefCase.build(cfg["problem"], cfg["sv"], "structured", cfg["n"])
METRIC = "Vanka sweep + SpMV GDOF/s (frac. of HBM roofline); FGMRES solve s vs CPU"


def splitmix64_uniform(n, seed=0x5EED):
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) ^ np.arange(n, dtype=np.uint64)) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return ((z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) * 2.0 - 1.0


def peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={dev}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                      text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.15)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for name, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


_JSON_FD = None


def quiet_stdout():
    """Route fd 1 to stderr for the whole run (NCCL prints its version banner
    to stdout from inside communicator creation, also for the lazily created
    point-to-point communicators) and keep the original stdout for the one
    JSON line."""
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(obj):
    line = (json.dumps(obj) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(line.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, line)


def dist_setup():
    # keep rank 0's stdout to the one JSON line: NCCL prints its version
    # banner to stdout at NCCL_DEBUG=VERSION/INFO (set SAG_NCCL_DEBUG to see it)
    os.environ["NCCL_DEBUG"] = os.environ.get("SAG_NCCL_DEBUG", "WARN")
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def dist_max(v, ws):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def spmv_bytes(nrows, ncols, nnz):
    # 12 nnz + 4 (n_r + 1) + 8 n_c + 8 n_r
    return 12 * nnz + 4 * (nrows + 1) + 8 * ncols + 8 * nrows


def vanka_bytes(f, tot_idx, n):
    # factors (a_factor + aux) + patch index lists + 24 n
    return f.a_factor_bytes + f.aux_bytes + 4 * tot_idx + 24 * n


def vanka_patch_bytes(f, n):
    # the patch kernel's own stream: blobs (factors, headers, dof indices),
    # r (each entry once), one local result per slot
    return f.device_bytes + 8 * n + 8 * f.nslots


def ncu_traffic(workload, kernel):
    """DRAM bytes per launch of `kernel` ("vanka_patch": the patch stage's
    kernels of one sweep, "vanka_gather", "spmv") on `workload` (and level)
    from the newest committed ncu capture (profiles/<round>/ncu_traffic.json,
    {"workloads": {workload: {kernel: bytes}}}), or None when no capture of
    that kernel on that workload exists."""
    import glob
    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_traffic.json"))):
        try:
            with open(path) as fh:
                d = json.load(fh)
        except Exception:
            continue
        w = d.get("workloads", {}).get(workload, {})
        if kernel in w:
            best = w[kernel]
    return best


def config_dict(cfg, k0):
    """The `config` object, identical in both arms."""
    return {"workload": cfg["workload"], "k0_rows": int(k0.nrows), "k0_nnz": int(k0.nnz)}


def golden_solve(config):
    """The reference's solve_stokes report on this config's exact inputs,
    measured in the build container (tests/golden/fullsize_config<N>.json)."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", f"fullsize_config{config}.json")) as f:
            return json.load(f)["solve"]
    except Exception:
        return None


def host_cpu():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "model": model}


# ------------------------------------------------------------------ CPU legs
def cpu_steps(k0csr, nxyz, steps, threads, budget_s=None):
    """The reference's own spmv + apply_vanka (oracle/_ref) on `threads` host
    threads, each running whole steps. Returns (steps_done, wall_s)."""
    import oracle as O
    rk = O.RefMat.from_csr(O.Csr(k0csr.nrows, k0csr.ncols, k0csr.rp, k0csr.ci, k0csr.v))
    rv = O.RefVanka.build(rk, *nxyz)
    x = splitmix64_uniform(k0csr.nrows)
    rk.spmv(x)
    rv.apply(x)  # warm
    done = [0] * threads
    t0 = time.perf_counter()
    deadline = t0 + budget_s if budget_s else None

    def worker(i):
        todo = steps // threads + (1 if i < steps % threads else 0)
        for _ in range(todo):
            if deadline and time.perf_counter() > deadline and done[i] > 0:
                break
            rv.apply(x)
            rk.spmv(x)
            done[i] += 1

    th = [threading.Thread(target=worker, args=(i,)) for i in range(threads)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return sum(done), time.perf_counter() - t0


def ref_solve_1core(case, cfg, repeats):
    """solve_stokes (preconditioner.cpp:229-259) of the reference (oracle/_ref)
    with DC-all V(1,1), FGMRES(30), rtol 1e-8, pinned to ONE host core (the
    reference is single-threaded): min wall time over `repeats` solves; the
    preconditioner's setup timed apart."""
    import oracle as O
    core = max(os.sched_getaffinity(0))
    prev = os.sched_getaffinity(0)
    os.sched_setaffinity(0, {core})   # the calling thread: taskset -c <core>
    try:
        conf = dict(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500,
                    enclosed_flow=case.enclosed, eta_u=cfg.get("eta_u", 1.0),
                    eta_p=cfg.get("eta_p", 1.0), omega0=cfg.get("omega0", 1.0))
        t0 = time.perf_counter()
        d = O.RefDC(case, conf)
        setup = time.perf_counter() - t0
        rhs = case.rhs()
        times, rep = [], None
        for _ in range(repeats):
            t1 = time.perf_counter()
            _, rep = d.solve(rhs)
            times.append(time.perf_counter() - t1)
    finally:
        os.sched_setaffinity(0, prev)
    return {"solve_s": min(times), "solves_s": times, "repeats": repeats,
            "prec_setup_s": setup, "iterations": rep["iterations"],
            "final_relative_residual": rep["final_relative_residual"],
            "core": core, **host_cpu()}


def run_reference(args, ws, rank):
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    t0 = time.perf_counter()
    case = ref_case(cfg)
    k0 = case.k0().csr()
    setup_s = time.perf_counter() - t0
    threads = os.cpu_count() or 1
    if args.warmup:
        cpu_steps(k0, (case.n_x0, case.n_y0, case.n_p0), threads, threads)
    # one step = `threads` concurrent whole passes (every host thread busy
    # whatever K is), bounded in wall time
    done, wall = cpu_steps(k0, (case.n_x0, case.n_y0, case.n_p0), args.steps * threads, threads,
                           budget_s=45.0)
    val = done * k0.nrows / wall / 1e9
    steps_done = done / threads
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GDOF/s", "n_gpus": ws,
        "steps": args.steps, "steps_done": round(steps_done, 3), "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / max(steps_done, 1e-9),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference build_case cavity + splitmix64 x (SURVEY 8(d))",
        "config": config_dict(cfg, k0),
        "cpu_baseline": {"value": val, "unit": "GDOF/s", "cores": threads, "kind": "reference",
                         "sample": f"{done} whole passes (apply_vanka + spmv on K0), "
                                   f"{threads} threads x independent passes"},
        "e2e": {"value": val, "unit": "GDOF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "setup_s": setup_s, "host": host_cpu(),
    }
    if not args.no_solve:
        # the whole reference solve on one core of this host:
        # config 1 five times, and this config's once
        sol = {"config1": ref_solve_1core(case if args.config == 1 else ref_case(CONFIGS[1]),
                                          CONFIGS[1], 5)}
        if args.config != 1:
            sol[f"config{args.config}"] = ref_solve_1core(case, cfg, 1)
        line["solve"] = sol
    emit(line)


# ------------------------------------------------------- GPU arm, N > 1
def run_dist(args, ws, rank, local):
    """Strong scaling across the ranks of one node through the
    C-ABI (sag_dist_*: the path gpu::DistDCPreconditioner drives): K0's rows
    and Vanka patches partitioned in rank-local numbering by libsag's planner,
    forward / reverse halos and the FGMRES all-reduces over NCCL (NVLink),
    levels below level 0 agglomerated. The step is the partitioned Vanka
    sweep + SpMV; the solve is the whole distributed FGMRES(30) + DC-all as one
    CUDA graph (collectives captured)."""
    import torch
    import torch.distributed as dist

    import paper_2306_06795_b200 as S

    cfg = CONFIGS[args.config]
    if cfg["sv"]:
        raise SystemExit("bench --gpus N: the partitioned path covers Taylor-Hood configs")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    t0 = time.perf_counter()
    case = host_case(cfg)
    k0 = case.k0()
    levels = case.levels()
    host_setup_s = time.perf_counter() - t0
    n = k0.nrows
    stream = torch.cuda.Stream(device=dev)
    ctx = S.Context(local, stream=stream.cuda_stream)
    uid = [S.nccl_unique_id() if rank == 0 else None]
    if ws > 1:
        dist.broadcast_object_list(uid, src=0)
    comm = S.Comm(ctx, ws, rank, nccl_id=uid[0])
    scfg = S.SolverConfig(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500,
                          enclosed_flow=case.enclosed)
    t1 = time.perf_counter()
    ds = S.DistSolver(comm, k0, case.nxyz0, levels, scfg)
    torch.cuda.synchronize(dev)
    setup_gpu_s = time.perf_counter() - t1
    nl = ds.nl
    xg = splitmix64_uniform(n)
    with torch.cuda.stream(stream):
        x = torch.from_numpy(xg[ds.l2g]).to(dev)
        delta = torch.empty(nl, dtype=torch.float64, device=dev)
        y = torch.empty(nl, dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    for _ in range(max(args.warmup, 3)):
        ds.step(x, delta, y)
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local) if rank == 0 else None
    barrier(ws)
    l0n = ctx.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        ds.step(x, delta, y)
    e1.record(stream)
    e1.synchronize()
    launches = ctx.launch_count() - l0n
    t_steps = dist_max(e0.elapsed_time(e1) / 1e3, ws)
    # e2e: this rank's local inputs from pinned host memory, outputs back
    xh = torch.from_numpy(xg[ds.l2g]).pin_memory().numpy()
    dh = torch.empty(nl, dtype=torch.float64).pin_memory().numpy()
    yh = torch.empty(nl, dtype=torch.float64).pin_memory().numpy()
    ke = max(args.steps // 4, 5)
    for _ in range(2):
        ds.step(xh, dh, yh)
    barrier(ws)
    te0 = time.perf_counter()
    for _ in range(ke):
        ds.step(xh, dh, yh)
    t_e2e = dist_max((time.perf_counter() - te0) / ke, ws)
    clk = clocks.stop() if clocks else None
    solve = None
    if not args.no_solve:
        rhs = case.rhs()[ds.l2g]
        ds.solve(rhs)  # warm-up: graph capture
        torch.cuda.synchronize(dev)
        barrier(ws)
        ts = time.perf_counter()
        xs, rep = ds.solve(rhs)
        t_solve = dist_max(time.perf_counter() - ts, ws)
        g = golden_solve(args.config)
        solve = {"gpu_s": t_solve, "iterations": rep.iterations,
                 "final_relative_residual": rep.final_relative_residual,
                 "converged": rep.converged, "setup_s": setup_gpu_s,
                 "path": "sag_dist_solve_stokes (partitioned K0/L0, agglomerated levels >= 1, "
                         "NCCL all-reduces and halos, one CUDA graph)"}
        if g:
            solve["reference"] = {k: g[k] for k in ("iterations", "cpu_s_1core",
                                                    "final_relative_residual")}
    ghosts = dist_max(float(ds.ghosts), ws)
    own_max = dist_max(float(ds.n_own), ws)
    if rank == 0:
        peak, peak_kind = peak_hbm()
        out = {
            "metric": METRIC, "value": n / (t_steps / args.steps) / 1e9, "unit": "GDOF/s",
            "n_gpus": ws, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": 1e3 * t_steps / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: reference build_case cavity + splitmix64 x (SURVEY 8(d))",
            "config": config_dict(cfg, k0),
            "layout": {"parallelism": f"row/patch partition x{ws}, NCCL halos (sag_dist)",
                       "max_owned_dofs_per_rank": int(own_max),
                       "max_ghost_dofs_per_rank": int(ghosts),
                       "l2": "inputs exceed L2; no flush"},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "kernel": "partitioned step (Vanka sweep + SpMV)",
                         "achieved": None, "peak": peak, "unit": "GB/s", "frac": None,
                         "traffic": None, "peak_kind": peak_kind,
                         "note": "per-kernel roofline: the single-GPU line (bench.py without "
                                 "--dist); the partitioned kernels are the same kernels"},
            "e2e": {"value": n / t_e2e / 1e9, "unit": "GDOF/s",
                    "h2d_bytes_per_step": 8 * nl, "d2h_bytes_per_step": 16 * nl,
                    "call": "sag_dist_step, pinned host buffers (rank-local vectors)"},
            "setup": {"host_reference_setup_s": host_setup_s, "gpu_setup_s": setup_gpu_s},
        }
        if solve:
            out["solve"] = solve
        if clk:
            out["clocks"] = clk
        emit(out)
    del ds, comm


# ------------------------------------------------------------------ GPU arm
def level_measure(S, ctx, timed, k, nxyz, sv_triples, kper):
    """One level's Vanka sweep and SpMV on the device (splitmix64 input):
    times (CUDA events), SURVEY 8(d) formula bytes, the patch stage's
    representation bytes and its launch classes."""
    import torch
    dev = torch.device("cuda", ctx.device)
    K = S.SparseMatrix.from_csr(k, ctx)
    p = S.build_patches(K, *nxyz, sv_triples=sv_triples)
    f = S.factor_patches(K, p, nxyz[0] + nxyz[1])
    n = k.nrows
    x = torch.from_numpy(splitmix64_uniform(n)).to(dev)
    d = torch.empty_like(x)
    y = torch.empty_like(x)
    lib = S.lib()
    xp, dp = S.C.c_void_p(x.data_ptr()), S.C.c_void_p(d.data_ptr())
    for _ in range(3):
        S.apply_vanka(f, x, out=d)
        S.spmv(K, x, out=y)
    t_patch = timed(lambda: S._check(lib.sag_apply_vanka_stage(ctx.h, f.h, xp, dp, 1)), kper) / kper
    t_gather = timed(lambda: S._check(lib.sag_apply_vanka_stage(ctx.h, f.h, xp, dp, 2)), kper) / kper
    t_vanka = timed(lambda: S.apply_vanka(f, x, out=d), kper) / kper
    t_spmv = timed(lambda: S.spmv(K, x, out=y), kper) / kper
    tot_idx = p.total_velocity + p.total_pressure
    b_v = vanka_bytes(f, tot_idx, n)
    b_p = vanka_patch_bytes(f, n)
    b_s = spmv_bytes(n, n, k.nnz)
    cls = f.classes()
    return {"rows": n, "nnz": int(k.nnz), "patches": f.npatch,
            "vanka_sweep_us": 1e6 * t_vanka, "vanka_patch_us": 1e6 * t_patch,
            "vanka_gather_us": 1e6 * t_gather, "spmv_us": 1e6 * t_spmv,
            "vanka_gdofs": n / t_vanka / 1e9, "spmv_gdofs": n / t_spmv / 1e9,
            "vanka_sweep_formula_bytes": b_v, "vanka_sweep_formula_gbs": b_v / t_vanka / 1e9,
            "vanka_patch_bytes": b_p, "vanka_patch_gbs": b_p / t_patch / 1e9,
            "spmv_bytes": b_s, "spmv_gbs": b_s / t_spmv / 1e9,
            "patch_classes": [{"kernel": c[0], "patches": c[3], "blob_bytes": c[4]} for c in cls],
            "_f": f, "_K": K, "_x": x}


def run_ours(args, ws, rank, local):
    import torch

    import paper_2306_06795_b200 as S

    cfg = CONFIGS[args.config]
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    t0 = time.perf_counter()
    case = host_case(cfg)
    k0 = case.k0()
    host_setup_s = time.perf_counter() - t0
    # libsag launches on a torch-owned stream: tensors, NCCL work and libsag
    # kernels share it, and tearing the context down never destroys a stream
    # torch still references
    stream = torch.cuda.Stream(device=dev)
    ctx = S.Context(local, stream=stream.cuda_stream)
    t1 = time.perf_counter()
    K0 = S.SparseMatrix.from_csr(k0, ctx)
    patches = S.build_patches(K0, *case.nxyz0, sv_triples=case.sv)
    f = S.factor_patches(K0, patches, case.n_x0 + case.n_y0)
    ctx.synchronize()
    factor_s = time.perf_counter() - t1
    n = k0.nrows
    x_host = splitmix64_uniform(n)
    x = torch.from_numpy(x_host).to(dev)
    delta = torch.empty(n, dtype=torch.float64, device=dev)
    y = torch.empty(n, dtype=torch.float64, device=dev)

    def step():
        S.apply_vanka(f, x, out=delta)
        S.spmv(K0, x, out=y)

    def timed(fn, k):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / 1e3

    for _ in range(max(args.warmup, 3)):
        step()
    ctx.synchronize()
    clocks = ClockSampler(local)
    barrier(ws)
    ctx.synchronize()
    launches0 = ctx.launch_count()
    t_steps = timed(step, args.steps)
    launches = ctx.launch_count() - launches0
    ctx.synchronize()
    barrier(ws)
    t_steps = dist_max(t_steps, ws)

    # per-level breakdown (same stream, CUDA events): K0 and ISO0, level 0 of
    # the low-order hierarchy (for SV the level with the most Vanka bytes)
    kper = max(args.steps // 2, 10)
    lv = {"K0": level_measure(S, ctx, timed, k0, case.nxyz0, case.sv, kper)}
    if not args.no_levels:
        iso0, _, nxyz1 = case.level(0)
        lv["ISO0"] = level_measure(S, ctx, timed, iso0, nxyz1, False, kper)
        del iso0
    clk = clocks.stop()

    # e2e: the same step through the C-ABI with pinned HOST buffers, every step
    # x host->device and delta, y device->host: sag_vanka_spmv (x crosses the
    # link once, y's copy overlaps the sweep) and, for comparison, the two
    # reference-shaped calls sag_apply_vanka + sag_spmv (x copied twice)
    xh = torch.from_numpy(x_host).pin_memory().numpy()
    dh = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    yh = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    ke = max(args.steps // 4, 5)

    def e2e(fn):
        for _ in range(2):
            fn()
        barrier(ws)
        te0 = time.perf_counter()
        for _ in range(ke):
            fn()
        return dist_max((time.perf_counter() - te0) / ke, ws)

    t_e2e = e2e(lambda: S.vanka_spmv_step(f, K0, xh, dh, yh))
    step_plan = S.vanka_step_plan(f)  # which form the first call's timing chose
    # the same call with the stage pipeline forced on (8 stages) and off (x in,
    # then compute + chunked copies out)
    os.environ["SAG_STEP_STAGES"] = "8"
    t_e2e8 = e2e(lambda: S.vanka_spmv_step(f, K0, xh, dh, yh))
    os.environ["SAG_STEP_STAGES"] = "1"
    t_e2e1 = e2e(lambda: S.vanka_spmv_step(f, K0, xh, dh, yh))
    del os.environ["SAG_STEP_STAGES"]
    t_e2e2 = e2e(lambda: (S.apply_vanka(f, xh, out=dh), S.spmv(K0, xh, out=yh)))

    peak, peak_kind = peak_hbm()
    L0 = lv["K0"]
    t_patch = L0["vanka_patch_us"] * 1e-6
    b_p = L0["vanka_patch_bytes"]
    ms_step = 1e3 * t_steps / args.steps
    value = ws * n / (t_steps / args.steps) / 1e9
    cls = L0["patch_classes"]
    kname = " + ".join(f"{c['kernel']} x{c['patches']}" for c in cls)
    wl = cfg["workload"]
    levels_out = {}
    for name, m in lv.items():
        mm = {k: v for k, v in m.items() if not k.startswith("_")}
        mm["vanka_patch_frac"] = mm["vanka_patch_gbs"] / peak
        mm["spmv_frac"] = mm["spmv_gbs"] / peak
        key = wl if name == "K0" else f"{wl}/{name}"
        mm["vanka_patch_traffic"] = ncu_traffic(key, "vanka_patch")
        mm["vanka_gather_traffic"] = ncu_traffic(key, "vanka_gather")
        mm["spmv_traffic"] = ncu_traffic(key, "spmv")
        levels_out[name] = mm
    out = {
        "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": ws, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference build_case cavity + splitmix64 x (SURVEY 8(d))",
        "config": config_dict(cfg, k0),
        "layout": {"patches": f.npatch, "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU",
                   "l2": "inputs (K0 + factors > 1 GB) exceed the 126 MB L2; no flush"},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": f"Vanka patch stage on K0: {kname}",
                     "achieved": b_p / t_patch / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": b_p / t_patch / 1e9 / peak,
                     "traffic": ncu_traffic(wl, "vanka_patch"),
                     "algorithmic_bytes": b_p, "peak_kind": peak_kind,
                     "bytes_def": "factor blobs + 8 n (r) + 8 slots (local results)"},
        "levels": levels_out,
        "e2e": {"value": ws * n / t_e2e / 1e9, "unit": "GDOF/s",
                "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 2 * 8 * n,
                "call": "sag_vanka_spmv, pinned host buffers",
                "pipeline": step_plan,
                "pipelined_value": ws * n / t_e2e8 / 1e9,
                "unpipelined_value": ws * n / t_e2e1 / 1e9,
                "two_calls_value": ws * n / t_e2e2 / 1e9,
                "two_calls_note": "sag_apply_vanka + sag_spmv, x copied in twice"},
        "setup": {"host_reference_setup_s": host_setup_s, "gpu_patch_factor_s": factor_s},
    }
    if clk:
        out["clocks"] = clk
    del lv, L0

    if not args.no_solve:
        scfg = S.SolverConfig(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500,
                              enclosed_flow=case.enclosed, eta_u=cfg.get("eta_u", 1.0),
                              eta_p=cfg.get("eta_p", 1.0), omega0=cfg.get("omega0", 1.0))
        K0s, dc, _ = case.device(scfg, ctx)
        rhs = case.rhs()
        S.solve_stokes(K0s, rhs, dc, scfg)  # warm (graph capture)
        barrier(ws)
        ts = time.perf_counter()
        xs, rep = S.solve_stokes(K0s, rhs, dc, scfg)
        t_solve = dist_max(time.perf_counter() - ts, ws)
        # one DC-all application (preconditioner.cpp:114-153) on the device
        r = torch.from_numpy(splitmix64_uniform(n)).to(dev)
        z = torch.empty_like(r)
        dc.apply(r, out=z)
        t_apply = timed(lambda: dc.apply(r, out=z), 10) / 10
        g = golden_solve(args.config)
        out["solve"] = {"gpu_s": t_solve, "iterations": rep.iterations,
                        "ms_per_iteration": 1e3 * t_solve / max(rep.iterations, 1),
                        "dc_apply_ms": 1e3 * t_apply,
                        "final_relative_residual": rep.final_relative_residual,
                        "converged": rep.converged, "dc_info": dc.info()}
        if g:
            out["solve"]["reference"] = {
                "iterations": g["iterations"],
                "final_relative_residual": g["final_relative_residual"],
                "cpu_s_1core": g["cpu_s_1core"],
                "note": "reference solve_stokes on these inputs, 1 core of the build "
                        "container (tests/golden/fullsize_config<N>.json); the reference "
                        "arm (--impl reference) re-times it on this host"}

    if rank == 0 and ws == 1 and not args.no_setup and not case.sv:
        # the low-order hierarchy built by the reference (host) and with the
        # setup's strength graphs and sparse products on the device
        # (gpu::build_monolithic_hierarchy), compared bitwise
        out["setup"]["hierarchy"] = case.hierarchy_gpu(local)
    if rank == 0 and ws == 1 and not args.no_setup:
        # FEM assembly (sys0, quadrisect + sys1, K0) again on the device,
        # compared with the reference-built systems field by field
        out["setup"]["fem_assembly"] = case.assembly_gpu(local)

    if rank == 0 and ws == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        done, wall = cpu_steps(k0, case.nxyz0, 4 * threads, threads, budget_s=20.0)
        cpuv = done * n / wall / 1e9
        out["cpu_baseline"] = {"value": cpuv, "unit": "GDOF/s", "cores": threads,
                               "kind": "reference",
                               "sample": f"{done} whole steps (apply_vanka + spmv on K0) of the "
                                         f"reference build (oracle/_ref), {threads} threads"}
    if rank == 0:
        emit(out)


def run_3d(args, ws, rank, local):
    """Config 5 at the kernel level: one 3-component Vanka sweep
    (sag_apply_vanka3, CTA per patch) + one SpMV on the 3D K0 (mesh3d)."""
    import torch

    import oracle as O
    import paper_2306_06795_b200 as S
    from paper_2306_06795_b200 import mesh3d

    n3 = args.n3d
    t0 = time.perf_counter()
    N, rp, ci, v, nxyz, rhs = mesh3d.k0_csr(n3)
    host_setup_s = time.perf_counter() - t0
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    ctx = S.Context(local, stream=stream.cuda_stream)
    k = O.Csr(N, N, rp, ci, v)
    K = S.SparseMatrix.from_csr(k, ctx)
    t1 = time.perf_counter()
    f = S.VankaFactorization3(K, *nxyz)
    ctx.synchronize()
    factor_s = time.perf_counter() - t1
    xh = splitmix64_uniform(N)
    with torch.cuda.stream(stream):
        x = torch.from_numpy(xh).to(dev)
        d = torch.empty_like(x)
        y = torch.empty_like(x)
    torch.cuda.synchronize(dev)

    def step():
        f.apply(x, out=d)
        S.spmv(K, x, out=y)

    def timed(fn, kk):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(kk):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / 1e3

    for _ in range(max(args.warmup, 3)):
        step()
    ctx.synchronize()
    clocks = ClockSampler(local)
    l0 = ctx.launch_count()
    t_steps = timed(step, args.steps)
    launches = ctx.launch_count() - l0
    kper = max(args.steps // 2, 10)
    t_v = timed(lambda: f.apply(x, out=d), kper) / kper
    t_s = timed(lambda: S.spmv(K, x, out=y), kper) / kper
    clk = clocks.stop()
    xp = torch.from_numpy(xh).pin_memory().numpy()
    dp = torch.empty(N, dtype=torch.float64).pin_memory().numpy()
    yp = torch.empty(N, dtype=torch.float64).pin_memory().numpy()
    for _ in range(2):
        f.apply(xp, out=dp)
        S.spmv(K, xp, out=yp)
    ke = max(args.steps // 4, 5)
    te = time.perf_counter()
    for _ in range(ke):
        f.apply(xp, out=dp)
        S.spmv(K, xp, out=yp)
    t_e2e = (time.perf_counter() - te) / ke
    peak, peak_kind = peak_hbm()
    b_v = f.device_bytes + 8 * N + 8 * f.nslots + 4 * f.nslots + 4 * (N + 1) + 8 * N
    b_s = spmv_bytes(N, N, int(rp[-1]))
    out = {
        "metric": METRIC, "value": N / (t_steps / args.steps) / 1e9, "unit": "GDOF/s",
        "n_gpus": 1, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": 1e3 * t_steps / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: 3D TH cavity {n3}^3 x 6 tets (mesh3d), splitmix64 x",
        "config": {"workload": f"th3d_cavity_{n3}x{n3}x{n3}", "k0_rows": N,
                   "k0_nnz": int(rp[-1])},
        "layout": {"patches": f.npatch, "max_patch_velocity_dofs": f.max_nv,
                   "velocity_dofs": int(sum(nxyz[:3])), "pressure_dofs": int(nxyz[3])},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": "apply3_kernel + gather (CTA per patch)",
                     "achieved": b_v / t_v / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": b_v / t_v / 1e9 / peak, "traffic": None, "peak_kind": peak_kind,
                     "algorithmic_bytes": b_v,
                     "bytes_def": "blobs (3 inverse blocks, U_hat, B_hat, S^-1, dofs) + r + "
                                  "slots written, slot ids and results read, delta"},
        "kernels": {"vanka3_sweep_us": 1e6 * t_v, "spmv_us": 1e6 * t_s,
                    "vanka3_gdofs": N / t_v / 1e9, "spmv_gdofs": N / t_s / 1e9,
                    "spmv_frac": b_s / t_s / 1e9 / peak},
        "e2e": {"value": N / t_e2e / 1e9, "unit": "GDOF/s", "h2d_bytes_per_step": 16 * N,
                "d2h_bytes_per_step": 16 * N,
                "call": "sag_apply_vanka3 + sag_spmv, pinned host buffers"},
        "setup": {"host_assembly_s": host_setup_s, "gpu_factor_s": factor_s},
    }
    if clk:
        out["clocks"] = clk
    if not args.no_cpu:
        ref = O.OracleVanka3(k, *nxyz)
        t2 = time.perf_counter()
        ref.apply(xh)
        O.Oracle.spmv(k, xh)
        cpu = time.perf_counter() - t2
        out["cpu_baseline"] = {"value": N / cpu / 1e9, "unit": "GDOF/s", "cores": 1,
                               "kind": "port",
                               "sample": "one sweep + SpMV of oracle.c's 3-component restatement "
                                         "(the reference has no 3D path)"}
    emit(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--n3d", type=int, default=32, help="config 5: hexes per side")
    ap.add_argument("--no-levels", action="store_true",
                    help="skip the ISO0 level measurement")
    ap.add_argument("--no-setup", action="store_true",
                    help="skip the device-assisted hierarchy setup measurement")
    ap.add_argument("--dist", action="store_true",
                    help="use the partitioned (halo-exchange) step even at N = 1")
    args = ap.parse_args()
    quiet_stdout()
    ws, rank, local = dist_setup()
    if args.impl == "reference" and args.config == 5:
        emit({"impl": "reference", "unavailable": "the reference has no 3D path (SPEC.md:8)"})
    elif args.impl == "reference":
        run_reference(args, ws, rank)
    elif args.config == 5:
        run_3d(args, ws, rank, local)
    elif ws > 1 or args.dist:
        run_dist(args, ws, rank, local)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
