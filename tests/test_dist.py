"""CPU (gloo, world size 2): the partitioned hot step of paper_2306_06795_b200.dist
-- patch/row partition, forward halo of x, rank-local Vanka + SpMV, reverse
halo of the Vanka partial sums -- reproduces the single-process result.
The rank-local kernels are the C restatement (oracle/) here, as the checker;
on B200 the same DistStep drives libsag kernels over NCCL."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_2306_06795_b200.dist import DistStep, build_partition

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = dict(np.load(os.path.join(GOLD, name + ".npz")))
        nr, nc = (int(v) for v in g["k0_shape"])
        k0 = O.Csr(nr, nc, g["k0_rp"], g["k0_ci"], g["k0_v"])
        pptr, pidx, vptr, vidx, nx = (g["patch_" + a] for a in ("pptr", "pidx", "vptr", "vidx", "nx"))
        plans = build_partition(world, nr, k0.rp, k0.ci, k0.v, pptr, pidx, vptr, vidx)
        plan = plans[rank]
        lo, hi = plan.patch_lo, plan.patch_hi
        sub = O.Patches((pptr[lo:hi + 1] - pptr[lo]).astype(np.int32), pidx[pptr[lo]:pptr[hi]].copy(),
                        (vptr[lo:hi + 1] - vptr[lo]).astype(np.int32), vidx[vptr[lo]:vptr[hi]].copy(),
                        nx[lo:hi].copy())
        nxyz = [int(v) for v in g["nxyz0"]]
        fv = O.OracleVanka(k0, sub, nxyz[0] + nxyz[1])
        # global PoU weights (the rank's own patches see only part of each
        # boundary dof's multiplicity)
        w = g["factor_weights"]
        C.memmove(fv.f.weights, w.ctypes.data, 8 * nr)
        rows = O.Csr(len(plan.owned), nc, plan.rows_rp, plan.rows_ci, plan.rows_v)

        def local_vanka(x):
            return torch.from_numpy(fv.apply(x.numpy()))

        def local_spmv(x):
            return torch.from_numpy(O.Oracle.spmv(rows, x.numpy()))

        step = DistStep(plan, local_vanka, local_spmv, torch, dist, "cpu")
        x = torch.full((nr,), float("nan"), dtype=torch.float64)
        own = torch.as_tensor(plan.owned, dtype=torch.int64)
        x[own] = torch.from_numpy(g["x"][plan.owned])
        delta, y = step(x)
        q.put((rank, plan.owned, delta.numpy()[plan.owned], y.numpy(), plan.ghost_count()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["th_cavity_8", "th_cavity_16"])
def test_partitioned_step_matches_single_process(name):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    g = dict(np.load(os.path.join(GOLD, name + ".npz")))
    seen = np.zeros(len(g["x"]), dtype=bool)
    for _ in range(world):
        rank, owned, delta, y, ghosts = q.get()
        assert ghosts > 0                       # a real halo exists
        assert not seen[owned].any()            # ownership is a partition
        seen[owned] = True
        assert np.allclose(delta, g["apply_vanka"][owned], rtol=1e-13, atol=1e-15)
        assert np.array_equal(y, g["spmv"][owned])  # same rows, same order
    assert seen.all()


def test_partition_covers_and_is_deterministic():
    from paper_2306_06795_b200.dist import build_partition
    g = dict(np.load(os.path.join(GOLD, "th_cavity_16.npz")))
    nr = int(g["k0_shape"][0])
    args = (nr, g["k0_rp"], g["k0_ci"], g["k0_v"], g["patch_pptr"], g["patch_pidx"],
            g["patch_vptr"], g["patch_vidx"])
    for world in (1, 2, 3, 4):
        a = build_partition(world, *args)
        b = build_partition(world, *args)
        owned = np.concatenate([p.owned for p in a])
        assert np.array_equal(np.sort(owned), np.arange(nr))
        for pa, pb in zip(a, b):
            assert np.array_equal(pa.owned, pb.owned)
            for q in pa.fwd_recv:
                assert np.array_equal(pa.fwd_recv[q], a[q].fwd_send[pa.rank])
            for q in pa.rev_send:
                assert np.array_equal(pa.rev_send[q], a[q].rev_recv[pa.rank])
        if world == 1:
            assert a[0].ghost_count() == 0
