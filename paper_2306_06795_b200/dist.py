"""Row/patch partition of the hot step across ranks.

Each rank owns a contiguous range of Vanka patches (pressure seeds; the
reference numbers pressure dofs by mesh vertex, so contiguous ranges are
strips of the domain) and the dofs whose lowest-numbered containing patch it
owns. It computes
  * the SpMV rows of its owned dofs, and
  * the additive Vanka contributions of its own patches,
exchanging with its neighbours only
  * forward halo: x at the ghost dofs its rows and patches read, and
  * reverse halo: its partial Vanka sums at dofs owned by other ranks,
over torch.distributed point-to-point (NCCL over NVLink on B200, gloo in the
CPU tests). Vectors stay global-length on every rank (only owned + ghost
entries are meaningful), so the local kernels run unchanged on global
indices. The partition is computed identically on every rank from the
reference-built K0 and its patch lists (no communication to set up).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class RankPlan:
    rank: int
    nranks: int
    n: int
    patch_lo: int
    patch_hi: int
    owned: np.ndarray                    # sorted owned dofs
    rows_rp: np.ndarray                  # CSR of the owned rows (global columns)
    rows_ci: np.ndarray
    rows_v: np.ndarray
    fwd_send: dict = field(default_factory=dict)   # q -> my owned dofs q reads
    fwd_recv: dict = field(default_factory=dict)   # q -> ghost dofs owned by q I read
    rev_send: dict = field(default_factory=dict)   # q -> dofs owned by q my patches touch
    rev_recv: dict = field(default_factory=dict)   # q -> my owned dofs q's patches touch

    def ghost_count(self):
        return int(sum(len(v) for v in self.fwd_recv.values()))


def _patch_dofs(pptr, pidx, vptr, vidx, lo, hi):
    return np.unique(np.concatenate([vidx[vptr[lo]:vptr[hi]], pidx[pptr[lo]:pptr[hi]]]))


def build_partition(nranks: int, n: int, rp, ci, v, pptr, pidx, vptr, vidx):
    """Plans for every rank (deterministic; every rank may call this)."""
    npatch = len(pptr) - 1
    bounds = [(npatch * r) // nranks for r in range(nranks + 1)]
    # owner of a dof: rank of the lowest-numbered patch containing it
    first_patch = np.full(n, np.iinfo(np.int64).max, dtype=np.int64)
    pid_v = np.repeat(np.arange(npatch), np.diff(vptr))
    pid_p = np.repeat(np.arange(npatch), np.diff(pptr))
    np.minimum.at(first_patch, vidx, pid_v)
    np.minimum.at(first_patch, pidx, pid_p)
    owner = np.empty(n, dtype=np.int64)
    has = first_patch != np.iinfo(np.int64).max
    owner[has] = np.searchsorted(np.asarray(bounds[1:]), first_patch[has], side="right")
    # dofs in no patch: by index range
    owner[~has] = np.minimum((np.arange(n)[~has] * nranks) // max(n, 1), nranks - 1)

    plans = []
    reads = []
    touches = []
    for r in range(nranks):
        lo, hi = bounds[r], bounds[r + 1]
        owned = np.nonzero(owner == r)[0]
        # owned rows' CSR
        starts = rp[owned].astype(np.int64)
        lens = rp[owned + 1].astype(np.int64) - starts
        rows_rp = np.zeros(len(owned) + 1, dtype=np.int64)
        np.cumsum(lens, out=rows_rp[1:])
        idx = (np.arange(rows_rp[-1], dtype=np.int64) - np.repeat(rows_rp[:-1], lens)
               + np.repeat(starts, lens))
        rows_rp = rows_rp.astype(np.int32)
        rows_ci = ci[idx].astype(np.int32)
        rows_v = v[idx].astype(np.float64)
        pd = _patch_dofs(pptr, pidx, vptr, vidx, lo, hi)
        need = np.unique(np.concatenate([rows_ci, pd])) if len(pd) or len(rows_ci) else pd
        reads.append(need[owner[need] != r])
        touches.append(pd[owner[pd] != r])
        plans.append(RankPlan(r, nranks, n, lo, hi, owned, rows_rp, rows_ci, rows_v))
    for r in range(nranks):
        g = reads[r]
        for q in np.unique(owner[g]):
            sel = g[owner[g] == q]
            plans[r].fwd_recv[int(q)] = sel
            plans[int(q)].fwd_send[r] = sel
        t = touches[r]
        for q in np.unique(owner[t]):
            sel = t[owner[t] == q]
            plans[r].rev_send[int(q)] = sel
            plans[int(q)].rev_recv[r] = sel
    return plans


def exchange(sends: dict, recvs: dict, src, dst, add: bool, torch, dist):
    """Point-to-point exchange. sends/recvs: q -> index tensors (on src/dst's
    device). add=False: dst[idx] = received; add=True: dst[idx] += received,
    applied in ascending rank order (deterministic)."""
    ops, rbufs = [], {}
    for q in sorted(sends):
        ops.append(dist.P2POp(dist.isend, src.index_select(0, sends[q]).contiguous(), q))
    for q in sorted(recvs):
        rbufs[q] = torch.empty(len(recvs[q]), dtype=src.dtype, device=dst.device)
        ops.append(dist.P2POp(dist.irecv, rbufs[q], q))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for q in sorted(recvs):
        if add:
            dst.index_add_(0, recvs[q], rbufs[q])
        else:
            dst.index_copy_(0, recvs[q], rbufs[q])


class DistStep:
    """One partitioned hot step: delta = apply_vanka(x), y = K0 x, on this
    rank's share. `local_vanka(x_full) -> delta_full` and
    `local_spmv(x_full) -> y_owned` are the rank-local kernels (libsag on
    the GPU)."""

    def __init__(self, plan: RankPlan, local_vanka, local_spmv, torch, dist, device):
        self.plan, self.torch, self.dist = plan, torch, dist
        self.local_vanka, self.local_spmv = local_vanka, local_spmv
        t = lambda a: torch.as_tensor(np.asarray(a, dtype=np.int64), device=device)
        self.fwd_send = {q: t(i) for q, i in plan.fwd_send.items()}
        self.fwd_recv = {q: t(i) for q, i in plan.fwd_recv.items()}
        self.rev_send = {q: t(i) for q, i in plan.rev_send.items()}
        self.rev_recv = {q: t(i) for q, i in plan.rev_recv.items()}

    def halo(self, x):
        exchange(self.fwd_send, self.fwd_recv, x, x, False, self.torch, self.dist)

    def __call__(self, x):
        """x: global-length vector with the owned entries valid. Returns
        (delta with owned entries complete, y for the owned rows)."""
        self.halo(x)
        delta = self.local_vanka(x)
        exchange(self.rev_send, self.rev_recv, delta, delta, True, self.torch, self.dist)
        y = self.local_spmv(x)
        return delta, y
