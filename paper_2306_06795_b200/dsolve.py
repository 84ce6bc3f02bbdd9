"""Distributed solve_stokes: FGMRES(m) with the DC-all preconditioner over a
row/patch partition, one process per GPU.

Per rank (partition.RankSystem, rank-local numbering):
  * K0 and the low-order level 0 (L0, same dofs) are distributed: SpMV over
    the owned rows, Vanka over the rank's own patches with the global
    partition-of-unity weights, halo exchanges with the neighbours only
    (forward: owned values to the ranks that read them as ghosts; reverse:
    partial Vanka sums at ghosts, added by the owner in rank order);
  * the coarser levels are agglomerated: the restriction is a partial
    (P0 restricted to the owned rows)^T r on every rank followed by an
    all-reduce of the level-1 vector (1.3 MB at config 2), the V-cycle below
    level 0 runs replicated (libsag's device V-cycle, the coarsest pinned with
    the norm of L0 as preconditioner.cpp:49-53 does), and the prolongation is
    the owned rows of P0;
  * FGMRES dots and norms are masked partial reductions + an all-reduce of
    one scalar; every scalar stays in device memory (reduction -> all-reduce
    -> axpy is stream-ordered); the host reads one column of the Hessenberg
    matrix per Arnoldi step and runs the Givens rotations itself, in the
    reference's operation order (krylov.cpp:75-100).
Summation order differs from one process only where partial sums from
several ranks meet (dots, the reverse halo, the restriction); at one rank the
operations are the single-GPU ones.

The kernels come from a backend: :class:`LibsagBackend` (libsag's sm_100a
kernels through the C-ABI, the product path) or, in the CPU tests, a checker
backend supplied by the tests. Communication is a :class:`Comm` over
torch.distributed (NCCL on B200; gloo staged through host memory when
several ranks share one device, and in the CPU tests).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np


# ----------------------------------------------------------------- comm --
class Comm:
    """torch.distributed point-to-point + all-reduce on backend vectors.
    stage=True copies device tensors through host memory (gloo)."""

    def __init__(self, dist, torch, stage=False):
        self.dist, self.torch, self.stage = dist, torch, stage
        self.rank = dist.get_rank()
        self.size = dist.get_world_size()

    def _host(self, t):
        return t.cpu() if (self.stage and t.is_cuda) else t

    def allreduce(self, t, op="sum"):
        if self.size == 1:
            return t
        o = self.dist.ReduceOp.SUM if op == "sum" else self.dist.ReduceOp.MAX
        h = self._host(t)
        self.dist.all_reduce(h, op=o)
        if h is not t:
            t.copy_(h)
        return t

    def all_gather_object(self, obj):
        if self.size == 1:
            return [obj]
        out = [None] * self.size
        self.dist.all_gather_object(out, obj)
        return out

    def barrier(self):
        if self.size > 1:
            self.dist.barrier()

    def fence(self, flag):
        """Every rank's preceding work on its stream is complete before any
        rank's following work: NCCL -- an all-reduce of one element, ordered
        on the device; gloo -- stream synchronisation and a barrier."""
        if self.size == 1:
            return
        if self.stage:
            self.torch.cuda.current_stream().synchronize()
            self.dist.barrier()
        else:
            self.dist.all_reduce(flag)

    def start(self, sends: dict, recvs: dict):
        """Posts a grouped point-to-point exchange (sends: q -> tensor to send;
        recvs: q -> tensor to receive into). With NCCL the transfers run on
        NCCL's stream while the caller keeps launching work on its own."""
        if not sends and not recvs:
            return None
        ops, back = [], []
        for q in sorted(sends):
            ops.append(self.dist.P2POp(self.dist.isend, self._host(sends[q]).contiguous(), q))
        for q in sorted(recvs):
            h = self._host(recvs[q])
            if h is not recvs[q]:
                back.append((recvs[q], h))
            ops.append(self.dist.P2POp(self.dist.irecv, h, q))
        return self.dist.batch_isend_irecv(ops), back

    def finish(self, handle):
        """Completes an exchange: the caller's stream waits for it (NCCL), the
        staged receives are copied back (gloo)."""
        if handle is None:
            return
        reqs, back = handle
        for req in reqs:
            req.wait()
        for dst, h in back:
            dst.copy_(h)



# -------------------------------------------------------------- backend --
class LibsagBackend:
    """Rank-local kernels on the GPU: libsag (include/sag.h) on device
    pointers of torch tensors, all on the context's (torch-owned) stream."""

    def __init__(self, ctx, device, torch, stream=None):
        """stream: the torch.cuda.Stream libsag's context launches on (needed
        to capture the preconditioner into a CUDA graph)."""
        from . import lib, _check  # noqa: F401  (fails loudly without libsag)
        self.ctx, self.device, self.torch = ctx, device, torch
        self.stream = stream
        self.L, self._check = lib(), _check
        import ctypes as C
        self.C = C

    # allocation / transfer
    def vec(self, n):
        return self.torch.zeros(max(n, 1), dtype=self.torch.float64, device=self.device)[:n]

    def ivec(self, a):
        return self.torch.as_tensor(np.asarray(a, dtype=np.int32), device=self.device)

    def u8(self, a):
        return self.torch.as_tensor(np.asarray(a, dtype=np.uint8), device=self.device)

    def from_host(self, a):
        return self.torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=self.device)

    def to_host(self, t):
        return t.cpu().numpy()

    def p(self, t):
        return self.C.c_void_p(t.data_ptr()) if t is not None else None

    # setup objects
    def matrix(self, nrows, ncols, rp, ci, v):
        from . import SparseMatrix
        return SparseMatrix(nrows, ncols, rp, ci, v, self.ctx)

    def vanka(self, nl, ext, patches, n_u, weights):
        from . import Patches, SparseMatrix, factor_patches
        k = SparseMatrix(nl, nl, *ext, ctx=self.ctx)
        pt = Patches.from_lists(*patches, ctx=self.ctx)
        f = factor_patches(k, pt, n_u)
        f.set_weights(weights)
        return f

    def coarse(self, levels, cfg, norm0):
        """The agglomerated V-cycle below level 0: libsag's device V-cycle
        (HoAmgPreconditioner form: one V-cycle of `levels` from x = 0)."""
        from . import HoAmgPreconditioner, SparseMatrix
        lv = [(SparseMatrix.from_csr(k, self.ctx),
               SparseMatrix.from_csr(p, self.ctx) if p is not None else None, nxyz)
              for k, p, nxyz in levels]
        h = HoAmgPreconditioner(lv[0][0], lv, cfg)
        if cfg.enclosed_flow:
            self._check(self.L.sag_dc_set_coarse_pin(self.ctx.h, h.h, self.C.c_double(norm0)))
        return h

    def norm_inf(self, m):
        out = self.C.c_double()
        self._check(self.L.sag_matrix_norm_inf(self.ctx.h, m.h, self.C.byref(out)))
        return out.value

    # kernels
    def spmv(self, m, x, y, epi="store", aux=None):
        e = {"store": 0, "resid": 1, "add": 2}[epi]
        self._check(self.L.sag_spmv_fused(self.ctx.h, m.h, self.p(x), self.p(y), self.p(aux), e))

    def vanka_apply(self, f, r, delta):
        self._check(self.L.sag_apply_vanka(self.ctx.h, f.h, self.p(r), self.p(delta)))

    def vanka_add(self, f, r, x):
        self._check(self.L.sag_apply_vanka_add(self.ctx.h, f.h, self.p(r), self.p(x),
                                               self.C.c_double(1.0)))

    def coarse_apply(self, h, b, x):
        self._check(self.L.sag_dc_apply(self.ctx.h, h.h, self.p(b), self.p(x)))

    def dot(self, a, b, mask, out):
        self._check(self.L.sag_dot_async(self.ctx.h, a.numel(), self.p(a), self.p(b),
                                         self.p(mask), self.p(out)))

    def axpy_s(self, s, sign, x, y):
        self._check(self.L.sag_axpy_async(self.ctx.h, y.numel(), self.p(s), float(sign),
                                          self.p(x), self.p(y)))

    def div_s(self, x, s, take_sqrt, y):
        self._check(self.L.sag_div_async(self.ctx.h, y.numel(), self.p(x), self.p(s),
                                         int(take_sqrt), self.p(y)))

    def sub_mean(self, x, s, count, y):
        self._check(self.L.sag_sub_mean_async(self.ctx.h, y.numel(), self.p(x), self.p(s),
                                              float(count), self.p(y)))

    def fgmres1_coef(self, ssq_r, h00, ssq_w, y0):
        self._check(self.L.sag_fgmres1_coef_async(self.ctx.h, self.p(ssq_r), self.p(h00),
                                                  self.p(ssq_w), self.p(y0)))

    def axpby(self, a, x, b, y):
        self._check(self.L.sag_axpby_async(self.ctx.h, y.numel(), float(a), self.p(x), float(b),
                                           self.p(y)))

    def gather(self, idx, src, dst):
        self._check(self.L.sag_gather_async(self.ctx.h, idx.numel(), self.p(idx), self.p(src),
                                            self.p(dst)))

    def scatter(self, idx, src, dst, add):
        self._check(self.L.sag_scatter_async(self.ctx.h, idx.numel(), self.p(idx), self.p(src),
                                             self.p(dst), int(add)))

    def raw(self, n):
        """A device buffer of its own allocation (cudaMalloc via sag_alloc): a
        CUDA IPC handle maps the whole allocation, so buffers shared with peer
        ranks must not be sub-allocated by torch's caching allocator."""
        return _RawBuffer(self, n)

    def ipc_handle(self, t):
        h = (self.C.c_ubyte * 64)()
        self._check(self.L.sag_ipc_get_handle(self.ctx.h, self.p(t), h))
        return bytes(h)

    def ipc_open(self, handle: bytes) -> int:
        h = (self.C.c_ubyte * 64).from_buffer_copy(handle)
        ptr = self.C.c_void_p()
        self._check(self.L.sag_ipc_open_handle(self.ctx.h, h, self.C.byref(ptr)))
        return ptr.value

    def vanka_add_push(self, f, r, x, slot, nbr, peers):
        arr = (self.C.c_void_p * max(len(peers), 1))(*peers)
        self._check(self.L.sag_apply_vanka_add_push(self.ctx.h, f.h, self.p(r), self.p(x),
                                                    self.C.c_double(1.0), self.p(slot),
                                                    self.p(nbr), len(peers), arr))

    def push(self, idx, src, peer_ptr: int):
        self._check(self.L.sag_push_async(self.ctx.h, idx.numel(), self.p(idx), self.p(src),
                                          self.C.c_void_p(peer_ptr)))

    def launches(self):
        return self.ctx.launch_count()


# --------------------------------------------------------------- solver --
@dataclass
class DistReport:
    converged: bool
    iterations: int
    final_relative_residual: float
    residual_history: list


class _Level:
    """A distributed level: its local rows split into interior rows (owned
    columns only) and boundary rows, its own Vanka patches split into interior
    patches (owned dofs only) and boundary patches, relaxation workspaces.
    The interior parts run while the halo exchange is in flight."""

    def __init__(self, be, rs, ll, mrelax):
        nl = rs.nl
        self.K_int = be.matrix(nl, nl, *ll.rows_int)
        self.K_bnd = be.matrix(nl, nl, *ll.rows_bnd) if len(ll.rows_bnd[1]) else None
        ext = (ll.ext_rp, ll.ext_ci, ll.ext_v)
        self.f_int = self.f_bnd = None
        if len(ll.patches_int[0]) > 1:
            self.f_int = be.vanka(nl, ext, ll.patches_int, rs.n_u_loc, ll.weights)
        if len(ll.patches_bnd[0]) > 1:
            self.f_bnd = be.vanka(nl, ext, ll.patches_bnd, rs.n_u_loc, ll.weights)
        k = be.matrix(nl, nl, ll.rows_rp, ll.rows_ci, ll.rows_v)
        self.norm_inf_local = be.norm_inf(k)
        del k
        self.kry = _Krylov(be, nl, mrelax)
        self.r = be.vec(nl)
        self.corr = be.vec(nl)


class _Krylov:
    def __init__(self, be, n, m):
        self.m = m
        self.sc = be.vec(m + 4)   # device scalars: ||b||^2, ||r||^2, h column
        self.V = [be.vec(n) for _ in range(m + 1)]
        self.Z = [be.vec(n) for _ in range(m)]
        self.w = be.vec(n)
        self.r = be.vec(n)


class _RawBuffer:
    """n doubles of device memory owned by libsag (numel / data_ptr like a tensor)."""

    def __init__(self, be, n):
        self.be, self.n = be, n
        ptr = be.C.c_void_p()
        be._check(be.L.sag_alloc(be.ctx.h, max(n, 1) * 8, be.C.byref(ptr)))
        be._check(be.L.sag_memcpy(be.ctx.h, ptr, (be.C.c_double * max(n, 1))(), max(n, 1) * 8))
        self.ptr = ptr.value

    def numel(self):
        return self.n

    def data_ptr(self):
        return self.ptr

    def __del__(self):
        try:
            self.be.L.sag_free(self.be.ctx.h, self.be.C.c_void_p(self.ptr))
        except Exception:
            pass


class PeerHalo:
    """The reverse halo over peer memory (the sweep's only collective): each
    rank maps, by CUDA IPC, the receive buffers its neighbours keep for it and
    writes its partial sums at their dofs straight into them (NVLink stores,
    `sag_push_async`); one fence (Comm.fence) orders every rank's stores before
    the owners add them, in rank order. Two buffer sets alternate, so a rank's
    next stores never overwrite sums its neighbour has not added yet (a forward
    halo and a fence separate them)."""

    def __init__(self, rs, be, comm):
        self.be, self.comm = be, comm
        self.recv = [{q: be.raw(len(i)) for q, i in rs.rev_recv.items()} for _ in range(2)]
        mine = {q: [be.ipc_handle(self.recv[k][q]) for k in range(2)] for q in rs.rev_recv}
        allh = comm.all_gather_object(mine)
        self.dst = {q: [be.ipc_open(allh[q][rs.rank][k]) for k in range(2)] for q in rs.rev_send}
        self.flag = be.vec(1)
        self.k = 0
        # per local dof: where its partial sum goes (neighbour index, slot), for
        # the gather that stores straight into the owners' buffers
        self.order = sorted(rs.rev_send)
        slot = np.full(rs.nl, -1, dtype=np.int32)
        nbr = np.zeros(rs.nl, dtype=np.uint8)
        for qi, q in enumerate(self.order):
            slot[rs.rev_send[q]] = np.arange(len(rs.rev_send[q]), dtype=np.int32)
            nbr[rs.rev_send[q]] = qi
        self.fusable = len(self.order) <= 8
        self.slot, self.nbr = be.ivec(slot), be.u8(nbr)
        self.fused = self.unfused = 0   # reverse halos done each way

    def add_push(self, f_bnd, v, z):
        """z += apply_vanka(v) over the boundary patches, each ghost's partial
        sum stored into its owner's buffer by the same kernel; then the fence."""
        self.be.vanka_add_push(f_bnd, v, z, self.slot, self.nbr,
                               [self.dst[q][self.k] for q in self.order])
        self.comm.fence(self.flag)
        self.fused += 1

    def start(self, d, ix_send):
        for q, idx in ix_send.items():
            self.be.push(idx, d, self.dst[q][self.k])
        self.comm.fence(self.flag)
        self.unfused += 1

    def finish(self, d, ix_recv):
        for q in sorted(ix_recv):
            self.be.scatter(ix_recv[q], self.recv[self.k][q], d, True)
        self.k ^= 1

    def close(self):
        """Unmaps the neighbours' buffers (call after a fence: no stores in flight)."""
        for ptrs in self.dst.values():
            for p in ptrs:
                self.be.L.sag_ipc_close_handle(self.be.ctx.h, self.be.C.c_void_p(p))
        self.dst = {}


class DistStep:
    """The partitioned hot step on one rank: the halos, the masked reductions
    and the distributed K0 (local SpMV rows + own Vanka patches).

    step(x, delta, y): delta = apply_vanka(x) (vanka.cpp:151-184) and y = K0 x
    (sparse.cpp:78-91) on the rank's owned dofs -- the bench's unit of work."""

    def __init__(self, rs, be, comm, mrelax=1, peer=None):
        """peer: reverse halo over peer memory (PeerHalo; default from
        SAG_P2P_HALO=1) instead of NCCL send / receive."""
        self.rs, self.be, self.comm = rs, be, comm
        nl = rs.nl
        self.mask = be.u8(rs.owned)
        self.ones = be.from_host(np.ones(nl))
        self.sc = be.vec(4)   # device scalars of the projection
        self._ix = {k: {q: be.ivec(i) for q, i in getattr(rs, k).items()}
                    for k in ("fwd_send", "fwd_recv", "rev_send", "rev_recv")}
        self._buf = {k: {q: be.vec(len(i)) for q, i in getattr(rs, k).items()}
                     for k in ("fwd_send", "fwd_recv", "rev_send", "rev_recv")}
        self.k0 = _Level(be, rs, rs.levels["K0"], mrelax)
        if peer is None:
            peer = os.environ.get("SAG_P2P_HALO") == "1"
        self.peer = PeerHalo(rs, be, comm) if peer and comm.size > 1 else None

    def close(self):
        """Releases the peer-memory halo in the only safe order: a fence (no
        rank's stores are in flight), every rank unmaps its neighbours'
        buffers, a barrier (nobody still maps ours), then our receive buffers
        are freed. Idempotent; also the context-manager exit."""
        if self.peer is None:
            return
        self.comm.fence(self.peer.flag)
        self.be.torch.cuda.synchronize(self.be.device)
        self.peer.close()
        self.comm.barrier()
        self.peer.recv = []
        self.peer = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def step(self, x, delta, y):
        """delta = apply_vanka(x), y = K0 x: interior patches and rows under
        the forward halo, boundary rows under the reverse halo."""
        be, L = self.be, self.k0
        h = self.halo_start(x)
        self._vanka_int(L, x, delta)
        be.spmv(L.K_int, x, y)
        self.halo_finish(h, x)
        h = self._bnd_reduce_start(L, x, delta)
        if L.K_bnd is not None:
            be.spmv(L.K_bnd, x, y, "add")
        self.reduce_finish(h, delta)

    def _bnd_reduce_start(self, L, v, z):
        """z += the boundary patches' contributions, then the reverse halo
        posted; over peer memory the boundary gather itself stores the ghosts'
        partial sums into their owners' buffers (compute + collective in one
        kernel)."""
        if self.peer is not None and L.f_bnd is not None and self.peer.fusable:
            self.peer.add_push(L.f_bnd, v, z)
            return "peer"
        if L.f_bnd is not None:
            self.be.vanka_add(L.f_bnd, v, z)
        return self.reduce_start(z)

    # ---- communication ------------------------------------------------
    def halo_start(self, x):
        """Forward halo, posted: owned values the neighbours read as ghosts."""
        be, ix, buf = self.be, self._ix, self._buf
        for q, i in ix["fwd_send"].items():
            be.gather(i, x, buf["fwd_send"][q])
        return self.comm.start(buf["fwd_send"], buf["fwd_recv"])

    def halo_finish(self, h, x):
        self.comm.finish(h)
        for q in sorted(self._ix["fwd_recv"]):
            self.be.scatter(self._ix["fwd_recv"][q], self._buf["fwd_recv"][q], x, False)

    def reduce_start(self, d):
        """Reverse halo, posted: partial sums at ghosts to their owners."""
        be, ix, buf = self.be, self._ix, self._buf
        if self.peer is not None:
            self.peer.start(d, ix["rev_send"])
            return "peer"
        for q, i in ix["rev_send"].items():
            be.gather(i, d, buf["rev_send"][q])
        return self.comm.start(buf["rev_send"], buf["rev_recv"])

    def reduce_finish(self, h, d):
        """... added by the owner in rank order."""
        if h == "peer":
            self.peer.finish(d, self._ix["rev_recv"])
            return
        self.comm.finish(h)
        for q in sorted(self._ix["rev_recv"]):
            self.be.scatter(self._ix["rev_recv"][q], self._buf["rev_recv"][q], d, True)

    def _norm_inf(self, L):
        t = self.be.from_host(np.array([L.norm_inf_local]))
        self.comm.allreduce(t, "max")
        return float(self.be.to_host(t)[0])

    # ---- reductions into device scalars ---------------------------------
    def dot(self, a, b, s):
        """s (a 1-element device view) = global (a, b) over the owned rows."""
        self.be.dot(a, b, self.mask, s)
        self.comm.allreduce(s)
        return s

    # ---- operators ------------------------------------------------------
    def apply_op(self, L, x, y, epi="store", aux=None):
        """y = K x (store), aux - K x (resid) or y + K x (add) on the owned
        rows; interior rows under the forward halo of x."""
        be = self.be
        h = self.halo_start(x)
        be.spmv(L.K_int, x, y, epi, aux)
        self.halo_finish(h, x)
        if L.K_bnd is not None:
            if epi == "resid":      # boundary rows: y = y - K_b x (y holds aux there)
                be.spmv(L.K_bnd, x, y, "resid", y)
            else:
                be.spmv(L.K_bnd, x, y, "add")

    def _vanka_int(self, L, v, z):
        if L.f_int is not None:
            self.be.vanka_apply(L.f_int, v, z)
        else:
            self.be.axpby(0.0, z, 0.0, z)

    def vanka(self, L, v, z):
        """z = apply_vanka(v) over the partition: interior patches under the
        forward halo, boundary patches added after it, partial sums at ghosts
        to their owners."""
        h = self.halo_start(v)
        self._vanka_int(L, v, z)
        self.halo_finish(h, v)
        h = self._bnd_reduce_start(L, v, z)
        self.reduce_finish(h, z)


class DistSolver(DistStep):
    """solve_stokes (preconditioner.cpp:229-259) with the DC preconditioner
    (preconditioner.cpp:114-153) on one rank of a partition.

    rs: this rank's partition.RankSystem; levels: the global low-order
    hierarchy [(K, P, nxyz), ...] (host CSR) -- level 0 is distributed
    through rs, levels 1.. are agglomerated; cfg: SolverConfig."""

    def __init__(self, rs, levels, cfg, be, comm, peer=None):
        if cfg.variant not in (0, 1, 2):
            raise ValueError("DistSolver: DC-all / DC-LO / DC-HO only")
        mrelax = max(cfg.nu1, cfg.nu2, 1)
        super().__init__(rs, be, comm, mrelax, peer)
        self.cfg = cfg
        nl = rs.nl
        self.l0 = _Level(be, rs, rs.levels["L0"], mrelax)
        self.outer = _Krylov(be, nl, cfg.restart)
        self.din, self.dout = be.vec(nl), be.vec(nl)
        self.t = be.vec(nl)
        self.b0, self.x0 = be.vec(nl), be.vec(nl)
        self.gam_rc, self.gam_e = be.vec(nl), be.vec(nl)
        self.gin, self.gout = be.vec(nl), be.vec(nl)
        # CUDA graph of the preconditioner: NCCL (or a single rank) and
        # sync-free relaxations only; gloo staging synchronises with the host
        self.graph, self.graph_error, self._napply = None, None, 0
        self.stream = getattr(be, "stream", None)
        # (several ranks: collectives inside a captured graph are opt-in,
        # SAG_DIST_GRAPH=1 -- this build has not been run on more than one GPU)
        self.use_graph = (self.stream is not None and not comm.stage
                          and max(cfg.nu1, cfg.nu2) <= 1
                          and (comm.size == 1 or os.environ.get("SAG_DIST_GRAPH") == "1"))
        self.nlev = len(levels)
        norm0 = self._norm_inf(self.l0)
        if self.nlev > 1:
            self.P = be.matrix(nl, rs.n1, rs.p_rp, rs.p_ci, rs.p_v)
            self.R = be.matrix(rs.n1, nl, rs.r_rp, rs.r_ci, rs.r_v)
            self.rc, self.xc = be.vec(rs.n1), be.vec(rs.n1)
            self.coarse = be.coarse(levels[1:], cfg, norm0)
        else:
            # level 0 is the coarsest: agglomerate it whole (every rank solves)
            own = np.nonzero(rs.owned)[0]
            self.own_l = be.ivec(own)
            self.own_g = be.ivec(rs.l2g[own])
            self.l2g = be.ivec(rs.l2g)
            self.tmp = be.vec(len(own))
            self.gb, self.gx = be.vec(rs.n), be.vec(rs.n)
            self.coarse = be.coarse(levels, cfg, norm0)

    # ---- fgmres (krylov.cpp:17-121) ---------------------------------------
    def fgmres(self, L, b, x, prec, tol, max_iters, m, kry, x_zero=False, final=True,
               bd=1e-30):
        """fgmres(matrix_operator(L.K), b, x, prec, {tol, max_iters, restart m})
        (krylov.cpp:17-121); x_zero: x is known to be zero on entry (it is
        zeroed here and r = b exactly, as spmv of a zero vector is zero)."""
        be = self.be
        sc = kry.sc
        host = lambda k0, k1: be.to_host(sc[k0:k1])  # noqa: E731
        self.dot(b, b, sc[0:1])
        bnorm = math.sqrt(float(host(0, 1)[0]))
        ref = bnorm if bnorm > 0.0 else 1.0
        hist = []
        if x_zero:
            be.axpby(0.0, b, 0.0, x)
            be.axpby(1.0, b, 0.0, kry.r)
            be.axpby(1.0, sc[0:1], 0.0, sc[1:2])
            rnorm = bnorm
        else:
            self.apply_op(L, x, kry.r, "resid", b)
            self.dot(kry.r, kry.r, sc[1:2])
            rnorm = math.sqrt(float(host(1, 2)[0]))
        hist.append(rnorm)
        if rnorm / ref <= tol:
            return DistReport(True, 0, rnorm / ref, hist)
        it, converged, first = 0, False, True
        h = np.zeros((m + 1) * m)
        cs, sn = np.zeros(m), np.zeros(m)
        base = 2
        while it < max_iters:
            if not first:   # restart from the true residual (krylov.cpp:43-53)
                self.apply_op(L, x, kry.r, "resid", b)
                self.dot(kry.r, kry.r, sc[1:2])
                rnorm = math.sqrt(float(host(1, 2)[0]))
                if rnorm / ref <= tol:
                    converged = True
                    break
            first = False
            be.div_s(kry.r, sc[1:2], True, kry.V[0])
            g = np.zeros(m + 1)
            g[0] = rnorm
            h[:] = 0.0
            j = 0
            while j < m and it < max_iters:
                prec(kry.V[j], kry.Z[j])
                self.apply_op(L, kry.Z[j], kry.w)
                for i in range(j + 1):  # modified Gram-Schmidt (krylov.cpp:63-67)
                    s = self.dot(kry.w, kry.V[i], sc[base + i:base + i + 1])
                    be.axpy_s(s, -1.0, kry.V[i], kry.w)
                self.dot(kry.w, kry.w, sc[base + j + 1:base + j + 2])
                col = host(base, base + j + 2)
                for i in range(j + 1):
                    h[i * m + j] = col[i]
                wnorm = math.sqrt(float(col[j + 1]))
                h[(j + 1) * m + j] = wnorm
                breakdown = wnorm < bd
                if not breakdown:       # v_(j+1) = w / ||w|| (krylov.cpp:70-73)
                    be.div_s(kry.w, sc[base + j + 1:base + j + 2], True, kry.V[j + 1])
                for i in range(j):      # Givens (krylov.cpp:75-93)
                    t = cs[i] * h[i * m + j] + sn[i] * h[(i + 1) * m + j]
                    h[(i + 1) * m + j] = -sn[i] * h[i * m + j] + cs[i] * h[(i + 1) * m + j]
                    h[i * m + j] = t
                denom = float(np.hypot(h[j * m + j], h[(j + 1) * m + j]))
                if denom > 0.0:
                    cs[j] = h[j * m + j] / denom
                    sn[j] = h[(j + 1) * m + j] / denom
                else:
                    cs[j], sn[j] = 1.0, 0.0
                h[j * m + j] = cs[j] * h[j * m + j] + sn[j] * h[(j + 1) * m + j]
                h[(j + 1) * m + j] = 0.0
                g[j + 1] = -sn[j] * g[j]
                g[j] = cs[j] * g[j]
                it += 1
                rnorm = abs(g[j + 1])
                hist.append(rnorm)
                j += 1
                if rnorm / ref <= tol or breakdown:
                    break
            y = np.zeros(j)             # back substitution (krylov.cpp:102-107)
            for i in range(j - 1, -1, -1):
                acc = g[i]
                for k in range(i + 1, j):
                    acc -= h[i * m + k] * y[k]
                y[i] = acc / h[i * m + i]
            for i in range(j):          # x += y_i z_i (krylov.cpp:108-110)
                be.axpby(float(y[i]), kry.Z[i], 1.0, x)
            if rnorm / ref <= tol:
                converged = True
                break
        final_rel = float("nan")
        if final:                       # final true residual (krylov.cpp:116-119)
            self.apply_op(L, x, kry.r, "resid", b)
            self.dot(kry.r, kry.r, sc[1:2])
            final_rel = math.sqrt(float(host(1, 2)[0])) / ref
            if final_rel <= tol:
                converged = True
        return DistReport(converged, it, final_rel, hist)

    # ---- vanka_relax, Krylov-wrapped (vanka.cpp:199-208) -----------------
    def relax_kw(self, L, x, b, nu, x_zero):
        if nu <= 0:
            if x_zero:
                self.be.axpby(0.0, b, 0.0, x)
            return
        if x_zero:
            r = b                                   # spmv of a zero vector is exactly zero
        else:
            self.apply_op(L, x, L.r, "resid", b)
            r = L.r
        if nu == 1:
            self._relax1(L, x, r, x_zero)
            return
        prec = lambda v, z: self.vanka(L, v, z)  # noqa: E731
        if x_zero:
            self.fgmres(L, r, x, prec, 0.0, nu, nu, L.kry, x_zero=True, final=False)
        else:
            self.fgmres(L, r, L.corr, prec, 0.0, nu, nu, L.kry, x_zero=True, final=False)
            self.be.axpby(1.0, L.corr, 1.0, x)

    def _relax1(self, L, x, r, x_zero):
        """nu = 1: x += y_0 z_0 with the one-step FGMRES on device scalars
        (krylov.cpp:42-110 with m = 1, tol 0): no host synchronisation, so a
        DC application is one stream of kernels and collectives."""
        be, k = self.be, L.kry
        sc = k.sc
        self.dot(r, r, sc[0:1])                       # ||r||^2
        be.div_s(r, sc[0:1], True, k.V[0])            # v_0 = r / ||r||
        self.vanka(L, k.V[0], k.Z[0])                 # z_0 = M v_0
        self.apply_op(L, k.Z[0], k.w)                 # w = K z_0
        self.dot(k.w, k.V[0], sc[1:2])                # h_00
        be.axpy_s(sc[1:2], -1.0, k.V[0], k.w)         # w -= h_00 v_0
        self.dot(k.w, k.w, sc[2:3])                   # ||w||^2 = h_10^2
        be.fgmres1_coef(sc[0:1], sc[1:2], sc[2:3], sc[3:4])
        if x_zero:
            be.axpby(0.0, x, 0.0, x)
        be.axpy_s(sc[3:4], 1.0, k.Z[0], x)            # x += y_0 z_0 (vanka.cpp:208)

    # ---- V-cycle level 0 (preconditioner.cpp:57-81) ---------------------------
    def cycle0(self, b, x, skip_finest):
        cf, be = self.cfg, self.be
        if self.nlev == 1:              # coarsest (preconditioner.cpp:60-63), agglomerated
            be.axpby(0.0, self.gb, 0.0, self.gb)
            be.gather(self.own_l, b, self.tmp)
            be.scatter(self.own_g, self.tmp, self.gb, False)
            self.comm.allreduce(self.gb)
            be.coarse_apply(self.coarse, self.gb, self.gx)
            be.gather(self.l2g, self.gx, x)
            return
        relax = not skip_finest
        pre = relax and cf.nu1 > 0
        if pre:
            self.relax_kw(self.l0, x, b, cf.nu1, True)
            self.apply_op(self.l0, x, self.l0.r, "resid", b)
            r = self.l0.r
        else:
            be.axpby(0.0, b, 0.0, x)
            r = b
        be.spmv(self.R, r, self.rc)                 # partial restriction (owned rows)
        self.comm.allreduce(self.rc)
        be.coarse_apply(self.coarse, self.rc, self.xc)
        be.spmv(self.P, self.xc, x, "add")          # x += P xc on the owned rows
        if relax and cf.nu2 > 0:
            self.relax_kw(self.l0, x, b, cf.nu2, False)

    # ---- DCPreconditioner::apply (preconditioner.cpp:114-153), TH ------------
    def dc_apply(self, r, z):
        cf, be, rs = self.cfg, self.be, self.rs
        nu_loc = rs.n_u_loc
        relax_fine = cf.variant != 1
        pre = relax_fine and cf.nu1 > 0
        x = z
        if pre:
            self.relax_kw(self.k0, x, r, cf.nu1, True)
            self.apply_op(self.k0, x, self.t, "resid", r)
            r1 = self.t
        else:
            be.axpby(0.0, r, 0.0, x)
            r1 = r
        # eta weighting (transfer.cpp:127-135) and TH restriction (copy)
        be.axpby(cf.eta_u, r1[:nu_loc], 0.0, self.b0[:nu_loc])
        be.axpby(cf.eta_p, r1[nu_loc:], 0.0, self.b0[nu_loc:])
        skip = cf.variant == 2
        if cf.gamma <= 1:
            self.cycle0(self.b0, self.x0, skip)
            be.axpby(1.0, self.x0, 1.0, x)          # x += prolong(e) (TH: copy)
        else:
            be.axpby(1.0, self.b0, 0.0, self.gam_rc)
            be.axpby(0.0, self.b0, 0.0, self.gam_e)
            for gi in range(cf.gamma):
                if gi > 0:
                    self.apply_op(self.l0, self.gam_e, self.b0, "resid", self.gam_rc)
                else:
                    be.axpby(1.0, self.gam_rc, 0.0, self.b0)
                self.cycle0(self.b0, self.x0, skip)
                be.axpby(1.0, self.x0, 1.0, self.gam_e)
            be.axpby(1.0, self.gam_e, 1.0, x)
        if relax_fine and cf.nu2 > 0:
            self.relax_kw(self.k0, x, r, cf.nu2, False)

    # ---- solve_stokes (preconditioner.cpp:229-259) --------------------------
    def project(self, src, dst, k):
        """dst = src with the global pressure mean removed (pressure block is
        the local tail [n_u_loc, nl))."""
        nu = self.rs.n_u_loc
        s = self.sc[k:k + 1]
        self.be.dot(src[nu:], self.ones[nu:], self.mask[nu:], s)
        self.comm.allreduce(s)
        if dst is not src:
            self.be.axpby(1.0, src[:nu], 0.0, dst[:nu])
        self.be.sub_mean(src[nu:], s, float(self.rs.n_p), dst[nu:])

    def _prec_body(self):
        """gin -> gout: project, DC apply, project (preconditioner.cpp:241-250)."""
        if self.cfg.enclosed_flow:
            self.project(self.gin, self.din, 0)
            self.dc_apply(self.din, self.dout)
            self.project(self.dout, self.gout, 1)
        else:
            self.dc_apply(self.gin, self.gout)

    def apply_prec(self, v, z):
        """The preconditioner on fixed buffers; with nu = 1 it contains no
        host synchronisation, so after one eager application it is captured
        into a CUDA graph (collectives included) and replayed."""
        be = self.be
        be.axpby(1.0, v, 0.0, self.gin)
        if self.graph is not None:
            self.graph.replay()
        else:
            self._prec_body()
            self._napply += 1
            if self._napply == 1 and self.use_graph:
                self._capture()
        be.axpby(1.0, self.gout, 0.0, z)

    def _capture(self):
        torch = self.be.torch
        g = torch.cuda.CUDAGraph()
        try:
            # relaxed: libsag's pointer-kind queries (cudaPointerGetAttributes)
            # are legal while this thread captures
            with torch.cuda.graph(g, stream=self.stream, capture_error_mode="relaxed"):
                try:
                    self._prec_body()
                except Exception as e:  # noqa: BLE001
                    self.graph_error = repr(e)
                    raise
        except Exception as e:
            self.use_graph = False
            self.graph_error = self.graph_error or repr(e)
            raise RuntimeError("DistSolver: capturing the preconditioner into a CUDA graph "
                               f"failed ({self.graph_error}); set use_graph = False") from e
        self.graph = g

    def solve(self, rhs_local, x):
        """rhs_local: backend vector (nl, owned entries valid); x: output (nl)."""
        cf = self.cfg
        self.be.axpby(0.0, rhs_local, 0.0, x)
        return self.fgmres(self.k0, rhs_local, x, self.apply_prec, cf.tol, cf.max_iters,
                           cf.restart, self.outer, x_zero=True, final=True)
