"""Row/patch partition of the solve across ranks in rank-local numbering
(SURVEY.md 8(e)).

Ownership: rank r owns the contiguous range of Vanka patches [lo_r, hi_r)
(pressure seeds are numbered by mesh vertex, so ranges are strips of the
domain) and every dof whose lowest-numbered K0 patch it owns. The fine levels that live on the n0 dofs --
K0 and, for Taylor-Hood, level 0 of the low-order hierarchy (the P1isoP2/P1
operator on the same dofs, transfer.cpp:97-110) -- are distributed by that
map; the coarser levels are agglomerated (every rank holds them whole).

Rank-local numbering: the rank's local dofs are its owned dofs plus the ghost
dofs that its owned rows and its patches read, numbered in ascending GLOBAL
order. Because the map is monotone,
  * every CSR row keeps its column order, so a local SpMV row sums in the
    reference's order (sparse.cpp:84-87);
  * every patch keeps its sorted velocity list with the x dofs first, so the
    local patch factors are bitwise the global ones (vanka.cpp:88-140);
  * the [x | y | p] block order of the global system (fem.cpp:422-438) holds
    locally too, so velocity/pressure splits are one threshold.
Owned entries are scattered through the local vector; reductions use the
owned mask.

Everything here is host-side integer planning (numpy), computed identically on
every rank from the reference-built global CSR arrays (no communication).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def _ranges(starts, lens):
    """Flat index of the concatenated ranges [starts[i], starts[i] + lens[i])."""
    starts = np.asarray(starts, dtype=np.int64)
    lens = np.asarray(lens, dtype=np.int64)
    tot = int(lens.sum())
    if tot == 0:
        return np.zeros(0, dtype=np.int64)
    off = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    return np.arange(tot, dtype=np.int64) - np.repeat(off[:-1], lens) + np.repeat(starts, lens)


def _rows_of(rp, rows):
    rp = np.asarray(rp, dtype=np.int64)
    rows = np.asarray(rows, dtype=np.int64)
    return _ranges(rp[rows], rp[rows + 1] - rp[rows]), rp[rows + 1] - rp[rows]


def th_patches(rp, ci, n_x, n_y, n_p):
    """build_patches (vanka.cpp:11-42) for one pressure seed per patch, as
    integer host planning: patch i seeds pressure row n_u + i; its velocity
    set is the (sorted, unique -- canonical CSR) columns c < n_u of that row,
    nx = #{c < n_x}. Returns (pptr, pidx, vptr, vidx, nx) int32."""
    n_u = n_x + n_y
    rows = np.arange(n_u, n_u + n_p, dtype=np.int64)
    idx, lens = _rows_of(rp, rows)
    cols = np.asarray(ci)[idx]
    pid = np.repeat(np.arange(n_p, dtype=np.int64), lens)
    keep = cols < n_u
    vidx = cols[keep].astype(np.int32)
    vpid = pid[keep]
    cnt = np.bincount(vpid, minlength=n_p)
    if n_p and (cnt == 0).any():
        bad = int(np.nonzero(cnt == 0)[0][0])
        raise ValueError(f"build_patches: pressure row {bad} couples to no velocity DoFs")
    vptr = np.zeros(n_p + 1, dtype=np.int32)
    np.cumsum(cnt, out=vptr[1:])
    nx = np.bincount(vpid[vidx < n_x], minlength=n_p).astype(np.int32)
    pptr = np.arange(n_p + 1, dtype=np.int32)
    pidx = rows.astype(np.int32)
    return pptr, pidx, vptr, vidx, nx


def pou_weights(n, pidx, vidx):
    """Partition-of-unity weights w_d = 1 / multiplicity (vanka.cpp:67-73)
    over ALL patches of a level (global)."""
    mult = np.bincount(np.concatenate([np.asarray(vidx, dtype=np.int64),
                                       np.asarray(pidx, dtype=np.int64)]), minlength=n)
    mult = mult.astype(np.float64)
    return np.divide(1.0, mult, out=np.zeros(n), where=mult > 0)


@dataclass
class LocalLevel:
    """One distributed level on a rank, in local numbering."""
    rows_rp: np.ndarray      # nl x nl CSR: owned rows complete, ghost rows empty (SpMV)
    rows_ci: np.ndarray
    rows_v: np.ndarray
    ext_rp: np.ndarray       # nl x nl CSR: every local row restricted to local columns
    ext_ci: np.ndarray       #   (the patch blocks K[d_i, d_j] for factoring)
    ext_v: np.ndarray
    patches: tuple           # (pptr, pidx, vptr, vidx, nx) of the rank's own patches, local ids
    weights: np.ndarray      # global PoU weights at the local dofs
    nxyz: tuple              # global (n_x, n_y, n_p) of the level
    # interior / boundary split for overlapping the halo exchanges: interior
    # patches touch owned dofs only, interior rows read owned columns only
    patches_int: tuple = None
    patches_bnd: tuple = None
    rows_int: tuple = None   # (rp, ci, v), nl x nl, boundary rows empty
    rows_bnd: tuple = None   # (rp, ci, v), nl x nl, interior rows empty


@dataclass
class RankSystem:
    rank: int
    nranks: int
    n: int                   # global dofs of the distributed levels
    n_u: int                 # global velocity dofs
    n_p: int                 # global pressure dofs
    l2g: np.ndarray          # local -> global (ascending), int64
    owned: np.ndarray        # uint8 mask over local dofs
    n_u_loc: int             # local velocity dofs (the local [x|y|p] split)
    patch_lo: int
    patch_hi: int
    fwd_send: dict = field(default_factory=dict)   # q -> local ids (owned) q reads
    fwd_recv: dict = field(default_factory=dict)   # q -> local ids (ghosts owned by q)
    rev_send: dict = field(default_factory=dict)   # q -> local ids (ghosts owned by q my patches touch)
    rev_recv: dict = field(default_factory=dict)   # q -> local ids (owned) q's patches touch
    levels: dict = field(default_factory=dict)     # "K0", "L0" -> LocalLevel
    p_rp: np.ndarray = None  # nl x n1 CSR: P0's owned rows, ghost rows empty (prolongation)
    p_ci: np.ndarray = None
    p_v: np.ndarray = None
    r_rp: np.ndarray = None  # n1 x nl CSR: (owned rows of P0)^T (partial restriction)
    r_ci: np.ndarray = None
    r_v: np.ndarray = None
    n1: int = 0

    @property
    def nl(self) -> int:
        return len(self.l2g)

    @property
    def n_own(self) -> int:
        return int(self.owned.sum())

    def ghost_count(self) -> int:
        return self.nl - self.n_own

    def local_of(self, g):
        """Local ids of global dofs g (all must be local)."""
        loc = np.searchsorted(self.l2g, g)
        assert np.array_equal(self.l2g[loc], g)
        return loc


def _owner_map(n, nranks, pptr, pidx, vptr, vidx):
    """Rank of the lowest-numbered patch containing each dof; patch ranges
    [bounds[r], bounds[r + 1]) per rank."""
    npatch = len(pptr) - 1
    bounds = np.array([(npatch * r) // nranks for r in range(nranks + 1)], dtype=np.int64)
    first = np.full(n, np.iinfo(np.int64).max, dtype=np.int64)
    np.minimum.at(first, np.asarray(vidx, dtype=np.int64),
                  np.repeat(np.arange(npatch), np.diff(vptr)))
    np.minimum.at(first, np.asarray(pidx, dtype=np.int64),
                  np.repeat(np.arange(npatch), np.diff(pptr)))
    owner = np.empty(n, dtype=np.int64)
    has = first != np.iinfo(np.int64).max
    owner[has] = np.searchsorted(bounds[1:], first[has], side="right")
    owner[~has] = np.minimum((np.arange(n)[~has] * nranks) // max(n, 1), nranks - 1)
    return owner, bounds


def _patch_dofs(pt, lo, hi):
    pptr, pidx, vptr, vidx, _ = pt
    return np.concatenate([np.asarray(vidx[vptr[lo]:vptr[hi]], dtype=np.int64),
                           np.asarray(pidx[pptr[lo]:pptr[hi]], dtype=np.int64)])


def _local_csr(rp, ci, v, l2g, g2l, rows_mask):
    """nl x nl CSR over local rows (rows_mask: which local rows carry entries),
    columns restricted to local dofs and renumbered (order preserved)."""
    nl = len(l2g)
    sel = np.nonzero(rows_mask)[0]
    idx, lens = _rows_of(rp, l2g[sel])
    cols = g2l[np.asarray(ci)[idx]]
    keep = cols >= 0
    rowid = np.repeat(sel, lens)[keep]
    out_rp = np.zeros(nl + 1, dtype=np.int64)
    np.cumsum(np.bincount(rowid, minlength=nl), out=out_rp[1:])
    return out_rp.astype(np.int32), cols[keep].astype(np.int32), np.asarray(v)[idx][keep].copy()


def build_rank_systems(nranks, k0, l0, p0, nxyz0, nxyz_l0, ranks=None):
    """Plans for the ranks in `ranks` (default: all) of a Taylor-Hood system.

    k0, l0: n x n CSR (objects with rp/ci/v) of K0 and of level 0 of the
    low-order hierarchy (same dofs, transfer.cpp:97-110); p0: its prolongator
    (n x n1) or None when level 0 is the coarsest; nxyz0 / nxyz_l0: block
    sizes. Deterministic: every rank may build every plan."""
    n_x, n_y, n_p = (int(v) for v in nxyz0)
    n = n_x + n_y + n_p
    if tuple(int(v) for v in nxyz_l0) != (n_x, n_y, n_p) or l0.nrows != n:
        raise ValueError("partition: the low-order level 0 must live on the K0 dofs "
                         "(Taylor-Hood transfer)")
    n_u = n_x + n_y
    pk = th_patches(k0.rp, k0.ci, n_x, n_y, n_p)
    pl = th_patches(l0.rp, l0.ci, n_x, n_y, n_p)
    owner, bounds = _owner_map(n, nranks, *pk[:4])
    wk = pou_weights(n, pk[1], pk[3])
    wl = pou_weights(n, pl[1], pl[3])
    ranks = list(range(nranks)) if ranks is None else list(ranks)

    # ghosts of every rank (needed for the peers' send lists)
    need_all, touch_all = [], []
    for r in range(nranks):
        lo, hi = int(bounds[r]), int(bounds[r + 1])
        own = np.nonzero(owner == r)[0]
        cols = [np.asarray(m.ci)[_rows_of(m.rp, own)[0]] for m in (k0, l0)]
        pd = np.concatenate([_patch_dofs(pk, lo, hi), _patch_dofs(pl, lo, hi)])
        need = np.unique(np.concatenate(cols + [pd]).astype(np.int64))
        need_all.append(need[owner[need] != r])
        pdu = np.unique(pd)
        touch_all.append(pdu[owner[pdu] != r])

    out = []
    for r in ranks:
        lo, hi = int(bounds[r]), int(bounds[r + 1])
        own = np.nonzero(owner == r)[0].astype(np.int64)
        l2g = np.union1d(own, need_all[r]).astype(np.int64)
        nl = len(l2g)
        g2l = np.full(n, -1, dtype=np.int64)
        g2l[l2g] = np.arange(nl)
        owned = (owner[l2g] == r).astype(np.uint8)
        rs = RankSystem(r, nranks, n, n_u, n_p, l2g, owned,
                        int(np.searchsorted(l2g, n_u)), lo, hi)
        for q in range(nranks):
            if q == r:
                continue
            g = need_all[r][owner[need_all[r]] == q]
            if len(g):
                rs.fwd_recv[q] = g2l[g].astype(np.int32)
            g = need_all[q][owner[need_all[q]] == r]
            if len(g):
                rs.fwd_send[q] = g2l[g].astype(np.int32)
            g = touch_all[r][owner[touch_all[r]] == q]
            if len(g):
                rs.rev_send[q] = g2l[g].astype(np.int32)
            g = touch_all[q][owner[touch_all[q]] == r]
            if len(g):
                rs.rev_recv[q] = g2l[g].astype(np.int32)
        allrows = np.ones(nl, dtype=bool)
        for name, m, pt, w in (("K0", k0, pk, wk), ("L0", l0, pl, wl)):
            rrp, rci, rv = _local_csr(m.rp, m.ci, m.v, l2g, g2l, owned.astype(bool))
            erp, eci, ev = _local_csr(m.rp, m.ci, m.v, l2g, g2l, allrows)
            pptr, pidx, vptr, vidx, nx = pt
            lp = ((pptr[lo:hi + 1] - pptr[lo]).astype(np.int32),
                  g2l[pidx[pptr[lo]:pptr[hi]]].astype(np.int32),
                  (vptr[lo:hi + 1] - vptr[lo]).astype(np.int32),
                  g2l[vidx[vptr[lo]:vptr[hi]]].astype(np.int32),
                  nx[lo:hi].astype(np.int32))
            assert (lp[1] >= 0).all() and (lp[3] >= 0).all()
            ll = LocalLevel(rrp, rci, rv, erp, eci, ev, lp, w[l2g].copy(), (n_x, n_y, n_p))
            ll.patches_int, ll.patches_bnd = _split_patches(lp, owned.astype(bool))
            ll.rows_int, ll.rows_bnd = _split_rows(rrp, rci, rv, owned.astype(bool))
            rs.levels[name] = ll
        if p0 is not None:
            rs.n1 = int(p0.ncols)
            prp, pci, pv = _local_csr_cols_global(p0, l2g, owned.astype(bool))
            rs.p_rp, rs.p_ci, rs.p_v = prp, pci, pv
            rs.r_rp, rs.r_ci, rs.r_v = _transpose(nl, rs.n1, prp, pci, pv)
        out.append(rs)
    return out


def _local_csr_cols_global(p, l2g, rows_mask):
    """nl x ncols CSR: the global rows of p at the local dofs where rows_mask,
    other rows empty, columns kept global (the agglomerated coarse space)."""
    nl = len(l2g)
    sel = np.nonzero(rows_mask)[0]
    idx, lens = _rows_of(p.rp, l2g[sel])
    rp = np.zeros(nl + 1, dtype=np.int64)
    cnt = np.zeros(nl, dtype=np.int64)
    cnt[sel] = lens
    np.cumsum(cnt, out=rp[1:])
    return rp.astype(np.int32), np.asarray(p.ci)[idx].astype(np.int32), np.asarray(p.v)[idx].copy()


def _transpose(nrows, ncols, rp, ci, v):
    """transpose (sparse.cpp:93-111): rows of the result list the source rows
    in ascending order."""
    rowid = np.repeat(np.arange(nrows, dtype=np.int64), np.diff(rp).astype(np.int64))
    order = np.argsort(ci, kind="stable")
    trp = np.zeros(ncols + 1, dtype=np.int64)
    np.cumsum(np.bincount(ci, minlength=ncols), out=trp[1:])
    return trp.astype(np.int32), rowid[order].astype(np.int32), np.asarray(v)[order].copy()


def _select_patches(pt, keep):
    """The patches with keep[i], in their order (local patch lists)."""
    pptr, pidx, vptr, vidx, nx = pt
    ids = np.nonzero(keep)[0]
    pl = (pptr[ids + 1] - pptr[ids]).astype(np.int64)
    vl = (vptr[ids + 1] - vptr[ids]).astype(np.int64)
    npp = np.zeros(len(ids) + 1, dtype=np.int32)
    nvp = np.zeros(len(ids) + 1, dtype=np.int32)
    np.cumsum(pl, out=npp[1:])
    np.cumsum(vl, out=nvp[1:])
    return (npp, pidx[_ranges(pptr[ids], pl)].astype(np.int32), nvp,
            vidx[_ranges(vptr[ids], vl)].astype(np.int32), nx[ids].astype(np.int32))


def _split_patches(pt, owned):
    """(interior, boundary): a patch is interior when every dof it touches is
    owned -- it needs no ghost values and contributes to no other rank."""
    pptr, pidx, vptr, vidx, _ = pt
    npatch = len(pptr) - 1
    bad = np.zeros(npatch, dtype=bool)
    pid_v = np.repeat(np.arange(npatch), np.diff(vptr))
    pid_p = np.repeat(np.arange(npatch), np.diff(pptr))
    np.logical_or.at(bad, pid_v, ~owned[vidx])
    np.logical_or.at(bad, pid_p, ~owned[pidx])
    return _select_patches(pt, ~bad), _select_patches(pt, bad)


def _split_rows(rp, ci, v, owned):
    """(interior, boundary) copies of an nl x nl CSR: a row is interior when
    all its columns are owned; each copy keeps the other rows empty."""
    nl = len(rp) - 1
    rowid = np.repeat(np.arange(nl), np.diff(rp))
    bad = np.zeros(nl, dtype=bool)
    np.logical_or.at(bad, rowid, ~owned[ci])
    out = []
    for sel in (~bad, bad):
        keep = sel[rowid]
        nrp = np.zeros(nl + 1, dtype=np.int64)
        np.cumsum(np.bincount(rowid[keep], minlength=nl), out=nrp[1:])
        out.append((nrp.astype(np.int32), ci[keep].copy(), v[keep].copy()))
    return out[0], out[1]
