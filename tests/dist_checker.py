"""Checker backend for paper_2306_06795_b200.dsolve in the CPU tests: the
rank-local kernels are the C restatement (oracle/, test infrastructure) on
torch CPU tensors, so the distributed solve's host logic -- partition, halo
plans, masked reductions, all-reduces, the agglomerated coarse levels, the
FGMRES control -- runs over gloo with world size 1 and 2 here. On B200 the same
DistSolver drives libsag (dsolve.LibsagBackend)."""
import ctypes as C

import numpy as np
import torch

import oracle as O


class _Mat:
    def __init__(self, nrows, ncols, rp, ci, v):
        self.csr = O.Csr(int(nrows), int(ncols), np.ascontiguousarray(rp, dtype=np.int32),
                         np.ascontiguousarray(ci, dtype=np.int32),
                         np.ascontiguousarray(v, dtype=np.float64))
        self.nrows, self.ncols = int(nrows), int(ncols)


class _Coarse:
    """MonolithicSolver::vcycle (preconditioner.cpp:57-88) of the restatement on
    `levels`, with the enclosed-flow pin 1e-12 * norm0 (preconditioner.cpp:49-53)."""

    def __init__(self, levels, cfg, norm0):
        L = len(levels)
        self.keep = [O.Csr(k.nrows, k.ncols, np.asarray(k.rp, np.int32),
                           np.asarray(k.ci, np.int32), np.asarray(k.v, np.float64))
                     for k, _, _ in levels]
        self.pkeep = [O.Csr(p.nrows, p.ncols, np.asarray(p.rp, np.int32),
                            np.asarray(p.ci, np.int32), np.asarray(p.v, np.float64))
                      for _, p, _ in levels if p is not None]
        ks = (O.or_csr * L)(*[O._ocsr(k) for k in self.keep])
        ps = (O.or_csr * max(L, 1))(*[O._ocsr(p) for p in self.pkeep])
        nxyz = np.array([v for l in levels for v in l[2]], dtype=np.int32)
        self._arr = (ks, ps, nxyz)
        self.m = O.or_mono()
        O._ocheck(O.olib().or_mono_setup(C.byref(self.m), L, ks, ps, O.ip(nxyz), 0))
        self.nu1, self.nu2 = cfg.nu1, cfg.nu2
        if cfg.enclosed_flow:
            bot = self.keep[-1]
            nc = bot.nrows
            d = bot.to_scipy().toarray()
            row = int(nxyz[-3] + nxyz[-2])
            d[row, row] += 1e-12 * norm0
            d = np.ascontiguousarray(d)
            piv = np.empty(nc, dtype=np.int32)
            O._ocheck(O.olib().or_lu_factor(nc, O.dp(d), O.ip(piv)))
            C.memmove(self.m.coarse_lu, d.ctypes.data, 8 * nc * nc)
            C.memmove(self.m.coarse_piv, piv.ctypes.data, 4 * nc)

    def apply(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(len(b))
        O._ocheck(O.olib().or_vcycle(C.byref(self.m), O.dp(b), O.dp(x), self.nu1, self.nu2))
        return x


class CheckerBackend:
    """Same interface as dsolve.LibsagBackend; vectors are CPU tensors."""

    torch = torch

    def vec(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def ivec(self, a):
        return torch.as_tensor(np.asarray(a, dtype=np.int64))

    def u8(self, a):
        return torch.as_tensor(np.asarray(a, dtype=np.uint8))

    def from_host(self, a):
        return torch.as_tensor(np.array(a, dtype=np.float64))

    def to_host(self, t):
        return t.numpy().copy()

    def matrix(self, nrows, ncols, rp, ci, v):
        return _Mat(nrows, ncols, rp, ci, v)

    def vanka(self, nl, ext, patches, n_u, weights):
        k = O.Csr(nl, nl, *[np.ascontiguousarray(a) for a in ext])
        pt = O.Patches(*[np.ascontiguousarray(a, dtype=np.int32) for a in patches])
        f = O.OracleVanka(k, pt, n_u)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        C.memmove(f.f.weights, w.ctypes.data, 8 * nl)
        return f

    def coarse(self, levels, cfg, norm0):
        return _Coarse(levels, cfg, norm0)

    def norm_inf(self, m):
        return O.olib().or_norm_inf(C.byref(O._ocsr(m.csr)))

    def spmv(self, m, x, y, epi="store", aux=None):
        s = O.Oracle.spmv(m.csr, x.numpy())
        if epi == "store":
            y.copy_(torch.from_numpy(s))
        elif epi == "resid":
            y.copy_(aux - torch.from_numpy(s))
        else:
            y.add_(torch.from_numpy(s))

    def vanka_apply(self, f, r, delta):
        delta.copy_(torch.from_numpy(f.apply(r.numpy())))

    def vanka_add(self, f, r, x):
        x.copy_(x + 1.0 * torch.from_numpy(f.apply(r.numpy())))

    def coarse_apply(self, h, b, x):
        x.copy_(torch.from_numpy(h.apply(b.numpy())))

    def dot(self, a, b, mask, out):
        m = mask.numpy().astype(bool)
        out[0] = float(np.dot(a.numpy()[m], b.numpy()[m]))

    def axpy_s(self, s, sign, x, y):
        h = float(s[0])
        y.copy_(y - h * x if sign < 0 else y + h * x)

    def div_s(self, x, s, take_sqrt, y):
        d = float(s[0])
        d = np.sqrt(d) if take_sqrt else d
        y.copy_(x / d if d != 0.0 else torch.zeros_like(x))

    def fgmres1_coef(self, ssq_r, h00, ssq_w, y0):
        beta, h, h10 = np.sqrt(float(ssq_r[0])), float(h00[0]), np.sqrt(float(ssq_w[0]))
        if beta == 0.0:
            y0[0] = 0.0
            return
        denom = float(np.hypot(h, h10))
        cs, sn = (h / denom, h10 / denom) if denom > 0.0 else (1.0, 0.0)
        y0[0] = cs * beta / (cs * h + sn * h10)

    def sub_mean(self, x, s, count, y):
        y.copy_(x - float(s[0]) / count)

    def axpby(self, a, x, b, y):
        if a == 0.0 and b == 0.0:
            y.zero_()
        elif b == 0.0:
            y.copy_(a * x)
        elif b == 1.0:
            y.copy_(y + a * x)
        else:
            y.copy_(a * x + b * y)

    def gather(self, idx, src, dst):
        dst.copy_(src[idx])

    def scatter(self, idx, src, dst, add):
        if add:
            dst[idx] += src
        else:
            dst[idx] = src
