"""TEST INFRASTRUCTURE ONLY -- the parity checker, never the product path.

ctypes bindings for
  * ``liboracle.so``  -- our plain-C restatement of the reference's solve-phase
    hot path (oracle/oracle.c, each function citing reference file:line), and
  * ``_ref/libstokesamg_ref.so`` -- the UNMODIFIED reference library compiled
    from /root/reference (oracle/Makefile) plus our marshalling shim
    (oracle/ref_shim.cpp).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE_SO = os.path.join(HERE, "liboracle.so")
_REF_SO = os.path.join(HERE, "_ref", "libstokesamg_ref.so")
REF_SRC = "/root/reference/proj/core"

i32p = C.POINTER(C.c_int)
f64p = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_longlong)
vp = C.c_void_p


def build(quiet: bool = True) -> None:
    """Compile the restatement always, and oracle/_ref when the reference
    sources are present (this container; GPU boxes use the prebuilt .so)."""
    targets = ["oracle"]
    if os.path.isdir(REF_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a, t):
    return a.ctypes.data_as(t)


def ip(a):
    return _ptr(a, i32p)


def dp(a):
    return _ptr(a, f64p)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


# --------------------------------------------------------------------------
# CSR container shared by both bindings
# --------------------------------------------------------------------------
@dataclass
class Csr:
    nrows: int
    ncols: int
    rp: np.ndarray
    ci: np.ndarray
    v: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rp[-1])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.v, self.ci, self.rp), shape=(self.nrows, self.ncols))

    @staticmethod
    def from_scipy(m) -> "Csr":
        m = m.tocsr()
        m.sort_indices()
        return Csr(m.shape[0], m.shape[1], m.indptr.astype(np.int32),
                   m.indices.astype(np.int32), m.data.astype(np.float64))


# --------------------------------------------------------------------------
# the restatement (liboracle.so)
# --------------------------------------------------------------------------
class or_csr(C.Structure):
    _fields_ = [("nrows", C.c_int), ("ncols", C.c_int), ("rp", i32p), ("ci", i32p),
                ("v", f64p)]


class or_patches(C.Structure):
    _fields_ = [("npatch", C.c_int), ("pptr", i32p), ("pidx", i32p), ("vptr", i32p),
                ("vidx", i32p), ("nx", i32p)]


class or_vanka(C.Structure):
    _fields_ = [("pat", or_patches), ("n", C.c_int), ("lu_off", i64p), ("aux_off", i64p),
                ("s_off", i64p), ("lu", f64p), ("piv", i32p), ("piv_off", i64p),
                ("uhat", f64p), ("bhat", f64p), ("sinv", f64p), ("weights", f64p),
                ("a_factor_bytes", C.c_int64), ("aux_bytes", C.c_int64),
                ("dense_inverse_bytes", C.c_int64)]


class or_patches3(C.Structure):
    _fields_ = [("npatch", C.c_int), ("pptr", i32p), ("pidx", i32p), ("vptr", i32p),
                ("vidx", i32p), ("cnt", i32p)]


class or_vanka3(C.Structure):
    _fields_ = [("pat", or_patches3), ("n", C.c_int), ("lu_off", i64p), ("piv_off", i64p),
                ("aux_off", i64p), ("s_off", i64p), ("lu", f64p), ("piv", i32p),
                ("uhat", f64p), ("bhat", f64p), ("sinv", f64p), ("weights", f64p)]


class or_fgmres_opts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iters", C.c_int), ("restart", C.c_int),
                ("breakdown", C.c_double)]


class or_report(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int),
                ("final_relative_residual", C.c_double), ("history_len", C.c_int)]


class or_mono(C.Structure):
    _fields_ = [("nlevels", C.c_int), ("k", C.POINTER(or_csr)), ("p", C.POINTER(or_csr)),
                ("nxyz", i32p), ("vanka", C.POINTER(or_vanka)), ("nc", C.c_int),
                ("coarse_lu", f64p), ("coarse_piv", i32p)]


class or_config(C.Structure):
    _fields_ = [("variant", C.c_int), ("eta_u", C.c_double), ("eta_p", C.c_double),
                ("omega0", C.c_double), ("nu1", C.c_int), ("nu2", C.c_int),
                ("gamma", C.c_int), ("restart", C.c_int), ("tol", C.c_double),
                ("max_iters", C.c_int), ("enclosed_flow", C.c_int)]


class or_dc(C.Structure):
    _fields_ = [("k0", or_csr), ("n_x0", C.c_int), ("n_y0", C.c_int), ("n_p0", C.c_int),
                ("stationary_fine", C.c_int), ("fine", or_vanka), ("mono", or_mono),
                ("cfg", or_config)]


_olib = None


def olib():
    global _olib
    if _olib is None:
        L = C.CDLL(_ORACLE_SO)
        L.or_norm2.restype = C.c_double
        L.or_dot.restype = C.c_double
        L.or_norm_inf.restype = C.c_double
        L.or_last_error.restype = C.c_char_p
        _olib = L
    return _olib


def _ocheck(rc):
    if rc != 0:
        raise OracleError(rc, olib().or_last_error().decode())


def _ocsr(m: Csr) -> or_csr:
    return or_csr(m.nrows, m.ncols, ip(m.rp), ip(m.ci), dp(m.v))


class Oracle:
    """Pythonic wrapper of the C restatement; arrays are numpy."""

    @staticmethod
    def spmv(m: Csr, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(m.nrows)
        olib().or_spmv(C.byref(_ocsr(m)), dp(x), dp(y))
        return y

    @staticmethod
    def norm2(v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        return olib().or_norm2(len(v), dp(v))

    @staticmethod
    def dot(a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        return olib().or_dot(len(a), dp(a), dp(b))

    @staticmethod
    def lu_solve_dense(a, b):
        a = np.array(a, dtype=np.float64, order="C")
        n = a.shape[0]
        piv = np.empty(n, dtype=np.int32)
        _ocheck(olib().or_lu_factor(n, dp(a), ip(piv)))
        x = np.array(b, dtype=np.float64)
        olib().or_lu_solve(n, dp(a), ip(piv), dp(x))
        return x

    @staticmethod
    def build_patches(k: Csr, n_x, n_y, n_p, sv_triples=False):
        p = or_patches()
        _ocheck(olib().or_build_patches(C.byref(_ocsr(k)), int(n_x), int(n_y), int(n_p), int(sv_triples),
                                        C.byref(p)))
        out = _patches_to_np(p)
        olib().or_patches_free(C.byref(p))
        return out


def _patches_to_np(p: or_patches):
    n = p.npatch
    pptr = np.ctypeslib.as_array(p.pptr, (n + 1,)).copy()
    vptr = np.ctypeslib.as_array(p.vptr, (n + 1,)).copy()
    return Patches(pptr, np.ctypeslib.as_array(p.pidx, (max(int(pptr[-1]), 1),))[:pptr[-1]].copy(),
                   vptr, np.ctypeslib.as_array(p.vidx, (max(int(vptr[-1]), 1),))[:vptr[-1]].copy(),
                   np.ctypeslib.as_array(p.nx, (max(n, 1),))[:n].copy())


@dataclass
class Patches:
    pptr: np.ndarray
    pidx: np.ndarray
    vptr: np.ndarray
    vidx: np.ndarray
    nx: np.ndarray

    @property
    def npatch(self):
        return len(self.pptr) - 1

    def to_c(self):
        return or_patches(self.npatch, ip(self.pptr), ip(self.pidx), ip(self.vptr),
                          ip(self.vidx), ip(self.nx))


class OracleVanka:
    """factor_patches (vanka.cpp:64-149) held by the restatement."""

    def __init__(self, k: Csr, patches: Patches, n_u: int):
        self._k = k
        self._patches = patches
        self.f = or_vanka()
        _ocheck(olib().or_factor_patches(C.byref(_ocsr(k)), C.byref(patches.to_c()), int(n_u),
                                         C.byref(self.f)))
        self.n = k.nrows

    def __del__(self):
        try:
            olib().or_vanka_free(C.byref(self.f))
        except Exception:
            pass

    def apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        d = np.empty(self.n)
        olib().or_apply_vanka(C.byref(self.f), dp(r), dp(d))
        return d

    def relax(self, x, b, mode, sweeps, omega=1.0):
        x = np.array(x, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        _ocheck(olib().or_vanka_relax(C.byref(_ocsr(self._k)), C.byref(self.f), dp(x), dp(b),
                                      int(mode), int(sweeps), C.c_double(omega)))
        return x

    def factors(self):
        f = self.f
        n = f.pat.npatch
        aux = f.aux_off[n]
        s = f.s_off[n]
        return dict(
            uhat=np.ctypeslib.as_array(f.uhat, (max(aux, 1),))[:aux].copy(),
            bhat=np.ctypeslib.as_array(f.bhat, (max(aux, 1),))[:aux].copy(),
            sinv=np.ctypeslib.as_array(f.sinv, (max(s, 1),))[:s].copy(),
            weights=np.ctypeslib.as_array(f.weights, (self.n,)).copy(),
            a_factor_bytes=f.a_factor_bytes, aux_bytes=f.aux_bytes,
            dense_inverse_bytes=f.dense_inverse_bytes)


class OracleVanka3:
    """The 3-component generalisation of build_patches / factor_patches /
    apply_vanka (vanka.cpp:11-184 with x, y, z blocks) for BASELINE config 5,
    which the reference does not support: parity of the 3D
    kernels is pinned to this restatement and to a dense check of it, not to
    the reference."""

    def __init__(self, k: Csr, n_x, n_y, n_z, n_p):
        self._k = k
        p = or_patches3()
        _ocheck(olib().or_build_patches3(C.byref(_ocsr(k)), int(n_x), int(n_y), int(n_z),
                                         int(n_p), C.byref(p)))
        self.f = or_vanka3()
        rc = olib().or_factor_patches3(C.byref(_ocsr(k)), C.byref(p), C.byref(self.f))
        n = p.npatch
        self.pptr = np.ctypeslib.as_array(p.pptr, (n + 1,)).copy()
        self.vptr = np.ctypeslib.as_array(p.vptr, (n + 1,)).copy()
        self.pidx = np.ctypeslib.as_array(p.pidx, (max(n, 1),))[:n].copy()
        self.vidx = np.ctypeslib.as_array(p.vidx, (max(int(self.vptr[-1]), 1),))[
            :self.vptr[-1]].copy()
        self.cnt = np.ctypeslib.as_array(p.cnt, (max(3 * n, 1),))[:3 * n].reshape(n, 3).copy()
        olib().or_patches3_free(C.byref(p))
        _ocheck(rc)
        self.n = k.nrows

    def __del__(self):
        try:
            olib().or_vanka3_free(C.byref(self.f))
        except Exception:
            pass

    def apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        d = np.empty(self.n)
        olib().or_apply_vanka3(C.byref(self.f), dp(r), dp(d))
        return d


class OracleDC:
    """DCPreconditioner (preconditioner.hpp:77-100) on a given hierarchy."""

    def __init__(self, k0: Csr, nxyz0, levels, cfg: dict, sv=False):
        # levels: list of (K Csr, P Csr or None, (n_x, n_y, n_p))
        self._keep = [k0, levels]
        L = len(levels)
        ks = (or_csr * L)(*[_ocsr(l[0]) for l in levels])
        ps = (or_csr * max(L, 1))(*[_ocsr(l[1]) for l in levels if l[1] is not None])
        nxyz = np.array([v for l in levels for v in l[2]], dtype=np.int32)
        self._keep += [ks, ps, nxyz]
        c = or_config(cfg.get("variant", 0), cfg.get("eta_u", 1.0), cfg.get("eta_p", 1.0),
                      cfg.get("omega0", 1.0), cfg.get("nu1", 1), cfg.get("nu2", 1),
                      cfg.get("gamma", 1), cfg.get("restart", 30), cfg.get("tol", 1e-8),
                      cfg.get("max_iters", 500), int(cfg.get("enclosed_flow", True)))
        self.d = or_dc()
        self.n = k0.nrows
        _ocheck(olib().or_dc_setup(C.byref(self.d), C.byref(_ocsr(k0)), *[int(v) for v in nxyz0], int(sv), L,
                                   ks, ps, ip(nxyz), C.byref(c)))

    def __del__(self):
        try:
            olib().or_dc_free(C.byref(self.d))
        except Exception:
            pass

    def apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.empty(self.n)
        _ocheck(olib().or_dc_apply(C.byref(self.d), dp(r), dp(z)))
        return z

    def vcycle(self, b, nu1=1, nu2=1):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(len(b))
        _ocheck(olib().or_vcycle(C.byref(self.d.mono), dp(b), dp(x), nu1, nu2))
        return x

    def solve(self, rhs, cap=1000):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        x = np.empty(self.n)
        rep = or_report()
        hist = np.zeros(cap)
        _ocheck(olib().or_solve_stokes(C.byref(self.d), dp(rhs), dp(x), C.byref(rep), dp(hist),
                                       cap))
        return x, dict(converged=bool(rep.converged), iterations=rep.iterations,
                       final_relative_residual=rep.final_relative_residual,
                       residual_history=hist[:min(rep.history_len, cap)].copy())


def oracle_fgmres(a: Csr, b, x0, prec, tol=1e-8, max_iters=500, restart=20, breakdown=1e-30,
                  cap=1000):
    """fgmres (krylov.cpp:17-121) restated; prec: None (identity) or OracleVanka."""
    OP = C.CFUNCTYPE(None, vp, f64p, f64p)
    n = a.nrows
    ac = _ocsr(a)

    def aop(ctx, x, y):
        olib().or_spmv(C.byref(ac), x, y)

    if prec is None:
        def pop(ctx, x, y):
            C.memmove(y, x, 8 * n)
    else:
        def pop(ctx, x, y):
            olib().or_apply_vanka(C.byref(prec.f), x, y)
    af, pf = OP(aop), OP(pop)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.array(x0, dtype=np.float64)
    rep = or_report()
    hist = np.zeros(cap)
    opt = or_fgmres_opts(tol, max_iters, restart, breakdown)
    _ocheck(olib().or_fgmres(n, af, None, dp(b), dp(x), pf, None, C.byref(opt), C.byref(rep),
                             dp(hist), cap))
    return x, dict(converged=bool(rep.converged), iterations=rep.iterations,
                   final_relative_residual=rep.final_relative_residual,
                   residual_history=hist[:min(rep.history_len, cap)].copy())


# --------------------------------------------------------------------------
# the reference itself (oracle/_ref/libstokesamg_ref.so)
# --------------------------------------------------------------------------
class RefFgmresOpts(C.Structure):
    _fields_ = or_fgmres_opts._fields_


class RefReport(C.Structure):
    _fields_ = or_report._fields_


class RefConfig(C.Structure):
    _fields_ = [("variant", C.c_int), ("eta_u", C.c_double), ("eta_p", C.c_double),
                ("omega0", C.c_double), ("nu1", C.c_int), ("nu2", C.c_int),
                ("gamma", C.c_int), ("restart", C.c_int), ("tol", C.c_double),
                ("max_iters", C.c_int), ("enclosed_flow", C.c_int), ("coarse_size", C.c_int)]


_rlib = None


def rlib():
    global _rlib
    if _rlib is None:
        L = C.CDLL(_REF_SO)
        for name in ["ref_mat_new", "ref_mat_from_triplets", "ref_case_build",
                     "ref_case_custom_th", "ref_case_k0", "ref_case_k1", "ref_case_sv_matrix",
                     "ref_vanka_build", "ref_build_patches", "ref_vanka_from_lists",
                     "ref_dc_new", "ref_dc_k0", "ref_dc_level_vanka", "ref_transpose"]:
            getattr(L, name).restype = vp
        L.ref_case_build.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_int, C.c_char_p,
                                     C.c_int]
        L.ref_case_custom_th.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int]
        L.ref_mat_new.argtypes = [C.c_int, C.c_int, C.c_longlong, i32p, i32p, f64p]
        L.ref_mat_from_triplets.argtypes = [C.c_int, C.c_int, C.c_longlong, i32p, i32p, f64p]
        for name in ["ref_case_k0", "ref_case_k1", "ref_dc_k0", "ref_transpose"]:
            getattr(L, name).argtypes = [vp]
        L.ref_case_sv_matrix.argtypes = [vp, C.c_int]
        L.ref_vanka_build.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_build_patches.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_vanka_from_lists.argtypes = [vp, C.c_int, i32p, i32p, i32p, i32p, i32p, C.c_int]
        L.ref_dc_new.argtypes = [vp, C.POINTER(RefConfig)]
        L.ref_dc_level_vanka.argtypes = [vp, C.c_int]
        L.ref_dc_level.argtypes = [vp, C.c_int, i32p, C.POINTER(vp), C.POINTER(vp)]
        L.ref_free.argtypes = [vp]
        L.ref_last_error.restype = C.c_char_p
        L.ref_norm_inf.restype = C.c_double
        L.ref_norm_inf.argtypes = [vp]
        for name in ["ref_mat_shape", "ref_mat_copy", "ref_spmv", "ref_case_info",
                     "ref_case_rhs", "ref_vanka_info", "ref_vanka_patches", "ref_vanka_factors",
                     "ref_vanka_lu", "ref_apply_vanka", "ref_vanka_relax", "ref_fgmres",
                     "ref_dc_set_parameters", "ref_dc_nlevels", "ref_dc_apply", "ref_dc_vcycle",
                     "ref_dc_counters", "ref_solve_stokes", "ref_transfer_restrict",
                     "ref_transfer_prolong", "ref_dense_lu_solve"]:
            getattr(L, name).argtypes = None
        _rlib = L
    return _rlib


def _rcheck(rc):
    if rc != 0:
        raise OracleError(rc, rlib().ref_last_error().decode())


def _rnonnull(h):
    if not h:
        raise OracleError(-1, rlib().ref_last_error().decode())
    return h


class RefMat:
    def __init__(self, handle):
        self.h = C.c_void_p(_rnonnull(handle))

    def __del__(self):
        try:
            rlib().ref_free(self.h)
        except Exception:
            pass

    @staticmethod
    def from_csr(m: Csr) -> "RefMat":
        return RefMat(rlib().ref_mat_new(m.nrows, m.ncols, m.nnz, ip(m.rp), ip(m.ci), dp(m.v)))

    @staticmethod
    def from_triplets(nr, nc, rows, cols, vals) -> "RefMat":
        r = np.asarray(rows, dtype=np.int32)
        c = np.asarray(cols, dtype=np.int32)
        v = np.asarray(vals, dtype=np.float64)
        return RefMat(rlib().ref_mat_from_triplets(nr, nc, len(r), ip(r), ip(c), dp(v)))

    def csr(self) -> Csr:
        nr, nc, nnz = C.c_int(), C.c_int(), C.c_longlong()
        rlib().ref_mat_shape(self.h, C.byref(nr), C.byref(nc), C.byref(nnz))
        rp = np.empty(nr.value + 1, dtype=np.int32)
        ci = np.empty(nnz.value, dtype=np.int32)
        v = np.empty(nnz.value)
        rlib().ref_mat_copy(self.h, ip(rp), ip(ci), dp(v))
        return Csr(nr.value, nc.value, rp, ci, v)

    def spmv(self, x):
        m = self.csr_shape()
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(m[0])
        _rcheck(rlib().ref_spmv(self.h, dp(x), dp(y)))
        return y

    def csr_shape(self):
        nr, nc, nnz = C.c_int(), C.c_int(), C.c_longlong()
        rlib().ref_mat_shape(self.h, C.byref(nr), C.byref(nc), C.byref(nnz))
        return nr.value, nc.value, nnz.value

    def norm_inf(self):
        return rlib().ref_norm_inf(self.h)


class RefVanka:
    def __init__(self, handle, k: RefMat | None = None):
        self.h = C.c_void_p(_rnonnull(handle))
        self.k = k
        info = np.zeros(7, dtype=np.int64)
        rlib().ref_vanka_info(self.h, info.ctypes.data_as(i64p))
        (self.npatch, self.tot_p, self.tot_v, self.a_factor_bytes, self.aux_bytes,
         self.dense_inverse_bytes, self.n) = [int(v) for v in info]

    def __del__(self):
        try:
            rlib().ref_free(self.h)
        except Exception:
            pass

    @staticmethod
    def build(k: RefMat, n_x, n_y, n_p, sv_triples=False) -> "RefVanka":
        return RefVanka(rlib().ref_vanka_build(k.h, n_x, n_y, n_p, int(sv_triples)), k)

    @staticmethod
    def from_patches(k: RefMat, patches: Patches, n_u) -> "RefVanka":
        return RefVanka(rlib().ref_vanka_from_lists(
            k.h, patches.npatch, ip(patches.pptr), ip(patches.pidx), ip(patches.vptr),
            ip(patches.vidx), ip(patches.nx), n_u), k)

    def patches(self) -> Patches:
        pptr = np.empty(self.npatch + 1, dtype=np.int32)
        vptr = np.empty(self.npatch + 1, dtype=np.int32)
        pidx = np.empty(max(self.tot_p, 1), dtype=np.int32)
        vidx = np.empty(max(self.tot_v, 1), dtype=np.int32)
        nx = np.empty(max(self.npatch, 1), dtype=np.int32)
        rlib().ref_vanka_patches(self.h, ip(pptr), ip(pidx), ip(vptr), ip(vidx), ip(nx))
        return Patches(pptr, pidx[:self.tot_p], vptr, vidx[:self.tot_v], nx[:self.npatch])

    def factors(self):
        p = self.patches()
        nv = np.diff(p.vptr).astype(np.int64)
        npp = np.diff(p.pptr).astype(np.int64)
        aux = int((nv * npp).sum())
        s = int((npp * npp).sum())
        u = np.empty(max(aux, 1))
        b = np.empty(max(aux, 1))
        si = np.empty(max(s, 1))
        w = np.empty(self.n)
        rlib().ref_vanka_factors(self.h, dp(u), dp(b), dp(si), dp(w))
        return dict(uhat=u[:aux], bhat=b[:aux], sinv=si[:s], weights=w,
                    a_factor_bytes=self.a_factor_bytes, aux_bytes=self.aux_bytes,
                    dense_inverse_bytes=self.dense_inverse_bytes)

    def apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        d = np.empty(self.n)
        _rcheck(rlib().ref_apply_vanka(self.h, dp(r), dp(d)))
        return d

    def relax(self, x, b, mode, sweeps, omega=1.0):
        x = np.array(x, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        _rcheck(rlib().ref_vanka_relax(self.k.h, self.h, dp(x), dp(b), C.c_int(mode),
                                       C.c_int(sweeps), C.c_double(omega)))
        return x


def ref_build_patches(k: RefMat, n_x, n_y, n_p, sv_triples=False) -> Patches:
    h = RefVanka(rlib().ref_build_patches(k.h, n_x, n_y, n_p, int(sv_triples)))
    return h.patches()


def ref_fgmres(a: RefMat, b, x0, prec_kind=0, prec=None, tol=1e-8, max_iters=500, restart=20,
               breakdown=1e-30, cap=1000):
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.array(x0, dtype=np.float64)
    rep = RefReport()
    hist = np.zeros(cap)
    opt = RefFgmresOpts(tol, max_iters, restart, breakdown)
    _rcheck(rlib().ref_fgmres(a.h, dp(b), dp(x), C.c_int(prec_kind),
                              prec.h if prec is not None else None, C.byref(opt), C.byref(rep),
                              dp(hist), C.c_int(cap)))
    return x, dict(converged=bool(rep.converged), iterations=rep.iterations,
                   final_relative_residual=rep.final_relative_residual,
                   residual_history=hist[:min(rep.history_len, cap)].copy())


class RefCase:
    """build_case (experiments.cpp:215-235) through the reference."""

    def __init__(self, handle):
        self.h = C.c_void_p(_rnonnull(handle))
        info = np.zeros(8, dtype=np.int32)
        rlib().ref_case_info(self.h, ip(info))
        (self.n_x0, self.n_y0, self.n_p0, self.n_x1, self.n_y1, self.n_p1, enc, sv) = [
            int(v) for v in info]
        self.enclosed = bool(enc)
        self.sv = bool(sv)
        self.n0 = self.n_x0 + self.n_y0 + self.n_p0

    def __del__(self):
        try:
            rlib().ref_free(self.h)
        except Exception:
            pass

    @staticmethod
    def build(problem="cavity", sv=False, mesh_kind="structured", n=8, mesh_path=None,
              refinement=0) -> "RefCase":
        return RefCase(rlib().ref_case_build(problem.encode(), int(sv), mesh_kind.encode(), n,
                                             mesh_path.encode() if mesh_path else None,
                                             refinement))

    @staticmethod
    def custom_th(n, tagger=0, jitter=0.0, force=0) -> "RefCase":
        return RefCase(rlib().ref_case_custom_th(n, tagger, jitter, force))

    @staticmethod
    def mesh_forced(path, k1, k2) -> "RefCase":
        """BASELINE config 4 on a mesh JSON (zero velocity, f = (sin k1 x, cos k2 y))."""
        L = rlib()
        L.ref_case_mesh_forced.restype = vp
        L.ref_case_mesh_forced.argtypes = [C.c_char_p, C.c_double, C.c_double]
        return RefCase(L.ref_case_mesh_forced(path.encode(), k1, k2))

    def rhs(self):
        r = np.empty(self.n0)
        rlib().ref_case_rhs(self.h, dp(r))
        return r

    def k0(self) -> RefMat:
        return RefMat(rlib().ref_case_k0(self.h))

    def k1(self) -> RefMat:
        return RefMat(rlib().ref_case_k1(self.h))


class RefDC:
    """DCPreconditioner (preconditioner.hpp:77-100) and solve_stokes through the
    reference."""

    def __init__(self, case: RefCase, cfg: dict):
        c = RefConfig(cfg.get("variant", 0), cfg.get("eta_u", 1.0), cfg.get("eta_p", 1.0),
                      cfg.get("omega0", 1.0), cfg.get("nu1", 1), cfg.get("nu2", 1),
                      cfg.get("gamma", 1), cfg.get("restart", 30), cfg.get("tol", 1e-8),
                      cfg.get("max_iters", 500), int(cfg.get("enclosed_flow", case.enclosed)),
                      cfg.get("coarse_size", 0))
        self.h = C.c_void_p(_rnonnull(rlib().ref_dc_new(case.h, C.byref(c))))
        self.n = case.n0
        self.nxyz0 = (case.n_x0, case.n_y0, case.n_p0)
        self.cfg = cfg

    def __del__(self):
        try:
            rlib().ref_free(self.h)
        except Exception:
            pass

    def set_parameters(self, eta_u, eta_p, omega0):
        _rcheck(rlib().ref_dc_set_parameters(self.h, C.c_double(eta_u), C.c_double(eta_p),
                                             C.c_double(omega0)))

    def k0(self) -> RefMat:
        return RefMat(rlib().ref_dc_k0(self.h))

    def nlevels(self) -> int:
        return rlib().ref_dc_nlevels(self.h)

    def level(self, l):
        out = np.zeros(4, dtype=np.int32)
        k = C.c_void_p()
        p = C.c_void_p()
        rlib().ref_dc_level(self.h, l, ip(out), C.byref(k), C.byref(p))
        return (RefMat(k.value), RefMat(p.value) if out[3] else None,
                (int(out[0]), int(out[1]), int(out[2])))

    def levels_csr(self):
        out = []
        for l in range(self.nlevels()):
            k, p, nxyz = self.level(l)
            out.append((k.csr(), p.csr() if p is not None else None, nxyz))
        return out

    def level_vanka(self, l) -> RefVanka:
        return RefVanka(rlib().ref_dc_level_vanka(self.h, l))

    def apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.empty(self.n)
        _rcheck(rlib().ref_dc_apply(self.h, dp(r), dp(z)))
        return z

    def vcycle(self, b, nu1=1, nu2=1):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(len(b))
        _rcheck(rlib().ref_dc_vcycle(self.h, dp(b), dp(x), C.c_int(nu1), C.c_int(nu2)))
        return x

    def counters(self):
        out = np.zeros(2, dtype=np.int64)
        rlib().ref_dc_counters(self.h, out.ctypes.data_as(i64p))
        return int(out[0]), int(out[1])

    def solve(self, rhs, cap=1000):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        x = np.empty(self.n)
        rep = RefReport()
        hist = np.zeros(cap)
        _rcheck(rlib().ref_solve_stokes(self.h, dp(rhs), dp(x), C.byref(rep), dp(hist),
                                        C.c_int(cap)))
        return x, dict(converged=bool(rep.converged), iterations=rep.iterations,
                       final_relative_residual=rep.final_relative_residual,
                       residual_history=hist[:min(rep.history_len, cap)].copy())


class RefPrec:
    """Any preconditioner variant (preconditioner.hpp:14: DC-all/LO/HO,
    HO-AMG, Uzawa) built by the reference from a case, and solve_stokes with
    it (experiments.cpp:124-140, :268-275)."""

    def __init__(self, case: RefCase, cfg: dict):
        c = RefConfig(cfg.get("variant", 0), cfg.get("eta_u", 1.0), cfg.get("eta_p", 1.0),
                      cfg.get("omega0", 1.0), cfg.get("nu1", 1), cfg.get("nu2", 1),
                      cfg.get("gamma", 1), cfg.get("restart", 30), cfg.get("tol", 1e-8),
                      cfg.get("max_iters", 500), int(cfg.get("enclosed_flow", case.enclosed)),
                      cfg.get("coarse_size", 0))
        L = rlib()
        L.ref_prec_new.restype = vp
        L.ref_prec_new.argtypes = [vp, C.POINTER(RefConfig)]
        self.h = C.c_void_p(_rnonnull(L.ref_prec_new(case.h, C.byref(c))))
        self.n = case.n0

    def __del__(self):
        try:
            rlib().ref_free(self.h)
        except Exception:
            pass

    def apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.empty(self.n)
        _rcheck(rlib().ref_prec_apply(self.h, dp(r), dp(z)))
        return z

    def solve(self, rhs, cap=1000):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        x = np.empty(self.n)
        rep = RefReport()
        hist = np.zeros(cap)
        _rcheck(rlib().ref_prec_solve(self.h, dp(rhs), dp(x), C.byref(rep), dp(hist),
                                      C.c_int(cap)))
        return x, dict(converged=bool(rep.converged), iterations=rep.iterations,
                       final_relative_residual=rep.final_relative_residual,
                       residual_history=hist[:min(rep.history_len, cap)].copy())


def ref_sort_permutation(keys) -> np.ndarray:
    """std::sort's permutation under from_triplets' comparator (sparse.cpp:44-46)
    on the reference's own Triplet, keys = row << 32 | col."""
    L = rlib()
    L.ref_sort_permutation.argtypes = [C.c_longlong, vp, vp]
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    p = np.empty(len(k), dtype=np.int32)
    _rcheck(L.ref_sort_permutation(len(k), k.ctypes.data, p.ctypes.data))
    return p


def ref_antiqsort_keys(n: int) -> np.ndarray:
    """McIlroy's quicksort adversary run against std::sort: keys that push
    introsort to its heap-sort fallback."""
    L = rlib()
    L.ref_antiqsort_keys.argtypes = [C.c_int, vp]
    k = np.empty(n, dtype=np.uint64)
    _rcheck(L.ref_antiqsort_keys(n, k.ctypes.data))
    return k


def splitmix64_uniform(n: int, seed: int = 0x5EED) -> np.ndarray:
    """x_i in U[-1,1) from splitmix64(seed ^ i); identical on
    host and device."""
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) ^ np.arange(n, dtype=np.uint64)) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return ((z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) * 2.0 - 1.0
