"""Reference-built inputs of the GPU path (the host application side).

The reference keeps mesh generation, FEM assembly and the SA hierarchy setup in
its own host C++ (north_star; the setup is discrete and
rounding-sensitive). ``libsag_stokesamg.so`` links the reference library
(compiled from its sources by hostapp/Makefile) and exposes
build_case + assemble_saddle_matrix + build_monolithic_hierarchy as ``sagh_*``
entry points; this module turns their output into device matrices for the
Python mirror of the solver API.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import DCPreconditioner, SolverConfig, SparseMatrix, Context, HERE

_HLIB = os.path.join(HERE, "libsag_stokesamg.so")
_h = None


def hlib():
    global _h
    if _h is None:
        if not os.path.exists(_HLIB):
            raise RuntimeError(f"{_HLIB} missing: run __graft_entry__.build()")
        L = C.CDLL(_HLIB)
        L.sagh_case_build.restype = C.c_void_p
        L.sagh_case_build.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_int, C.c_char_p,
                                      C.c_int, C.c_double, C.c_double]
        L.sagh_case_free.argtypes = [C.c_void_p]
        L.sagh_last_error.restype = C.c_char_p
        L.sagh_case_info.argtypes = [C.c_void_p, C.c_void_p]
        L.sagh_case_level.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.sagh_case_matrix_shape.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                             C.c_void_p]
        L.sagh_case_matrix_copy.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                            C.c_void_p]
        L.sagh_case_rhs.argtypes = [C.c_void_p, C.c_void_p]
        L.sagh_case_build_extra.argtypes = [C.c_void_p, C.c_int]
        L.sagh_case_info_extra.argtypes = [C.c_void_p, C.c_void_p]
        L.sagh_case_ho_level.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.sagh_case_sv_areas.argtypes = [C.c_void_p, C.c_void_p]
        L.sagh_case_solve_variant.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                              C.c_double, C.c_int, C.c_double, C.c_double,
                                              C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
        L.sagh_case_hierarchy_gpu.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.sagh_case_scalar_hierarchy_gpu.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.sagh_case_assembly_gpu.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        L.sagh_case_solve_dist.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                           C.c_void_p]
        L.sagh_case_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                      C.c_double, C.c_double, C.c_double, C.c_void_p, C.c_void_p,
                                      C.c_void_p]
        _h = L
    return _h


@dataclass
class Csr:
    nrows: int
    ncols: int
    rp: np.ndarray
    ci: np.ndarray
    v: np.ndarray

    @property
    def nnz(self):
        return int(self.rp[-1])


class HostCase:
    """build_case (experiments.cpp:215-235) + K0 + low-order hierarchy."""

    def __init__(self, problem="cavity", sv=False, mesh_kind="structured", n=64, mesh_path=None,
                 coarse_size=0, k1=0.0, k2=0.0):
        h = hlib().sagh_case_build(problem.encode(), int(sv), mesh_kind.encode(), int(n),
                                   mesh_path.encode() if mesh_path else None, int(coarse_size),
                                   float(k1), float(k2))
        if not h:
            raise RuntimeError("sagh_case_build: " + hlib().sagh_last_error().decode())
        self.h = C.c_void_p(h)
        info = np.zeros(7, dtype=np.int64)
        hlib().sagh_case_info(self.h, info.ctypes.data)
        (self.n_x0, self.n_y0, self.n_p0, self.nlevels, enc, sv_, self.n_scalar) = (
            int(v) for v in info)
        self.enclosed, self.sv = bool(enc), bool(sv_)
        self.n0 = self.n_x0 + self.n_y0 + self.n_p0
        self.nxyz0 = (self.n_x0, self.n_y0, self.n_p0)

    def __del__(self):
        try:
            hlib().sagh_case_free(self.h)
        except Exception:
            pass

    def matrix(self, which: int) -> Csr:
        nr, nc, nnz = C.c_int(), C.c_int(), C.c_longlong()
        rc = hlib().sagh_case_matrix_shape(self.h, which, C.byref(nr), C.byref(nc), C.byref(nnz))
        if rc:
            raise RuntimeError(hlib().sagh_last_error().decode())
        rp = np.empty(nr.value + 1, dtype=np.int32)
        ci = np.empty(nnz.value, dtype=np.int32)
        v = np.empty(nnz.value)
        hlib().sagh_case_matrix_copy(self.h, which, rp.ctypes.data, ci.ctypes.data, v.ctypes.data)
        return Csr(nr.value, nc.value, rp, ci, v)

    def k0(self) -> Csr:
        return self.matrix(0)

    def level(self, l):
        nxyz = np.zeros(3, dtype=np.int32)
        hlib().sagh_case_level(self.h, l, nxyz.ctypes.data)
        k = self.matrix(1 + 2 * l)
        p = self.matrix(2 + 2 * l) if l + 1 < self.nlevels else None
        return k, p, tuple(int(v) for v in nxyz)

    def levels(self):
        return [self.level(l) for l in range(self.nlevels)]

    def hierarchy_gpu(self, device=0):
        """The low-order hierarchy built again by the reference and by
        gpu::build_monolithic_hierarchy (SA setup products on the device),
        compared bitwise (sagh_case_hierarchy_gpu)."""
        out = np.zeros(8)
        if hlib().sagh_case_hierarchy_gpu(self.h, int(device), out.ctypes.data):
            raise RuntimeError(hlib().sagh_last_error().decode())
        return dict(reference_s=float(out[0]), device_assisted_s=float(out[1]),
                    host_part_s=float(out[2]), device_part_s=float(out[3]),
                    bitwise_equal=bool(out[4]), levels=int(out[5]),
                    soc_device=int(out[6]), soc_host=int(out[7]))

    def scalar_hierarchies_gpu(self, device=0):
        """build_scalar_hierarchy by the reference and on the device for A_x and
        the pressure auxiliary operator, compared bitwise."""
        out = np.zeros(4)
        if hlib().sagh_case_scalar_hierarchy_gpu(self.h, int(device), out.ctypes.data):
            raise RuntimeError(hlib().sagh_last_error().decode())
        return dict(bitwise_equal=bool(out[0]), operators=int(out[1]), levels=int(out[2]),
                    soc_device=int(out[3]))

    def assembly_gpu(self, device=0, time_reference=False):
        """The case's systems assembled again on the device (gpu::assemble_*:
        element loops, from_triplets and Dirichlet elimination in libsag) and
        compared with the reference's bitwise: diff bits per system (0 =
        identical; 1 A, 2 B, 4 Ap, 8 Mp, 16 rhs, 32 sizes, 64 coords, 128 bc,
        256 SV extras), K0 equality and timings."""
        out = np.zeros(8)
        if hlib().sagh_case_assembly_gpu(self.h, int(device), int(time_reference),
                                         out.ctypes.data):
            raise RuntimeError(hlib().sagh_last_error().decode())
        return dict(sys0_diff=int(out[0]), sys1_diff=int(out[1]), k0_equal=bool(out[2]),
                    device_s=float(out[3]), reference_s=float(out[4]) if out[4] >= 0 else None,
                    sys0_s=float(out[5]), sys1_s=float(out[6]), k0_s=float(out[7]))

    def solve_dist_dropin(self, device=0):
        """gpu::DistDCPreconditioner (the C++ multi-GPU drop-in) at one rank."""
        x = np.empty(self.n0)
        rep = np.zeros(2, dtype=np.int32)
        res = C.c_double()
        if hlib().sagh_case_solve_dist(self.h, device, x.ctypes.data, rep.ctypes.data,
                                       C.byref(res)):
            raise RuntimeError(hlib().sagh_last_error().decode())
        return x, dict(converged=bool(rep[0]), iterations=int(rep[1]),
                       final_relative_residual=res.value)

    def rhs(self):
        r = np.empty(self.n0)
        hlib().sagh_case_rhs(self.h, r.ctypes.data)
        return r

    def device(self, cfg: SolverConfig, ctx: Context = None, keep_host=False):
        """(K0, DCPreconditioner, host levels) uploaded through the C-ABI."""
        k0 = self.k0()
        K0 = SparseMatrix.from_csr(k0, ctx)
        lv = []
        host = []
        for k, p, nxyz in self.levels():
            lv.append((SparseMatrix.from_csr(k, ctx),
                       SparseMatrix.from_csr(p, ctx) if p is not None else None, nxyz))
            if keep_host:
                host.append((k, p, nxyz))
        dc = DCPreconditioner(K0, self.nxyz0, lv, cfg, sv=self.sv)
        if self.sv:
            pd = SparseMatrix.from_csr(self.matrix(1000), ctx)
            mm = SparseMatrix.from_csr(self.matrix(1001), ctx)
            A = [SparseMatrix.from_csr(self.matrix(1002 + 2 * s), ctx)
                 for s in range(self.n_scalar)]
            P = [SparseMatrix.from_csr(self.matrix(1003 + 2 * s), ctx)
                 for s in range(self.n_scalar - 1)]
            dc.set_sv_transfer(pd, mm, A, P)
        return K0, dc, (k0, host)

    def _extra(self, what):
        if hlib().sagh_case_build_extra(self.h, what):
            raise RuntimeError(hlib().sagh_last_error().decode())
        info = np.zeros(5, dtype=np.int64)
        hlib().sagh_case_info_extra(self.h, info.ctypes.data)
        return [int(v) for v in info]

    def hoamg_device(self, cfg: SolverConfig, ctx: Context = None):
        """(K0, HoAmgPreconditioner) from the reference's HO hierarchy
        (build_monolithic_hierarchy on sys0)."""
        from . import HoAmgPreconditioner
        nl = self._extra(1)[0]
        lv = []
        for l in range(nl):
            nxyz = np.zeros(3, dtype=np.int32)
            hlib().sagh_case_ho_level(self.h, l, nxyz.ctypes.data)
            k = SparseMatrix.from_csr(self.matrix(2000 + 2 * l), ctx)
            p = SparseMatrix.from_csr(self.matrix(2001 + 2 * l), ctx) if l + 1 < nl else None
            lv.append((k, p, tuple(int(v) for v in nxyz)))
        return lv[0][0], HoAmgPreconditioner(lv[0][0], lv, cfg, sv=self.sv)

    def uzawa_device(self, cfg: SolverConfig, ctx: Context = None):
        """(K0, UzawaPreconditioner) from the reference's scalar hierarchies."""
        from . import UzawaPreconditioner
        _, nx_l, ny_l, mp_l, n_el = self._extra(2)

        def sh(base, nl):
            a = [SparseMatrix.from_csr(self.matrix(base + 2 * s), ctx) for s in range(nl)]
            p = [SparseMatrix.from_csr(self.matrix(base + 2 * s + 1), ctx) for s in range(nl - 1)]
            return a, p
        B = SparseMatrix.from_csr(self.matrix(3000), ctx)
        areas = None
        if self.sv:
            areas = np.empty(n_el)
            hlib().sagh_case_sv_areas(self.h, areas.ctypes.data)
        u = UzawaPreconditioner(B, self.n_x0, self.n_y0, self.n_p0, sh(3100, nx_l),
                                sh(3200, ny_l), sh(3300, mp_l) if not self.sv else None,
                                sv_element_areas=areas, cfg=cfg)
        return SparseMatrix.from_csr(self.k0(), ctx), u

    def solve_dropin(self, device=0, nu=1, restart=30, tol=1e-8, max_iters=500, eta_u=1.0,
                     eta_p=1.0, omega0=1.0, variant=0):
        """The C++ drop-in (gpu::DCPreconditioner / HoAmgPreconditioner /
        UzawaPreconditioner + gpu::solve_stokes) end to end."""
        x = np.empty(self.n0)
        rep = np.zeros(2, dtype=np.int32)
        res = C.c_double()
        rc = hlib().sagh_case_solve_variant(self.h, device, variant, nu, restart, tol, max_iters,
                                            eta_u, eta_p, omega0, x.ctypes.data, rep.ctypes.data,
                                            C.byref(res))
        if rc:
            raise RuntimeError(hlib().sagh_last_error().decode())
        return x, dict(converged=bool(rep[0]), iterations=int(rep[1]),
                       final_relative_residual=res.value)
