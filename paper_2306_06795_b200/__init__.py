"""B200-native solve phase of the monolithic SA-AMG / additive-Vanka Stokes
solver (arXiv 2306.06795; reference implementation ``stokesamg``).

Python mirror of the reference's C++ solver API for the hot path, on top of
the C-ABI in ``include/sag.h`` (``libsag.so``, hand-written sm_100a kernels).
Names, argument meaning and error classes follow the reference:

===============================  ==============================================
reference (proj/core)            here
===============================  ==============================================
SparseMatrix (sparse.hpp:11-28)  :class:`SparseMatrix` (device CSR)
spmv (sparse.hpp:42)             :func:`spmv`
norm2 / dot (sparse.hpp:64-65)   :func:`norm2`, :func:`dot`
build_patches (vanka.hpp:20-21)  :func:`build_patches`
factor_patches (vanka.hpp:42)    :func:`factor_patches`
apply_vanka (vanka.hpp:47)       :func:`apply_vanka`
vanka_relax (vanka.hpp:53-55)    :func:`vanka_relax`
fgmres (krylov.hpp:33-35)        :func:`fgmres`
SolverConfig (precond.hpp:19)    :class:`SolverConfig`
DCPreconditioner (:77-100)       :class:`DCPreconditioner`
solve_stokes (:147-148)          :func:`solve_stokes`
errors.hpp:8-58                  :class:`Error` and subclasses
===============================  ==============================================

There is no CPU fallback: importing works anywhere, but every operation needs
``libsag.so`` and an sm_100 GPU and raises otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsag.so")

__all__ = [
    "spgemm", "transpose", "galerkin_triple", "smooth_prolongator", "evolution_soc",
    "saddle_matrix",
    "Error", "DimensionMismatch", "SingularMatrix", "SingularPatch", "ConfigError",
    "SolverStagnation", "ZeroDiagonal", "UnsupportedDiscretization", "CudaError", "Context", "SparseMatrix", "Patches",
    "VankaFactorization", "spmv", "norm2", "dot", "build_patches", "factor_patches",
    "apply_vanka", "vanka_spmv_step", "vanka_relax", "RelaxMode", "FgmresOptions", "KrylovReport", "fgmres",
    "SolverConfig", "Variant", "DCPreconditioner", "HoAmgPreconditioner", "UzawaPreconditioner",
    "solve_stokes", "default_context", "lib",
]


# ----------------------------------------------------------------- errors --
class Error(RuntimeError):
    """stokesamg::Error (errors.hpp:8-10)."""


class DimensionMismatch(Error):
    pass


class SingularMatrix(Error):
    pass


class SingularPatch(Error):
    pass


class ConfigError(Error):
    pass


class ZeroDiagonal(Error):
    pass


class UnsupportedDiscretization(Error):
    pass


class SolverStagnation(Error):
    pass


class CudaError(Error):
    """Device/driver failure (no reference analogue)."""


_ERRORS = {1: Error, 2: DimensionMismatch, 3: SingularMatrix, 4: SingularPatch,
           5: ConfigError, 6: SolverStagnation, 7: ZeroDiagonal,
           8: UnsupportedDiscretization, 100: CudaError, 101: Error}

i32p = C.POINTER(C.c_int)
f64p = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_longlong)
vp = C.c_void_p


class sag_fgmres_options(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iters", C.c_int), ("restart", C.c_int),
                ("breakdown", C.c_double)]


class sag_krylov_report(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int),
                ("final_relative_residual", C.c_double), ("history_len", C.c_int)]


class sag_solver_config(C.Structure):
    _fields_ = [("variant", C.c_int), ("eta_u", C.c_double), ("eta_p", C.c_double),
                ("omega0", C.c_double), ("nu1", C.c_int), ("nu2", C.c_int), ("gamma", C.c_int),
                ("restart", C.c_int), ("tol", C.c_double), ("max_iters", C.c_int),
                ("enclosed_flow", C.c_int), ("allow_sv_hoamg", C.c_int)]


class sag_scalar_hierarchy(C.Structure):
    _fields_ = [("nlevels", C.c_int), ("a", C.POINTER(vp)), ("p", C.POINTER(vp))]


class sag_level_desc(C.Structure):
    _fields_ = [("k", vp), ("p", vp), ("n_x", C.c_int), ("n_y", C.c_int), ("n_p", C.c_int)]


class sag_mesh2d(C.Structure):
    _fields_ = [("num_vertices", C.c_int), ("num_triangles", C.c_int), ("num_edges", C.c_int),
                ("vertices", vp), ("triangles", vp), ("tri_edges", vp)]


class sag_csr(C.Structure):
    _fields_ = [("nrows", C.c_int), ("ncols", C.c_int), ("row_offsets", vp),
                ("col_indices", vp), ("values", vp)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, vp, vp, C.c_longlong)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, vp, C.c_int, vp, vp, vp, C.c_int, vp, vp, vp)


class sag_comm_ops(C.Structure):
    _fields_ = [("user", vp), ("allreduce_sum", ALLREDUCE_FN), ("exchange", EXCHANGE_FN)]


#: every entry point declared in include/sag.h, with its ctypes signature
SIGNATURES = {
    "sag_last_error": (C.c_char_p, []),
    "sag_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "sag_create_on_stream": (C.c_int, [C.c_int, vp, C.POINTER(vp)]),
    "sag_destroy": (C.c_int, [vp]),
    "sag_synchronize": (C.c_int, [vp]),
    "sag_alloc": (C.c_int, [vp, C.c_size_t, C.POINTER(vp)]),
    "sag_free": (C.c_int, [vp, vp]),
    "sag_memcpy": (C.c_int, [vp, vp, vp, C.c_size_t]),
    "sag_launch_count": (C.c_int, [vp, i64p]),
    "sag_stream": (C.c_int, [vp, C.POINTER(vp)]),
    "sag_matrix_create": (C.c_int, [vp, C.c_int, C.c_int, C.c_longlong, vp, vp, vp, C.POINTER(vp)]),
    "sag_matrix_destroy": (C.c_int, [vp]),
    "sag_matrix_shape": (C.c_int, [vp, i32p, i32p, i64p]),
    "sag_spmv": (C.c_int, [vp, vp, vp, vp]),
    "sag_spmv_fused": (C.c_int, [vp, vp, vp, vp, vp, C.c_int]),
    "sag_norm2": (C.c_int, [vp, C.c_int, vp, f64p]),
    "sag_dot": (C.c_int, [vp, C.c_int, vp, vp, f64p]),
    "sag_build_patches": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "sag_patches_create": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, vp, C.POINTER(vp)]),
    "sag_patches_destroy": (C.c_int, [vp]),
    "sag_patches_info": (C.c_int, [vp, i64p]),
    "sag_patches_export": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    "sag_factor_patches": (C.c_int, [vp, vp, vp, C.c_int, C.POINTER(vp)]),
    "sag_vanka_destroy": (C.c_int, [vp]),
    "sag_vanka_stats": (C.c_int, [vp, i64p]),
    "sag_vanka_classes": (C.c_int, [vp, i64p, C.c_int, C.POINTER(C.c_int)]),
    "sag_vanka_export": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "sag_apply_vanka": (C.c_int, [vp, vp, vp, vp]),
    "sag_apply_vanka_stage": (C.c_int, [vp, vp, vp, vp, C.c_int]),
    "sag_vanka_spmv": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "sag_apply_vanka_add": (C.c_int, [vp, vp, vp, vp, C.c_double]),
    "sag_apply_vanka_add_push": (C.c_int, [vp, vp, vp, vp, C.c_double, vp, vp, C.c_int,
                                           C.POINTER(vp)]),
    "sag_vanka_set_weights": (C.c_int, [vp, vp, vp]),
    "sag_vanka_relax": (C.c_int, [vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_double]),
    "sag_fgmres": (C.c_int, [vp, vp, vp, vp, C.c_int, vp, C.POINTER(sag_fgmres_options),
                             C.POINTER(sag_krylov_report), vp, C.c_int]),
    "sag_solver_config_default": (C.c_int, [C.POINTER(sag_solver_config)]),
    "sag_solver_config_check": (C.c_int, [C.POINTER(sag_solver_config)]),
    "sag_dc_create": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                C.POINTER(sag_level_desc), C.POINTER(sag_solver_config),
                                C.POINTER(vp)]),
    "sag_dc_destroy": (C.c_int, [vp]),
    "sag_dc_set_parameters": (C.c_int, [vp, C.c_double, C.c_double, C.c_double]),
    "sag_dc_set_sv_transfer": (C.c_int, [vp, vp, vp, C.c_int, C.POINTER(vp), C.POINTER(vp)]),
    "sag_dc_apply": (C.c_int, [vp, vp, vp, vp]),
    "sag_dc_vcycle": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_int]),
    "sag_dc_counters": (C.c_int, [vp, i64p]),
    "sag_dc_info": (C.c_int, [vp, i64p, C.c_int]),
    "sag_dc_proj_trace": (C.c_int, [vp, vp, vp, C.c_longlong]),
    "sag_vanka_step_plan": (C.c_int, [vp, i64p, C.c_int]),
    "sag_solve_stokes": (C.c_int, [vp, vp, vp, vp, C.POINTER(sag_solver_config),
                                   C.POINTER(sag_krylov_report), vp, C.c_int]),
    "sag_uzawa_create": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(sag_scalar_hierarchy), C.POINTER(sag_scalar_hierarchy),
                                   C.POINTER(sag_scalar_hierarchy), vp,
                                   C.POINTER(sag_solver_config), C.POINTER(vp)]),
    "sag_uzawa_destroy": (C.c_int, [vp]),
    "sag_uzawa_apply": (C.c_int, [vp, vp, vp, vp]),
    "sag_solve_stokes_uzawa": (C.c_int, [vp, vp, vp, vp, vp, C.POINTER(sag_solver_config),
                                         C.POINTER(sag_krylov_report), vp, C.c_int]),
    # hierarchy setup products (bitwise the reference's)
    "sag_spgemm": (C.c_int, [vp, vp, vp, C.POINTER(vp)]),
    "sag_transpose": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "sag_galerkin": (C.c_int, [vp, vp, vp, C.POINTER(vp)]),
    "sag_smooth_prolongator": (C.c_int, [vp, vp, vp, C.c_double, C.POINTER(vp)]),
    "sag_matrix_export": (C.c_int, [vp, vp, vp, vp, vp]),
    "sag_tentative_prolongator": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, C.POINTER(vp), vp]),
    "sag_power_rho": (C.c_int, [vp, vp, vp, vp, C.c_int, f64p]),
    "sag_saddle_matrix": (C.c_int, [vp, vp, vp, C.POINTER(vp)]),
    "sag_evolution_soc": (C.c_int, [vp, vp, C.c_double, C.c_double, C.c_int, C.POINTER(vp)]),
    # 3 velocity components (config 5)
    "sag_factor_patches3": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(vp)]),
    "sag_vanka3_destroy": (C.c_int, [vp]),
    "sag_vanka3_stats": (C.c_int, [vp, i64p]),
    "sag_apply_vanka3": (C.c_int, [vp, vp, vp, vp]),
    # FEM assembly (bitwise the reference's)
    "sag_from_triplets": (C.c_int, [vp, C.c_int, C.c_int, C.c_longlong, vp, vp, vp,
                                    C.POINTER(vp)]),
    "sag_sort_permutation": (C.c_int, [vp, C.c_longlong, vp, vp, C.POINTER(C.c_int)]),
    "sag_assemble_p2": (C.c_int, [vp, C.POINTER(sag_mesh2d), C.c_int, vp, C.POINTER(vp),
                                  C.POINTER(vp), vp, vp, C.POINTER(vp), C.POINTER(vp), vp]),
    "sag_assemble_p1": (C.c_int, [vp, C.POINTER(sag_mesh2d), C.POINTER(vp), C.POINTER(vp)]),
    "sag_assemble_iso": (C.c_int, [vp, C.POINTER(sag_mesh2d), vp, C.POINTER(vp), C.POINTER(vp),
                                   vp, vp]),
    "sag_reduce_dirichlet": (C.c_int, [vp, vp, vp, C.c_int, vp, vp, vp, C.POINTER(vp),
                                       C.POINTER(vp), vp, vp, vp]),
    # partitioned solve (multi-GPU)
    "sag_nccl_unique_id": (C.c_int, [vp]),
    "sag_comm_create_nccl": (C.c_int, [vp, C.c_int, C.c_int, vp, C.POINTER(vp)]),
    "sag_comm_create_host": (C.c_int, [C.c_int, C.c_int, C.POINTER(sag_comm_ops),
                                       C.POINTER(vp)]),
    "sag_comm_destroy": (C.c_int, [vp]),
    "sag_comm_allreduce": (C.c_int, [vp, vp, vp, C.c_longlong]),
    "sag_dist_create": (C.c_int, [vp, vp, C.POINTER(sag_csr), C.c_int, C.c_int, C.c_int,
                                  C.c_int, vp, vp, vp, C.POINTER(sag_solver_config),
                                  C.POINTER(vp)]),
    "sag_dist_destroy": (C.c_int, [vp]),
    "sag_dist_info": (C.c_int, [vp, i64p]),
    "sag_dist_local_dofs": (C.c_int, [vp, vp, vp]),
    "sag_dist_step": (C.c_int, [vp, vp, vp, vp, vp]),
    "sag_dist_solve_stokes": (C.c_int, [vp, vp, vp, vp, C.POINTER(sag_krylov_report), vp,
                                        C.c_int]),
    "sag_plan_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(sag_csr), C.POINTER(sag_csr),
                                  C.POINTER(sag_csr), C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "sag_plan_destroy": (C.c_int, [vp]),
    "sag_plan_array": (C.c_int, [vp, C.c_int, C.c_int, vp, i64p]),
    # partitioned-solve primitives (device pointers, no host sync)
    "sag_dot_async": (C.c_int, [vp, C.c_int, vp, vp, vp, vp]),
    "sag_axpy_async": (C.c_int, [vp, C.c_int, vp, C.c_double, vp, vp]),
    "sag_div_async": (C.c_int, [vp, C.c_int, vp, vp, C.c_int, vp]),
    "sag_sub_mean_async": (C.c_int, [vp, C.c_int, vp, vp, C.c_double, vp]),
    "sag_fgmres1_coef_async": (C.c_int, [vp, vp, vp, vp, vp]),
    "sag_axpby_async": (C.c_int, [vp, C.c_int, C.c_double, vp, C.c_double, vp]),
    "sag_gather_async": (C.c_int, [vp, C.c_int, vp, vp, vp]),
    "sag_scatter_async": (C.c_int, [vp, C.c_int, vp, vp, vp, C.c_int]),
    "sag_matrix_norm_inf": (C.c_int, [vp, vp, f64p]),
    "sag_ipc_get_handle": (C.c_int, [vp, vp, vp]),
    "sag_ipc_open_handle": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "sag_ipc_close_handle": (C.c_int, [vp, vp]),
    "sag_push_async": (C.c_int, [vp, C.c_int, vp, vp, vp]),
    "sag_dc_set_coarse_pin": (C.c_int, [vp, vp, C.c_double]),
}

_lib = None


def lib():
    """Loads libsag.so (fails loudly: there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                            "(no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        msg = lib().sag_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, Error)(msg)


# --------------------------------------------------------------- vectors --
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _vec_in(x, n: int):
    """(pointer, keepalive) for a host (numpy) or device (torch CUDA) vector."""
    if _is_torch(x):
        if not x.is_cuda:
            x = x.detach().cpu().numpy()
        else:
            assert x.dtype.is_floating_point and x.element_size() == 8 and x.is_contiguous()
            if x.numel() != n:
                raise DimensionMismatch(f"vector length {x.numel()} != {n}")
            return C.c_void_p(x.data_ptr()), x
    a = np.ascontiguousarray(x, dtype=np.float64)
    if a.size != n:
        raise DimensionMismatch(f"vector length {a.size} != {n}")
    return C.c_void_p(a.ctypes.data), a


def _vec_out(out, n: int, like=None):
    if out is None:
        if like is not None and _is_torch(like) and like.is_cuda:
            import torch
            out = torch.empty(n, dtype=torch.float64, device=like.device)
        else:
            out = np.empty(n, dtype=np.float64)
    if _is_torch(out):
        return C.c_void_p(out.data_ptr()), out
    if out.dtype != np.float64 or not out.flags.c_contiguous or out.size != n:
        raise DimensionMismatch("output must be a contiguous float64 vector of length %d" % n)
    return C.c_void_p(out.ctypes.data), out


def _ints(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return C.c_void_p(a.ctypes.data), a


# --------------------------------------------------------------- context --
class Context:
    """One CUDA device + stream + workspaces (no reference analogue)."""

    def __init__(self, device: int = 0, stream: int = None):
        """``stream``: a caller-owned cudaStream_t (e.g. ``torch.cuda.Stream().cuda_stream``)
        to launch on; libsag then never destroys it (sag_create_on_stream)."""
        h = vp()
        if stream is None:
            _check(lib().sag_create(device, C.byref(h)))
        else:
            _check(lib().sag_create_on_stream(device, C.c_void_p(stream), C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            lib().sag_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(lib().sag_synchronize(self.h))

    def launch_count(self) -> int:
        v = C.c_longlong()
        _check(lib().sag_launch_count(self.h, C.byref(v)))
        return v.value

    def stream_ptr(self) -> int:
        s = vp()
        _check(lib().sag_stream(self.h, C.byref(s)))
        return s.value or 0


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("SAG_DEVICE", "0")))
    return _default_ctx


# ---------------------------------------------------------------- sparse --
class SparseMatrix:
    """Device CSR (sparse.hpp:11-28): canonical rows, int32 indices, fp64."""

    def __init__(self, nrows, ncols, row_offsets, col_indices, values, ctx: Context = None):
        self.ctx = ctx or default_context()
        rp, self._rp = _ints(row_offsets)
        ci, self._ci = _ints(col_indices)
        v = np.ascontiguousarray(values, dtype=np.float64)
        h = vp()
        _check(lib().sag_matrix_create(self.ctx.h, int(nrows), int(ncols), int(self._rp[-1]),
                                       rp, ci, C.c_void_p(v.ctypes.data), C.byref(h)))
        self.h = h
        self.nrows, self.ncols, self.nnz = int(nrows), int(ncols), int(self._rp[-1])
        del self._rp, self._ci

    @classmethod
    def _wrap(cls, h, ctx: Context) -> "SparseMatrix":
        m = cls.__new__(cls)
        m.ctx, m.h = ctx, h
        nr, nc, nnz = C.c_int(), C.c_int(), C.c_longlong()
        _check(lib().sag_matrix_shape(h, C.byref(nr), C.byref(nc), C.byref(nnz)))
        m.nrows, m.ncols, m.nnz = nr.value, nc.value, nnz.value
        return m

    def to_csr(self):
        """(row_offsets, col_indices, values) as numpy arrays (sag_matrix_export)."""
        rp = np.empty(self.nrows + 1, dtype=np.int32)
        ci = np.empty(max(self.nnz, 1), dtype=np.int32)
        v = np.empty(max(self.nnz, 1))
        _check(lib().sag_matrix_export(self.ctx.h, self.h, C.c_void_p(rp.ctypes.data),
                                       C.c_void_p(ci.ctypes.data), C.c_void_p(v.ctypes.data)))
        return rp, ci[:self.nnz], v[:self.nnz]

    @classmethod
    def from_csr(cls, m, ctx: Context = None) -> "SparseMatrix":
        """From any object with nrows/ncols/rp/ci/v (oracle.Csr) or a scipy matrix."""
        if hasattr(m, "rp"):
            return cls(m.nrows, m.ncols, m.rp, m.ci, m.v, ctx)
        m = m.tocsr()
        m.sort_indices()
        return cls(m.shape[0], m.shape[1], m.indptr, m.indices, m.data, ctx)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().sag_matrix_destroy(self.h)
        except Exception:
            pass


def spmv(m: SparseMatrix, x, out=None):
    """y = m x (sparse.cpp:78-91)."""
    xp, xk = _vec_in(x, m.ncols)
    yp, y = _vec_out(out, m.nrows, like=x)
    _check(lib().sag_spmv(m.ctx.h, m.h, xp, yp))
    return y


def _new(fn, ctx, *args):
    h = vp()
    _check(fn(ctx.h, *args, C.byref(h)))
    return SparseMatrix._wrap(h, ctx)


def from_triplets(nrows: int, ncols: int, rows, cols, values, ctx: Context = None) -> SparseMatrix:
    """from_triplets (sparse.cpp:43-66) on the device: duplicates summed in
    the order libstdc++'s std::sort leaves them, exact zeros dropped."""
    ctx = ctx or default_context()
    r = np.ascontiguousarray(rows, dtype=np.int32)
    c = np.ascontiguousarray(cols, dtype=np.int32)
    v = np.ascontiguousarray(values, dtype=np.float64)
    if not (len(r) == len(c) == len(v)):
        raise DimensionMismatch("from_triplets: rows, cols and values differ in length")
    h = vp()
    _check(lib().sag_from_triplets(ctx.h, int(nrows), int(ncols), len(v), r.ctypes.data,
                                   c.ctypes.data, v.ctypes.data, C.byref(h)))
    return SparseMatrix._wrap(h, ctx)


def sort_permutation(keys, ctx: Context = None):
    """(perm, heap_ranges): std::sort's permutation of uint64 keys reproduced
    on the device (the order from_triplets sums duplicates in)."""
    ctx = ctx or default_context()
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    p = np.empty(len(k), dtype=np.int32)
    nh = C.c_int()
    _check(lib().sag_sort_permutation(ctx.h, len(k), k.ctypes.data, p.ctypes.data, C.byref(nh)))
    return p, nh.value


def tentative_prolongator(node_to_agg, num_aggregates: int, nullvec, ctx: Context = None):
    """tentative_prolongator_with_nullvec (amg.cpp:184-205) on the device:
    (T, coarse nullvec)."""
    ctx = ctx or default_context()
    a = np.ascontiguousarray(node_to_agg, dtype=np.int32)
    nv = np.ascontiguousarray(nullvec, dtype=np.float64)
    if len(a) != len(nv):
        raise DimensionMismatch("tentative_prolongator: aggregation and nullvec differ in length")
    cn = np.empty(max(int(num_aggregates), 1))
    h = vp()
    _check(lib().sag_tentative_prolongator(ctx.h, len(a), int(num_aggregates), a.ctypes.data,
                                           nv.ctypes.data, C.byref(h), cn.ctypes.data))
    return SparseMatrix._wrap(h, ctx), cn[:int(num_aggregates)]


def power_rho(m: SparseMatrix, d_inv, x0, iters: int = 10) -> float:
    """power_rho_estimate (sparse.cpp:239-261) from a normalised start vector."""
    d = np.ascontiguousarray(d_inv, dtype=np.float64)
    x = np.ascontiguousarray(x0, dtype=np.float64)
    out = C.c_double()
    _check(lib().sag_power_rho(m.ctx.h, m.h, d.ctypes.data, x.ctypes.data, int(iters),
                               C.byref(out)))
    return out.value


def spgemm(a: SparseMatrix, b: SparseMatrix) -> SparseMatrix:
    """C = A B, bitwise the reference's spgemm (sparse.cpp:113-150)."""
    return _new(lib().sag_spgemm, a.ctx, a.h, b.h)


def transpose(a: SparseMatrix) -> SparseMatrix:
    """A^T (sparse.cpp:93-111)."""
    return _new(lib().sag_transpose, a.ctx, a.h)


def galerkin_triple(p: SparseMatrix, k: SparseMatrix) -> SparseMatrix:
    """P^T K P, bitwise the reference's galerkin_triple (sparse.cpp:152-156)."""
    return _new(lib().sag_galerkin, p.ctx, p.h, k.h)


def saddle_matrix(a: SparseMatrix, b: SparseMatrix) -> SparseMatrix:
    """[[A, B^T], [B, 0]] (assemble_saddle_matrix, fem.cpp:290-306)."""
    return _new(lib().sag_saddle_matrix, a.ctx, a.h, b.h)


def evolution_soc(a: SparseMatrix, omega: float, theta: float = 0.5, k: int = 2) -> SparseMatrix:
    """Strength graph of evolution_soc (amg.cpp:45-110) for omega = 4 / (3 rho),
    as a CSR of edge strengths (bitwise the reference's StrengthGraph)."""
    return _new(lib().sag_evolution_soc, a.ctx, a.h, C.c_double(omega), C.c_double(theta),
                int(k))


def smooth_prolongator(a: SparseMatrix, t: SparseMatrix, omega: float) -> SparseMatrix:
    """T - omega D^-1 A T (amg.cpp:226-236) for omega = omega_frac / rho."""
    return _new(lib().sag_smooth_prolongator, a.ctx, a.h, t.h, C.c_double(omega))


def norm2(v, ctx: Context = None) -> float:
    ctx = ctx or default_context()
    n = v.numel() if _is_torch(v) else len(v)
    p, k = _vec_in(v, n)
    out = C.c_double()
    _check(lib().sag_norm2(ctx.h, n, p, C.byref(out)))
    return out.value


def dot(a, b, ctx: Context = None) -> float:
    ctx = ctx or default_context()
    n = a.numel() if _is_torch(a) else len(a)
    pa, ka = _vec_in(a, n)
    pb, kb = _vec_in(b, n)
    out = C.c_double()
    _check(lib().sag_dot(ctx.h, n, pa, pb, C.byref(out)))
    return out.value


# ----------------------------------------------------------------- vanka --
@dataclass
class PatchLists:
    pressure_ptr: np.ndarray
    pressure: np.ndarray
    velocity_ptr: np.ndarray
    velocity: np.ndarray
    nx: np.ndarray


class Patches:
    """Vanka patch sets (vanka.hpp:11-15) on the device."""

    def __init__(self, h, ctx: Context):
        self.h, self.ctx = h, ctx
        info = np.zeros(5, dtype=np.int64)
        _check(lib().sag_patches_info(h, info.ctypes.data_as(i64p)))
        self.npatch, self.total_pressure, self.total_velocity, self.max_nv, self.max_np = (
            int(v) for v in info)

    @classmethod
    def from_lists(cls, pressure_ptr, pressure, velocity_ptr, velocity, nx,
                   ctx: Context = None) -> "Patches":
        ctx = ctx or default_context()
        arrs = [_ints(a) for a in (pressure_ptr, pressure, velocity_ptr, velocity, nx)]
        h = vp()
        _check(lib().sag_patches_create(ctx.h, len(arrs[4][1]), *[a[0] for a in arrs],
                                        C.byref(h)))
        return cls(h, ctx)

    def export(self) -> PatchLists:
        pp = np.empty(self.npatch + 1, dtype=np.int32)
        vpp = np.empty(self.npatch + 1, dtype=np.int32)
        pi = np.empty(max(self.total_pressure, 1), dtype=np.int32)
        vi = np.empty(max(self.total_velocity, 1), dtype=np.int32)
        nx = np.empty(max(self.npatch, 1), dtype=np.int32)
        _check(lib().sag_patches_export(self.ctx.h, self.h, *[C.c_void_p(a.ctypes.data)
                                                               for a in (pp, pi, vpp, vi, nx)]))
        return PatchLists(pp, pi[:self.total_pressure], vpp, vi[:self.total_velocity],
                          nx[:self.npatch])

    def __del__(self):
        try:
            lib().sag_patches_destroy(self.h)
        except Exception:
            pass


def build_patches(k: SparseMatrix, n_x: int, n_y: int, n_p: int,
                  sv_triples: bool = False) -> Patches:
    """build_patches (vanka.cpp:11-42)."""
    h = vp()
    _check(lib().sag_build_patches(k.ctx.h, k.h, n_x, n_y, n_p, int(sv_triples), C.byref(h)))
    return Patches(h, k.ctx)


class VankaFactorization:
    """factor_patches result (vanka.hpp:23-40), device resident."""

    def __init__(self, h, ctx: Context, k: SparseMatrix):
        self.h, self.ctx, self.k = h, ctx, k
        s = np.zeros(7, dtype=np.int64)
        _check(lib().sag_vanka_stats(h, s.ctypes.data_as(i64p)))
        (self.a_factor_bytes, self.aux_bytes, self.dense_inverse_bytes, self.device_bytes,
         self.npatch, self.n, self.nslots) = (int(v) for v in s)

    def classes(self):
        """The apply's launch classes: [(kernel, R, lanes per patch, patches,
        blob bytes)] in launch order."""
        out = np.zeros(4 * 16, dtype=np.int64)
        nc = C.c_int()
        _check(lib().sag_vanka_classes(self.h, out.ctypes.data_as(i64p), 16, C.byref(nc)))
        res = []
        for i in range(min(nc.value, 16)):
            R, lpp, npch, nb = (int(v) for v in out[4 * i:4 * i + 4])
            kern = ("vanka_fixed_kernel<6,3>" if lpp == 9 else
                    f"vanka_subwarp_kernel<{lpp}>" if lpp < 32 else f"vanka_patch_kernel<R={R}>")
            res.append((kern, R, lpp, npch, nb))
        return res

    def export(self, patches: PatchLists):
        nv = np.diff(patches.velocity_ptr).astype(np.int64)
        npp = np.diff(patches.pressure_ptr).astype(np.int64)
        aux = int((nv * npp).sum())
        ss = int((npp * npp).sum())
        u = np.empty(max(aux, 1))
        b = np.empty(max(aux, 1))
        s = np.empty(max(ss, 1))
        w = np.empty(self.n)
        _check(lib().sag_vanka_export(self.ctx.h, self.h, *[C.c_void_p(a.ctypes.data)
                                                             for a in (u, b, s, w)]))
        return dict(uhat=u[:aux], bhat=b[:aux], sinv=s[:ss], weights=w)

    def set_weights(self, w):
        """Global PoU weights for a rank holding part of the patches."""
        p, keep = _vec_in(w, self.n)
        _check(lib().sag_vanka_set_weights(self.ctx.h, self.h, p))

    def __del__(self):
        try:
            lib().sag_vanka_destroy(self.h)
        except Exception:
            pass


def factor_patches(k: SparseMatrix, patches: Patches, n_u: int) -> VankaFactorization:
    """factor_patches (vanka.cpp:64-149): batched block LU on the device."""
    h = vp()
    _check(lib().sag_factor_patches(k.ctx.h, k.h, patches.h, int(n_u), C.byref(h)))
    return VankaFactorization(h, k.ctx, k)


def apply_vanka(f: VankaFactorization, r, out=None):
    """delta = sum_i V_i^T W K_i^-1 V_i r (vanka.cpp:151-184)."""
    rp, rk = _vec_in(r, f.n)
    dp, d = _vec_out(out, f.n, like=r)
    _check(lib().sag_apply_vanka(f.ctx.h, f.h, rp, dp))
    return d


def vanka_step_plan(f: VankaFactorization):
    """Plan of the last pipelined host-buffer step of f (sag_vanka_step_plan)."""
    v = np.zeros(9, dtype=np.int64)
    _check(lib().sag_vanka_step_plan(f.h, v.ctypes.data_as(i64p), 9))
    return dict(stages=int(v[0]), ranges=int(v[1]), in_ranges=int(v[2]), row_ranges=int(v[3]),
                gather_ranges=int(v[4]), patch_windows=int(v[5]),
                choice={1: "pipelined", -1: "plain", 0: "untimed"}[int(v[6])],
                plain_ms=v[7] * 1e-6, pipelined_ms=v[8] * 1e-6)


def vanka_spmv_step(f: VankaFactorization, k: SparseMatrix, x, delta=None, y=None):
    """The hot step in one call: (apply_vanka(f, x), spmv(k, x)) with x read
    once (sag_vanka_spmv; vanka.cpp:151-184, sparse.cpp:78-91)."""
    xp, xk = _vec_in(x, f.n)
    dp, d = _vec_out(delta, f.n, like=x)
    yp, yy = _vec_out(y, k.nrows, like=x)
    _check(lib().sag_vanka_spmv(f.ctx.h, f.h, k.h, xp, dp, yp))
    return d, yy


class RelaxMode:
    KrylovWrapped = 0
    Stationary = 1


def vanka_relax(k: SparseMatrix, f: VankaFactorization, x, b, mode: int, sweeps: int,
                omega: float = 1.0):
    """vanka_relax (vanka.cpp:186-209); x is updated in place and returned."""
    if not _is_torch(x):
        if not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.c_contiguous):
            raise TypeError("x must be a contiguous float64 numpy array (updated in place)")
    xp, xk = _vec_out(x, k.nrows)
    bp, bk = _vec_in(b, k.nrows)
    _check(lib().sag_vanka_relax(k.ctx.h, k.h, f.h, xp, bp, int(mode), int(sweeps),
                                 float(omega)))
    return x


# ---------------------------------------------------------------- krylov --
@dataclass
class FgmresOptions:
    """krylov.hpp:17-22"""
    tol: float = 1e-8
    max_iters: int = 500
    restart: int = 20
    breakdown: float = 1e-30


@dataclass
class KrylovReport:
    """krylov.hpp:24-29"""
    converged: bool = False
    iterations: int = 0
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    final_relative_residual: float = 0.0


def fgmres(a: SparseMatrix, b, x, prec=None, opt: FgmresOptions = None) -> KrylovReport:
    """fgmres(matrix_operator(a), b, x, prec, opt) (krylov.cpp:17-121). ``prec``
    is None (identity), a VankaFactorization, a SparseMatrix (Jacobi on its
    diagonal) or a DCPreconditioner. x (guess) is updated in place."""
    opt = opt or FgmresOptions()
    if prec is None:
        kind, ph = 0, None
    elif isinstance(prec, VankaFactorization):
        kind, ph = 1, prec.h
    elif isinstance(prec, SparseMatrix):
        kind, ph = 2, prec.h
    elif isinstance(prec, DCPreconditioner):
        kind, ph = 3, prec.h
    elif isinstance(prec, UzawaPreconditioner):
        kind, ph = 4, prec.h
    else:
        raise ConfigError("unsupported preconditioner object")
    bp, bk = _vec_in(b, a.nrows)
    xp, xk = _vec_out(x, a.nrows)
    rep = sag_krylov_report()
    cap = opt.max_iters + 2
    hist = np.zeros(cap)
    o = sag_fgmres_options(opt.tol, opt.max_iters, opt.restart, opt.breakdown)
    _check(lib().sag_fgmres(a.ctx.h, a.h, bp, xp, kind, ph, C.byref(o), C.byref(rep),
                            C.c_void_p(hist.ctypes.data), cap))
    return KrylovReport(bool(rep.converged), rep.iterations,
                        hist[:min(rep.iterations + 1, cap)].copy(), rep.final_relative_residual)


# -------------------------------------------------------- preconditioner --
class Variant:
    """preconditioner.hpp:14"""
    DCall = 0
    DCLO = 1
    DCHO = 2
    HOAMG = 3
    Uzawa = 4


@dataclass
class SolverConfig:
    """preconditioner.hpp:19-36 (reference defaults)."""
    variant: int = Variant.DCall
    eta_u: float = 1.0
    eta_p: float = 1.0
    omega0: float = 1.0
    nu1: int = 2
    nu2: int = 2
    gamma: int = 1
    restart: int = 20
    tol: float = 1e-10
    max_iters: int = 200
    enclosed_flow: bool = False
    allow_sv_hoamg: bool = False

    def to_c(self) -> sag_solver_config:
        return sag_solver_config(int(self.variant), float(self.eta_u), float(self.eta_p),
                                 float(self.omega0), int(self.nu1), int(self.nu2),
                                 int(self.gamma), int(self.restart), float(self.tol),
                                 int(self.max_iters), int(bool(self.enclosed_flow)),
                                 int(bool(self.allow_sv_hoamg)))

    def check(self):
        c = self.to_c()
        _check(lib().sag_solver_config_check(C.byref(c)))


class DCPreconditioner:
    """DCPreconditioner (preconditioner.hpp:77-100) on a host-built hierarchy.

    ``k0``: SparseMatrix of the high-order system with block sizes ``nxyz0``;
    ``levels``: [(K_l SparseMatrix, P_l SparseMatrix | None, (n_x, n_y, n_p))]
    of the low-order monolithic hierarchy (amg.hpp:85-93, as produced by the
    reference's build_monolithic_hierarchy)."""

    def __init__(self, k0: SparseMatrix, nxyz0: Sequence[int], levels, cfg: SolverConfig,
                 sv: bool = False):
        self.ctx = k0.ctx
        self.k0 = k0
        self.levels = levels  # keep the device matrices alive
        self.cfg = cfg
        descs = (sag_level_desc * len(levels))()
        for i, (k, p, (nx, ny, npp)) in enumerate(levels):
            descs[i] = sag_level_desc(k.h.value if k is not None else None,
                                      p.h.value if p is not None else None, nx, ny, npp)
        h = vp()
        c = cfg.to_c()
        _check(lib().sag_dc_create(self.ctx.h, k0.h, int(nxyz0[0]), int(nxyz0[1]),
                                   int(nxyz0[2]), int(sv), len(levels), descs, C.byref(c),
                                   C.byref(h)))
        self.h = h
        self.n = k0.nrows
        self.n_p = int(nxyz0[2])
        self.sv = sv

    def set_sv_transfer(self, p_dup: SparseMatrix, m_mix: SparseMatrix, scalar_levels,
                        scalar_prolongators):
        self._sv_keep = (p_dup, m_mix, scalar_levels, scalar_prolongators)
        L = (vp * len(scalar_levels))(*[m.h.value for m in scalar_levels])
        P = (vp * max(len(scalar_prolongators), 1))(*[m.h.value for m in scalar_prolongators])
        _check(lib().sag_dc_set_sv_transfer(self.h, p_dup.h, m_mix.h, len(scalar_levels), L, P))

    def set_parameters(self, eta_u: float, eta_p: float, omega0: float):
        _check(lib().sag_dc_set_parameters(self.h, eta_u, eta_p, omega0))
        self.cfg.eta_u, self.cfg.eta_p, self.cfg.omega0 = eta_u, eta_p, omega0

    def apply(self, r, out=None):
        rp, rk = _vec_in(r, self.n)
        zp, z = _vec_out(out, self.n, like=r)
        _check(lib().sag_dc_apply(self.ctx.h, self.h, rp, zp))
        return z

    def vcycle(self, b, nu1: int, nu2: int, out=None):
        n1 = self.levels[0][0].nrows
        bp, bk = _vec_in(b, n1)
        xp, x = _vec_out(out, n1, like=b)
        _check(lib().sag_dc_vcycle(self.ctx.h, self.h, bp, xp, nu1, nu2))
        return x

    @property
    def fine_relax_units(self) -> int:
        return self._counters()[0]

    @property
    def level1_relax_units(self) -> int:
        return self._counters()[1]

    def _counters(self):
        v = np.zeros(2, dtype=np.int64)
        _check(lib().sag_dc_counters(self.h, v.ctypes.data_as(i64p)))
        return int(v[0]), int(v[1])

    def info(self):
        v = np.zeros(32, dtype=np.int64)
        _check(lib().sag_dc_info(self.h, v.ctypes.data_as(i64p), 32))
        nl = int(v[0])
        return dict(nlevels=nl, n0=int(v[1]), level_rows=[int(x) for x in v[2:2 + nl]],
                    factor_bytes=int(v[2 + nl]), graph_launches=int(v[3 + nl]),
                    proj_fused=bool(v[4 + nl]), proj_grid_levels=int(v[5 + nl]),
                    proj_ctas=int(v[6 + nl]), proj_workers=int(v[7 + nl]))

    def proj_trace(self):
        """Diagnostic: (tags, ns) of the last one-launch SV mass projection for
        worker CTA 0 and tail CTA 0 (needs SAG_PROJ_TRACE=1 at setup)."""
        cap = 8192
        buf = np.zeros(4 * cap, dtype=np.uint64)
        _check(lib().sag_dc_proj_trace(self.ctx.h, self.h, buf.ctypes.data, buf.size))
        return buf[:2 * cap].reshape(-1, 2), buf[2 * cap:].reshape(-1, 2)

    def size(self):
        return self.n

    def pressure_size(self):
        return self.n_p

    def __del__(self):
        try:
            lib().sag_dc_destroy(self.h)
        except Exception:
            pass


def HoAmgPreconditioner(k0: SparseMatrix, levels, cfg: SolverConfig, sv: bool = False):
    """HoAmgPreconditioner (preconditioner.hpp:103-118): one V-cycle of the
    monolithic hierarchy built on the high-order system itself (levels[0] is
    K0; build_monolithic_hierarchy(sys0) on the host). A DCPreconditioner
    object in HO-AMG mode (sag_dc_create with variant HOAMG)."""
    from dataclasses import replace
    c = replace(cfg, variant=Variant.HOAMG)
    return DCPreconditioner(k0, levels[0][2], levels, c, sv=sv)


def _scalar_desc(levels, prolongators):
    a = (vp * len(levels))(*[m.h.value for m in levels])
    p = (vp * max(len(prolongators), 1))(*([m.h.value for m in prolongators] or [None]))
    return sag_scalar_hierarchy(len(levels), a, p), (a, p)


class UzawaPreconditioner:
    """UzawaPreconditioner (preconditioner.hpp:118-141): scalar V-cycles on
    A_x and A_y, t = B du - r_p, then the Mp V-cycle (TH/ISO) or the exact SV
    element mass inverse. ``hx``/``hy``/``hp``: (matrices, prolongators) of the
    host-built ScalarHierarchy objects; ``sv_element_areas`` for SV."""

    def __init__(self, b: SparseMatrix, n_x: int, n_y: int, n_p: int, hx, hy, hp=None,
                 sv_element_areas=None, cfg: SolverConfig = None):
        self.ctx = b.ctx
        self.n = n_x + n_y + n_p
        self.n_p = n_p
        self._keep = (b, hx, hy, hp)
        dx, kx = _scalar_desc(*hx)
        dy, ky = _scalar_desc(*hy)
        dp, kp = _scalar_desc(*hp) if hp is not None else (None, None)
        areas = None
        if sv_element_areas is not None:
            areas = np.ascontiguousarray(sv_element_areas, dtype=np.float64)
        self._descs = (dx, dy, dp, kx, ky, kp, areas)
        c = (cfg or SolverConfig()).to_c()
        h = vp()
        _check(lib().sag_uzawa_create(
            self.ctx.h, b.h, int(n_x), int(n_y), int(n_p), C.byref(dx), C.byref(dy),
            C.byref(dp) if dp is not None else None,
            C.c_void_p(areas.ctypes.data) if areas is not None else None, C.byref(c),
            C.byref(h)))
        self.h = h

    def apply(self, r, out=None):
        rp, rk = _vec_in(r, self.n)
        zp, z = _vec_out(out, self.n, like=r)
        _check(lib().sag_uzawa_apply(self.ctx.h, self.h, rp, zp))
        return z

    def size(self):
        return self.n

    def pressure_size(self):
        return self.n_p

    def __del__(self):
        try:
            lib().sag_uzawa_destroy(self.h)
        except Exception:
            pass


def solve_stokes(k0: SparseMatrix, rhs, prec, cfg: SolverConfig, x=None):
    """solve_stokes (preconditioner.cpp:229-259) with a DC / HO-AMG or an Uzawa
    preconditioner: returns (x, KrylovReport)."""
    bp, bk = _vec_in(rhs, prec.n)
    xp, xo = _vec_out(x, prec.n, like=rhs)
    rep = sag_krylov_report()
    cap = cfg.max_iters + 2
    hist = np.zeros(cap)
    c = cfg.to_c()
    if isinstance(prec, UzawaPreconditioner):
        if k0.nrows != prec.n:
            raise DimensionMismatch("solve_stokes: K0 does not match the preconditioner size")
        _check(lib().sag_solve_stokes_uzawa(prec.ctx.h, k0.h, prec.h, bp, xp, C.byref(c),
                                            C.byref(rep), C.c_void_p(hist.ctypes.data), cap))
    else:
        if k0 is not prec.k0:
            raise ConfigError("solve_stokes: k0 must be the preconditioner's high-order operator")
        _check(lib().sag_solve_stokes(prec.ctx.h, prec.h, bp, xp, C.byref(c), C.byref(rep),
                                      C.c_void_p(hist.ctypes.data), cap))
    return xo, KrylovReport(bool(rep.converged), rep.iterations,
                            hist[:min(rep.history_len, cap)].copy(),
                            rep.final_relative_residual)


# ------------------------------------------------------- multi-GPU (8(e)) --
def _csr_struct(m, keep):
    rp = np.ascontiguousarray(m.rp, dtype=np.int32)
    ci = np.ascontiguousarray(m.ci, dtype=np.int32)
    v = np.ascontiguousarray(m.v, dtype=np.float64)
    keep.extend([rp, ci, v])
    return sag_csr(int(m.nrows), int(m.ncols), rp.ctypes.data, ci.ctypes.data, v.ctypes.data)


_PLAN_DTYPES = {0: np.int64, 1: np.int64, 2: np.uint8, 9: np.float64, 12: np.float64}


def partition_plan(nranks: int, rank: int, k0, l0, p0, nxyz):
    """libsag's partition plan of one rank (host only; sag_plan_*): a dict of
    the arrays partition.build_rank_systems states in numpy."""
    keep = []
    ks, ls = _csr_struct(k0, keep), _csr_struct(l0, keep)
    ps = _csr_struct(p0, keep) if p0 is not None else None
    h = vp()
    _check(lib().sag_plan_create(int(nranks), int(rank), C.byref(ks), C.byref(ls),
                                 C.byref(ps) if ps is not None else None, *map(int, nxyz),
                                 C.byref(h)))

    def arr(which, peer=0):
        cnt = C.c_longlong()
        _check(lib().sag_plan_array(h, which, peer, None, C.byref(cnt)))
        dt = _PLAN_DTYPES.get(which % 100, np.int32)
        out = np.empty(max(cnt.value, 1), dtype=dt)
        _check(lib().sag_plan_array(h, which, peer, out.ctypes.data, C.byref(cnt)))
        return out[:cnt.value]
    try:
        info = arr(0)
        res = {"info": info, "l2g": arr(1), "owned": arr(2)}
        for name, w in (("fwd_send", 3), ("fwd_recv", 4), ("rev_send", 5), ("rev_recv", 6)):
            res[name] = {q: arr(w, q) for q in range(nranks) if q != rank and len(arr(w, q))}
        for lvl, base in (("K0", 0), ("L0", 100)):
            res[lvl] = {k: arr(base + w) for k, w in (("ext_rp", 7), ("ext_ci", 8), ("ext_v", 9),
                                                       ("int_vidx", 10), ("bnd_vidx", 11),
                                                       ("weights", 12))}
        res["p_rp"], res["p_ci"] = arr(13), arr(14)
        return res
    finally:
        lib().sag_plan_destroy(h)


def nccl_unique_id() -> bytes:
    b = (C.c_ubyte * 128)()
    _check(lib().sag_nccl_unique_id(b))
    return bytes(b)


class Comm:
    """sag_comm: NCCL (nccl_id: 128 bytes from rank 0's nccl_unique_id) or the
    caller's host-staged collectives (allreduce(np.ndarray) in place,
    exchange(sends: [(peer, ndarray)], recvs: [(peer, ndarray)]))."""

    def __init__(self, ctx: Context, nranks: int, rank: int, nccl_id: bytes = None,
                 allreduce=None, exchange=None):
        self.ctx, self.size, self.rank = ctx, nranks, rank
        h = vp()
        if nccl_id is not None:
            b = (C.c_ubyte * 128).from_buffer_copy(nccl_id)
            _check(lib().sag_comm_create_nccl(ctx.h, nranks, rank, b, C.byref(h)))
            self._ops = None
        else:
            def ar(user, buf, n):
                try:
                    allreduce(np.ctypeslib.as_array(C.cast(buf, f64p), (n,)))
                    return 0
                except Exception:  # noqa: BLE001
                    return 1

            def ex(user, ns, to, sb, sc, nr, frm, rb, rc):
                try:
                    to_ = C.cast(to, i32p)
                    sb_ = C.cast(sb, C.POINTER(f64p))
                    sc_ = C.cast(sc, i64p)
                    fr_ = C.cast(frm, i32p)
                    rb_ = C.cast(rb, C.POINTER(f64p))
                    rc_ = C.cast(rc, i64p)
                    sends = [(to_[i], np.ctypeslib.as_array(sb_[i], (sc_[i],))) for i in range(ns)]
                    recvs = [(fr_[i], np.ctypeslib.as_array(rb_[i], (rc_[i],))) for i in range(nr)]
                    exchange(sends, recvs)
                    return 0
                except Exception:  # noqa: BLE001
                    return 1
            self._ops = sag_comm_ops(None, ALLREDUCE_FN(ar), EXCHANGE_FN(ex))
            _check(lib().sag_comm_create_host(nranks, rank, C.byref(self._ops), C.byref(h)))
        self.h = h

    @staticmethod
    def torch_host(ctx: Context, dist, torch):
        """Host-staged collectives over torch.distributed (gloo)."""
        def allreduce(a):
            t = torch.from_numpy(a)
            dist.all_reduce(t)

        def exchange(sends, recvs):
            ops = [dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(a)), q)
                   for q, a in sends]
            ops += [dist.P2POp(dist.irecv, torch.from_numpy(a), q) for q, a in recvs]
            if ops:
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
        return Comm(ctx, dist.get_world_size(), dist.get_rank(), allreduce=allreduce,
                    exchange=exchange)

    def __del__(self):
        try:
            lib().sag_comm_destroy(self.h)
        except Exception:
            pass


class DistSolver:
    """solve_stokes with the DC preconditioner over a row/patch partition, one
    rank per process (sag_dist_*). k0 and the levels are the GLOBAL host CSR
    arrays (every rank passes the same); vectors are rank-local: l2g / owned
    map them to the global numbering."""

    def __init__(self, comm: Comm, k0, nxyz0, levels, cfg: SolverConfig):
        self.comm, self.ctx, self.cfg = comm, comm.ctx, cfg
        keep = []
        ks = _csr_struct(k0, keep)
        lv = (sag_csr * len(levels))(*[_csr_struct(k, keep) for k, _, _ in levels])
        pv = (sag_csr * max(len(levels) - 1, 1))(*[_csr_struct(p, keep) for _, p, _ in levels[:-1]])
        nx = np.ascontiguousarray(np.array([v for _, _, t in levels for v in t]), dtype=np.int32)
        c = cfg.to_c()
        h = vp()
        _check(lib().sag_dist_create(self.ctx.h, comm.h, C.byref(ks), *map(int, nxyz0),
                                     len(levels), C.cast(lv, vp), C.cast(pv, vp),
                                     nx.ctypes.data, C.byref(c), C.byref(h)))
        self.h = h
        info = np.zeros(7, dtype=np.int64)
        _check(lib().sag_dist_info(h, info.ctypes.data_as(i64p)))
        self.nl, self.n_own, self.ghosts, self.neighbours, self.patches, self.n1, \
            self.n_u_loc = (int(v) for v in info)
        self.l2g = np.empty(self.nl, dtype=np.int64)
        self.owned = np.empty(self.nl, dtype=np.uint8)
        _check(lib().sag_dist_local_dofs(h, self.l2g.ctypes.data, self.owned.ctypes.data))

    def step(self, x, delta=None, y=None):
        xp, xk = _vec_in(x, self.nl)
        dp, d = _vec_out(delta, self.nl, like=x)
        yp, yy = _vec_out(y, self.nl, like=x)
        _check(lib().sag_dist_step(self.ctx.h, self.h, xp, dp, yp))
        return d, yy

    def solve(self, rhs, x=None):
        bp, bk = _vec_in(rhs, self.nl)
        xp, xo = _vec_out(x, self.nl, like=rhs)
        rep = sag_krylov_report()
        cap = self.cfg.max_iters + 2
        hist = np.zeros(cap)
        _check(lib().sag_dist_solve_stokes(self.ctx.h, self.h, bp, xp, C.byref(rep),
                                           C.c_void_p(hist.ctypes.data), cap))
        return xo, KrylovReport(bool(rep.converged), rep.iterations,
                                hist[:min(rep.history_len, cap)].copy(),
                                rep.final_relative_residual)

    def __del__(self):
        try:
            lib().sag_dist_destroy(self.h)
        except Exception:
            pass


# ---------------------------------------------- 3 components (config 5) --
class VankaFactorization3:
    """factor_patches generalised to [x | y | z | p] (BASELINE config 5; the
    reference is 2D only): one pressure seed per patch, one LU per velocity
    component, CTA-per-patch kernels (sag_factor_patches3 / sag_apply_vanka3)."""

    def __init__(self, k: SparseMatrix, n_x: int, n_y: int, n_z: int, n_p: int):
        self.ctx, self.k = k.ctx, k
        h = vp()
        _check(lib().sag_factor_patches3(k.ctx.h, k.h, int(n_x), int(n_y), int(n_z), int(n_p),
                                         C.byref(h)))
        self.h = h
        st = np.zeros(7, dtype=np.int64)
        _check(lib().sag_vanka3_stats(h, st.ctypes.data_as(i64p)))
        (self.npatch, self.n, self.device_bytes, self.max_nv, self.nslots, self.a_factor_bytes,
         self.aux_bytes) = (int(v) for v in st)

    def apply(self, r, out=None):
        rp, rk = _vec_in(r, self.n)
        dp, d = _vec_out(out, self.n, like=r)
        _check(lib().sag_apply_vanka3(self.ctx.h, self.h, rp, dp))
        return d

    def __del__(self):
        try:
            lib().sag_vanka3_destroy(self.h)
        except Exception:
            pass
