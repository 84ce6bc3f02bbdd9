"""CPU: the drop-in boundary. libsag.so / libsag_stokesamg.so load, export every
symbol include/sag.h declares, the Python mirror binds all of them, the pure
host-side entry points behave like the reference (SolverConfig defaults and
checks, preconditioner.hpp:19-36 / preconditioner.cpp:30-38), and without a
GPU the product path fails loudly instead of falling back to the CPU."""
import ctypes as C
import os
import re

import pytest

import paper_2306_06795_b200 as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sag.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(sag_\w+)\(", txt, re.M)))


def test_header_declares_the_boundary():
    syms = header_symbols()
    for must in ["sag_spmv", "sag_build_patches", "sag_factor_patches", "sag_apply_vanka",
                 "sag_vanka_relax", "sag_fgmres", "sag_dc_create", "sag_dc_apply",
                 "sag_dc_vcycle", "sag_solve_stokes", "sag_last_error"]:
        assert must in syms


def test_library_exports_every_declared_symbol():
    lib = S.lib()
    for s in header_symbols():
        assert hasattr(lib, s), s


def test_python_mirror_binds_every_declared_symbol():
    assert sorted(S.SIGNATURES) == header_symbols()


def test_config_defaults_match_reference():
    c = S.sag_solver_config()
    assert S.lib().sag_solver_config_default(C.byref(c)) == 0
    ref = S.SolverConfig()
    assert (c.variant, c.eta_u, c.eta_p, c.omega0, c.nu1, c.nu2, c.gamma, c.restart, c.tol,
            c.max_iters, c.enclosed_flow) == (ref.variant, ref.eta_u, ref.eta_p, ref.omega0,
                                              ref.nu1, ref.nu2, ref.gamma, ref.restart,
                                              ref.tol, ref.max_iters, int(ref.enclosed_flow))
    ref.check()


@pytest.mark.parametrize("field,value", [("eta_p", 0.0), ("gamma", 0), ("omega0", 2.5),
                                         ("tol", -1.0), ("nu1", -1), ("restart", 0),
                                         ("max_iters", 0)])
def test_config_invariants_enforced(field, value):
    # tests/test_preconditioner.cpp:42-60
    c = S.SolverConfig()
    setattr(c, field, value)
    with pytest.raises(S.ConfigError):
        c.check()


def test_no_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    with pytest.raises(S.CudaError):
        S.Context(0)


def test_host_adapter_exports():
    path = os.path.join(ROOT, "paper_2306_06795_b200", "libsag_stokesamg.so")
    if not os.path.exists(path):
        pytest.skip("host adapter not built")
    lib = C.CDLL(path)
    for s in ["sagh_case_build", "sagh_case_matrix_copy", "sagh_case_solve"]:
        assert hasattr(lib, s)
    # the C++ drop-in classes (stokesamg::gpu::DCPreconditioner, solve_stokes)
    out = os.popen(f"nm -DC {path}").read()
    assert "stokesamg::gpu::DCPreconditioner::DCPreconditioner" in out
    assert "stokesamg::gpu::solve_stokes" in out


def test_host_case_builds_reference_hierarchy():
    path = os.path.join(ROOT, "paper_2306_06795_b200", "libsag_stokesamg.so")
    if not os.path.exists(path):
        pytest.skip("host adapter not built")
    from paper_2306_06795_b200.cases import HostCase
    import numpy as np
    import oracle as O
    h = HostCase("cavity", False, "structured", 16)
    gold = dict(np.load(os.path.join(ROOT, "tests", "golden", "th_cavity_16.npz")))
    k0 = h.k0()
    assert np.array_equal(k0.rp, gold["k0_rp"]) and np.array_equal(k0.v, gold["k0_v"])
    assert h.nlevels == int(gold["nlevels"])
    for l in range(h.nlevels):
        k, p, nxyz = h.level(l)
        assert np.array_equal(k.v, gold[f"L{l}_k_v"])
        assert tuple(nxyz) == tuple(gold[f"L{l}_nxyz"])
    assert np.array_equal(h.rhs(), gold["rhs"])
    _ = O  # the host case and the oracle agree through the golden fixture


@pytest.mark.parametrize("name,args", [
    ("sag_spgemm", (None, None, None, None)),
    ("sag_transpose", (None, None, None)),
    ("sag_galerkin", (None, None, None, None)),
    ("sag_smooth_prolongator", (None, None, None, C.c_double(1.0), None)),
    ("sag_evolution_soc", (None, None, C.c_double(1.0), C.c_double(0.5), 2, None)),
    ("sag_saddle_matrix", (None, None, None, None)),
    ("sag_matrix_export", (None, None, None, None, None)),
    ("sag_dot_async", (None, 0, None, None, None, None)),
    ("sag_axpy_async", (None, 0, None, C.c_double(-1.0), None, None)),
    ("sag_gather_async", (None, 0, None, None, None)),
    ("sag_vanka_spmv", (None, None, None, None, None, None)),
    ("sag_apply_vanka_add", (None, None, None, None, C.c_double(1.0))),
    ("sag_dc_set_coarse_pin", (None, None, C.c_double(1.0))),
])
def test_entry_points_reject_null_handles(name, args):
    """The boundary's error convention (errors.hpp:8-58 + SAG_INVALID_ARGUMENT):
    a null handle is a status code and a message, never a crash -- checkable
    without a GPU."""
    fn = getattr(S.lib(), name)
    assert fn(*args) == 101
    assert S.lib().sag_last_error()


def test_host_case_device_setup_entry_exported():
    path = os.path.join(ROOT, "paper_2306_06795_b200", "libsag_stokesamg.so")
    if not os.path.exists(path):
        pytest.skip("host adapter not built")
    out = os.popen(f"nm -DC {path}").read()
    assert "stokesamg::gpu::build_monolithic_hierarchy" in out
    assert "stokesamg::gpu::build_scalar_hierarchy" in out
    lib = C.CDLL(path)
    assert hasattr(lib, "sagh_case_hierarchy_gpu") and hasattr(lib, "sagh_case_scalar_hierarchy_gpu")
