import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and libsag.so")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


_CASES = {}


def ref_case(n, sv=False, problem="cavity", cfg=None):
    """Reference-built case (oracle/_ref): (RefCase, RefDC, k0 Csr, levels Csr)."""
    import oracle as O
    key = (n, sv, problem, tuple(sorted((cfg or {}).items())))
    if key not in _CASES:
        c = O.RefCase.build(problem, sv, "structured", n)
        conf = dict(nu1=1, nu2=1, restart=30, tol=1e-8, max_iters=500,
                    enclosed_flow=c.enclosed)
        conf.update(cfg or {})
        d = O.RefDC(c, conf)
        _CASES[key] = (c, d, d.k0().csr(), d.levels_csr(), conf)
    return _CASES[key]


@pytest.fixture(scope="session")
def ctx():
    import paper_2306_06795_b200 as S
    return S.default_context()


def collect_results(q, procs, n, timeout=600):
    """n results from worker processes: fails fast when a worker dies (a dead
    worker never puts its result, and waiting for it would hang the suite)."""
    import queue
    import time
    out, deadline = [], time.time() + timeout
    while len(out) < n:
        try:
            out.append(q.get(timeout=2))
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            if dead:
                raise AssertionError(f"worker exited with {dead}")
            if time.time() > deadline:
                raise TimeoutError("workers did not report in time")
    return out
