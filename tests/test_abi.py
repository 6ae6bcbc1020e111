"""The C-ABI library loads and exports every symbol include/*.h declares.

CPU only: no compute entry point is called without a GPU (host utilities
such as the instance generator and the hyper-parameter helpers are).
"""
import ctypes as C
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(cimcs_[a-z_0-9]+)\s*\(", src))
    return names


def test_header_declares_the_seams():
    names = _declared()
    for f in ("cimcs_create", "cimcs_set_problems", "cimcs_build_coupling", "cimcs_run_cim",
              "cimcs_refit", "cimcs_score", "cimcs_solve", "cimcs_last_error"):
        assert f in names


def test_library_exports_every_declared_symbol():
    from paper_2405_00366_b200 import _lib
    L = _lib.load()
    missing = [n for n in _declared() if not hasattr(L, n)]
    assert not missing, missing
    assert set(_lib.EXPORTS) == _declared()


def test_abi_version_and_order():
    from paper_2405_00366_b200 import _lib, cimcs
    L = _lib.load()
    assert L.cimcs_abi_version() == 1
    assert cimcs.gemv_order("f64") == (8, 8)


def test_hyper_default_matches_reference_defaults():
    from paper_2405_00366_b200 import _lib, cimcs
    h = _lib.Hyper()
    _lib.load().cimcs_hyper_default(C.byref(h))
    d = cimcs.HyperParams()
    for f, _ in _lib.Hyper._fields_:
        assert getattr(h, f) == pytest.approx(float(getattr(d, f))), f
    # types.hpp:77-96
    assert (h.dt, h.n_steps, h.velo, h.jacobi_iters, h.dt_c) == (0.02, 1000, 51, 100, 0.1)


def test_hyper_validate_errors():
    from paper_2405_00366_b200 import cimcs
    cimcs.HyperParams().validate()
    for bad in (dict(dt=0.0), dict(n_steps=0), dict(tau=0.0), dict(g2=-1.0),
                dict(eta_init=0.1, eta_end=0.2), dict(velo=0)):
        with pytest.raises(cimcs.ConfigError):
            cimcs.HyperParams(**bad).validate()


def test_no_gpu_context_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2405_00366_b200 import cimcs
    with pytest.raises((cimcs.CudaError, cimcs.ConfigError)):
        cimcs.Context(0, "f64")


def test_python_mirror_rejects_empty_problem_and_bad_R():
    """The Python mirror raises the reference's InputError (types.hpp:16-33) before shaping
    any host array when no problem is set or R is outside [1, 16] (no GPU call is made)."""
    import numpy as np

    from paper_2405_00366_b200 import cimcs as P

    class Dummy(P.Context):
        def __init__(self):  # no device context: only the host-side checks are exercised
            self.B = self.N = 0

        def close(self):
            pass

    d = Dummy()
    hp = P.baseline_params(velo=1, n_steps=10)
    import pytest
    with pytest.raises(P.InputError):
        d.solve(2, "mfz-bn", hp, np.array([[1, 2]], np.uint64))
    d.B, d.N = 2, 8
    for R in (0, 17):
        with pytest.raises(P.InputError):
            d.solve(R, "mfz-bn", hp, np.zeros((2, max(R, 1)), np.uint64))
        with pytest.raises(P.InputError):
            d.score(R, np.zeros((2, 1, 8)), np.zeros((2, 1, 8), np.int32), 0.1)
