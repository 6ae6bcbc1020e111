"""ctypes face of the reference's OWN solver (oracle/_ref/libref_solver.so).

TEST INFRASTRUCTURE ONLY.  oracle/Makefile.ref compiles the reference's
model.cpp, solver_mfz.cpp, solver_pp.cpp, cdp.cpp and orchestrator.cpp
unmodified from /root/reference/proj against the sequential Eigen shim
(oracle/refshim/Eigen/Dense); this module calls alternating_minimize,
run_cim, cdp_minimize and the scorer through oracle/refshim/ref_solver_capi.cpp.
The reference exists only in the build container: on the GPU box the prebuilt
.so travels with the repo (oracle/_ref/ is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_ref", "libref_solver.so")
# the same sources built for speed (AVX2/FMA, reassociated reductions like
# Eigen's SIMD kernels): bench.py's timed CPU arm only, never a parity pin
SO_SIMD = os.path.join(HERE, "_ref", "libref_solver_simd.so")
_L = {}
_FAST = False


def available(fast: bool = False) -> bool:
    so = SO_SIMD if fast else SO
    if not os.path.exists(so) and os.path.isdir("/root/reference/proj"):
        subprocess.call(["make", "-s", "-C", HERE, "-f", "Makefile.ref"])
    return os.path.exists(so)


def use_fast(flag: bool = True):
    """Route the calls below to the SIMD timing build (bench.py)."""
    global _FAST
    _FAST = flag


def lib():
    so = SO_SIMD if _FAST else SO
    if so not in _L:
        from . import oracle as O
        L = C.CDLL(so)
        vp, i, d, u64 = C.c_void_p, C.c_int, C.c_double, C.c_uint64
        hp = C.POINTER(O._Hyper)
        L.ref_last_error.restype = C.c_char_p
        L.ref_alternating_minimize.argtypes = [i, i, vp, vp, vp, vp, i, hp, u64, vp, i, i, vp,
                                               vp, vp, vp, vp, C.c_char_p, i]
        L.ref_run_cim.argtypes = [i, i, vp, vp, i, hp, d, u64, vp, vp, vp, vp, vp]
        L.ref_cdp_minimize.argtypes = [i, i, vp, vp, vp, vp, i, hp, vp]
        L.ref_score.argtypes = [i, i, vp, vp, vp, vp, vp, vp, d, vp, vp, vp]
        _L[so] = L
    return _L[so]


def _arrs(inst):
    A = np.asfortranarray(inst.A, np.float64)
    y = np.ascontiguousarray(inst.y, np.float64)
    x = None if inst.x_true is None else np.ascontiguousarray(inst.x_true, np.float64)
    xi = None if inst.xi_true is None else np.ascontiguousarray(inst.xi_true, np.int32)
    return A, y, x, xi


def _p(a):
    return None if a is None else a.ctypes.data


def _check(rc):
    if rc:
        raise RuntimeError(f"reference error {rc}: {lib().ref_last_error().decode()}")


def alternating_minimize(inst, backend: int, hp, seed: int, R_init=None, cdp: int = 0,
                         track_best: bool = False) -> dict:
    """alternating_minimize(make_problem(inst), ...) of the reference (orchestrator.cpp:170-235)."""
    A, y, x, xi = _arrs(inst)
    M, N = A.shape
    R = np.zeros(N)
    s = np.zeros(N, np.int32)
    hist = np.zeros((hp.velo + 1, 7))
    nh, fa = C.c_int(), C.c_int()
    msg = C.create_string_buffer(256)
    r0 = None if R_init is None else np.ascontiguousarray(R_init, np.float64)
    h = hp.to_c()
    _check(lib().ref_alternating_minimize(N, M, _p(A), _p(y), _p(x), _p(xi), backend,
                                          C.byref(h), seed, _p(r0), cdp, int(track_best),
                                          _p(R), _p(s), _p(hist), C.byref(nh), C.byref(fa),
                                          msg, 256))
    return dict(R=R, sigma=s, history=hist[: nh.value], fail_alternation=fa.value,
                failed=fa.value >= 0, fail_reason=msg.value.decode())


def run_cim(inst, backend: int, hp, eta: float, seed: int, R) -> dict:
    A, y, _, _ = _arrs(inst)
    M, N = A.shape
    s = np.zeros(N, np.int32)
    e = np.zeros(N)
    amp = np.zeros(N)
    me = C.c_double()
    h = hp.to_c()
    Rv = np.ascontiguousarray(R, np.float64)
    _check(lib().ref_run_cim(N, M, _p(A), _p(y), backend, C.byref(h), eta, seed, _p(Rv), _p(s),
                             _p(e), _p(amp), C.byref(me)))
    return dict(sigma=s, e=e, amplitude=amp, min_e=me.value)


def cdp_minimize(inst, sigma, R_prev, hp, cdp: int = 0):
    A, y, _, _ = _arrs(inst)
    M, N = A.shape
    out = np.zeros(N)
    s = np.ascontiguousarray(sigma, np.int32)
    rp = np.ascontiguousarray(R_prev, np.float64)
    h = hp.to_c()
    _check(lib().ref_cdp_minimize(N, M, _p(A), _p(y), _p(s), _p(rp), cdp, C.byref(h), _p(out)))
    return out


def score(inst, R, sigma, lam: float):
    A, y, x, xi = _arrs(inst)
    M, N = A.shape
    o, r, hm = C.c_double(), C.c_double(), C.c_double()
    Rv = np.ascontiguousarray(R, np.float64)
    s = np.ascontiguousarray(sigma, np.int32)
    _check(lib().ref_score(N, M, _p(A), _p(y), _p(x), _p(xi), _p(Rv), _p(s), lam, C.byref(o),
                           C.byref(r), C.byref(hm)))
    return o.value, r.value, hm.value
