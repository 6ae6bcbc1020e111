"""ctypes front-end of the C oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: the CPU restatement of the reference MFZ-CIM
L0RBCS path used as the parity checker for the CUDA product.  Only tests/,
``__graft_entry__.smoke()`` and bench.py's CPU-baseline / ``--impl reference``
legs may import this module.  The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field, fields

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

LITERAL, CANON, EXPLICIT = 0, 1, 2
MFZ_CN, MFZ_BN, PP = 0, 1, 2
CDP_JACOBI, CDP_CG = 0, 1
PUMP_SIGMOID, PUMP_LINEAR = 0, 1
BACKENDS = {"mfz-cn": MFZ_CN, "mfz-bn": MFZ_BN, "pp": PP}


def build() -> str:
    src = os.path.join(_HERE, "oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        subprocess.check_call(["make", "-s", "-C", _HERE, "liboracle.so"])
    return _LIB_PATH


class _Hyper(C.Structure):
    _fields_ = [
        ("g2", C.c_double), ("j", C.c_double), ("K", C.c_double), ("beta", C.c_double),
        ("tau", C.c_double), ("dt", C.c_double), ("n_steps", C.c_int),
        ("p_thr", C.c_double), ("d", C.c_double), ("eta_init", C.c_double),
        ("eta_end", C.c_double), ("velo", C.c_int), ("dt_c", C.c_double),
        ("jacobi_iters", C.c_int), ("cg_max_iters", C.c_int), ("cg_tol", C.c_double),
        ("gamma", C.c_double), ("mfz_loss_minus_j", C.c_int), ("mu_abort", C.c_double),
        ("pump_kind", C.c_int), ("pump_end", C.c_double),
    ]


class _Record(C.Structure):
    _fields_ = [
        ("i", C.c_int32), ("support", C.c_int32), ("eta", C.c_double),
        ("hamiltonian", C.c_double), ("rmse", C.c_double), ("hamming", C.c_double),
        ("min_e", C.c_double), ("median_e", C.c_double),
    ]


class _Problem(C.Structure):
    _fields_ = [
        ("N", C.c_int), ("M", C.c_int), ("mode", C.c_int), ("nseg", C.c_int),
        ("gran", C.c_int), ("A", C.c_void_p), ("y", C.c_void_p), ("G", C.c_void_p),
        ("hz", C.c_void_p), ("D", C.c_void_p), ("work", C.c_void_p),
        ("x_true", C.c_void_p), ("xi_true", C.c_void_p),
    ]


class _Rng(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("mti", C.c_int), ("n_gauss", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        d, i, u64, vp = C.c_double, C.c_int, C.c_uint64, C.c_void_p
        L.orc_rng_raw.restype = u64
        L.orc_uniform_open.restype = d
        L.orc_uniform_below.restype = u64
        L.orc_uniform_below.argtypes = [vp, u64]
        L.orc_gauss.restype = d
        L.orc_rng_init.argtypes = [vp, u64]
        L.orc_mix_seed.restype = u64
        L.orc_mix_seed.argtypes = [u64, u64]
        L.orc_round_half_away.restype = C.c_longlong
        L.orc_round_half_away.argtypes = [d]
        L.orc_gen_dims.argtypes = [i, d, d, vp, vp]
        L.orc_gen_instance.argtypes = [i, d, d, d, u64, vp, vp, vp, vp]
        for f in ("orc_pump_sigmoid", "orc_pump_linear"):
            getattr(L, f).restype = d
            getattr(L, f).argtypes = [d, d, d]
        L.orc_eta_schedule.restype = d
        L.orc_eta_schedule.argtypes = [i, d, d, i]
        L.orc_trace_stride.argtypes = [i, i]
        L.orc_problem_init.argtypes = [vp, i, i, vp, vp, i, i, i]
        L.orc_problem_init_gram.argtypes = [vp, i, vp, vp]
        L.orc_canon_dot.restype = d
        L.orc_canon_dot.argtypes = [vp, vp, i, i, i]
        L.orc_local_field_cn.argtypes = [vp, vp, vp, d, vp]
        L.orc_local_field_bn.argtypes = [vp, vp, vp, d, vp]
        L.orc_mfz_step.argtypes = [i, vp, vp, d, vp, d, vp, vp, vp, vp]
        L.orc_run_mfz.argtypes = [vp, vp, vp, d, i, vp, vp, vp, vp, vp, i, vp, vp, vp, vp, i]
        L.orc_cdp_minimize.argtypes = [vp, vp, vp, i, vp, vp, vp]
        L.orc_measured_amplitude.argtypes = [i, vp, vp, vp, vp]
        L.orc_local_field_pp.argtypes = [vp, vp, vp, d, vp]
        L.orc_pp_step.argtypes = [i, vp, vp, vp, vp, d, vp, d, vp, vp, vp, vp, vp, vp, vp]
        L.orc_run_pp.argtypes = [vp, vp, vp, d, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        for f in ("orc_objective_at", "orc_hamiltonian_at"):
            getattr(L, f).restype = d
            getattr(L, f).argtypes = [vp, vp, vp, d]
        for f in ("orc_hamiltonian", "orc_objective"):
            getattr(L, f).restype = d
            getattr(L, f).argtypes = [i, i, vp, vp, vp, vp, d]
        L.orc_rmse.restype = d
        L.orc_rmse.argtypes = [i, vp, vp, vp, vp]
        L.orc_hamming.restype = d
        L.orc_hamming.argtypes = [i, vp, vp]
        L.orc_median.restype = d
        L.orc_median.argtypes = [i, vp]
        L.orc_alternating_minimize.argtypes = [vp, i, vp, vp, vp, i, i, vp, vp, vp, vp, vp,
                                               vp, vp, vp]
        L.orc_solve_batch.restype = d
        L.orc_solve_batch.argtypes = [i, i, i, vp, vp, vp, vp, vp, i, i, i, i, vp, vp, i, vp,
                                      vp, vp]
        L.orc_solve_batch_limited.restype = d
        L.orc_solve_batch_limited.argtypes = [i, i, i, i, vp, vp, vp, i, i, vp, vp, vp, vp]
        L.orc_pump_table.argtypes = [vp, vp]
        L.orc_hyper_validate.argtypes = [vp]
    return _lib


def _p(a):
    return a.ctypes.data if a is not None else None


# ----------------------------------------------------------------- errors
class ConfigError(RuntimeError):
    pass


class InputError(ValueError):
    pass


# ----------------------------------------------------------- hyperparams
@dataclass
class HyperParams:
    """types.hpp:77-96 (+ ⊕ pump_kind / pump_end)."""
    g2: float = 1e-7
    j: float = 1.0
    K: float = 1.0
    beta: float = 0.2
    tau: float = 1.0
    dt: float = 0.02
    n_steps: int = 1000
    p_thr: float = 1.0
    d: float = 0.4
    eta_init: float = 0.8
    eta_end: float = 0.18
    velo: int = 51
    dt_c: float = 0.1
    jacobi_iters: int = 100
    cg_max_iters: int = 10000
    cg_tol: float = 1e-10
    gamma: float = 1e-4
    mfz_loss_minus_j: bool = False
    mu_abort: float = 100.0
    pump_kind: int = PUMP_SIGMOID
    pump_end: float = 1.2

    def to_c(self) -> _Hyper:
        h = _Hyper()
        for f in fields(self):
            setattr(h, f.name, type(getattr(h, f.name))(getattr(self, f.name)))
        return h


def baseline_params(velo: int = 19, n_steps: int = 1000) -> HyperParams:
    """BASELINE configs 0-2: dt=0.01, linear pump 0->1.2, velo=19 (20 outer iterations)."""
    return HyperParams(dt=0.01, n_steps=n_steps, velo=velo, pump_kind=PUMP_LINEAR, pump_end=1.2)


# ---------------------------------------------------------------- RNG
class Rng:
    def __init__(self, seed: int):
        self._s = _Rng()
        lib().orc_rng_init(C.byref(self._s), C.c_uint64(seed))

    def raw(self) -> int:
        return lib().orc_rng_raw(C.byref(self._s))

    def uniform_open(self) -> float:
        return lib().orc_uniform_open(C.byref(self._s))

    def uniform_below(self, b: int) -> int:
        return lib().orc_uniform_below(C.byref(self._s), b)

    def gauss(self) -> float:
        return lib().orc_gauss(C.byref(self._s))

    def gauss_vector(self, n: int) -> np.ndarray:
        return np.array([self.gauss() for _ in range(n)])

    @property
    def gauss_count(self) -> int:
        return self._s.n_gauss

    @property
    def ptr(self):
        return C.byref(self._s)


def mix_seed(base: int, salt: int) -> int:
    return lib().orc_mix_seed(base, salt)


def round_half_away(v: float) -> int:
    return lib().orc_round_half_away(v)


def pump_schedule(t, p_thr, d):
    return lib().orc_pump_sigmoid(t, p_thr, d)


def pump_linear(t, p_end, T):
    return lib().orc_pump_linear(t, p_end, T)


def eta_schedule(i, eta_init, eta_end, velo):
    if velo < 1:
        raise ConfigError("eta_schedule: velo must be >= 1")
    return lib().orc_eta_schedule(i, eta_init, eta_end, velo)


def trace_stride(n_steps, cap=500):
    return lib().orc_trace_stride(n_steps, cap)


def pump_table(hp: HyperParams) -> np.ndarray:
    out = np.zeros(hp.n_steps)
    h = hp.to_c()
    lib().orc_pump_table(C.byref(h), _p(out))
    return out


# ------------------------------------------------------------- instances
@dataclass
class Instance:
    A: np.ndarray  # M x N, Fortran order (col-major like Eigen)
    y: np.ndarray
    x_true: np.ndarray | None = None
    xi_true: np.ndarray | None = None
    a: float = 0.0
    alpha: float = 0.0
    nu: float = 0.0
    seed: int = 0

    @property
    def N(self):
        return self.A.shape[1]

    @property
    def M(self):
        return self.A.shape[0]


def gen_instance(N, alpha, a, nu, seed) -> Instance:
    M, K = C.c_int(), C.c_int()
    if lib().orc_gen_dims(N, alpha, a, C.byref(M), C.byref(K)) or nu < 0:
        raise InputError("gen_instance: bad arguments")
    A = np.zeros((M.value, N), order="F")
    y = np.zeros(M.value)
    x = np.zeros(N)
    xi = np.zeros(N, dtype=np.int32)
    rc = lib().orc_gen_instance(N, alpha, a, nu, seed, _p(A), _p(y), _p(x), _p(xi))
    if rc:
        raise InputError("gen_instance: bad arguments")
    return Instance(A, y, x, xi, a, alpha, nu, seed)


# --------------------------------------------------------------- problem
class Problem:
    """make_problem(inst) with a chosen coupling mode (see oracle.h)."""

    def __init__(self, inst: Instance, mode=CANON, nseg=8, gran=8):
        self.inst = inst
        self.A = np.asfortranarray(inst.A, dtype=np.float64)
        self.y = np.ascontiguousarray(inst.y, dtype=np.float64)
        self._x = None if inst.x_true is None else np.ascontiguousarray(inst.x_true, np.float64)
        self._xi = None if inst.xi_true is None else np.ascontiguousarray(inst.xi_true, np.int32)
        self.N, self.M = self.A.shape[1], self.A.shape[0]
        self.mode = mode
        self._p = _Problem()
        rc = lib().orc_problem_init(C.byref(self._p), self.N, self.M, _p(self.A), _p(self.y),
                                    mode, nseg, gran)
        if rc:
            raise InputError("problem init failed")
        self._p.x_true = _p(self._x)
        self._p.xi_true = _p(self._xi)

    def __del__(self):
        try:
            lib().orc_problem_free(C.byref(self._p))
        except Exception:
            pass

    @classmethod
    def from_gram(cls, G, hz, x_true=None, xi_true=None):
        """make_problem(G_full, hz) (orchestrator.cpp:100-115): an assembled
        quadratic form (e.g. mri.assemble_operators) instead of an instance."""
        self = cls.__new__(cls)
        G = np.ascontiguousarray(G, np.float64)
        self._G = G
        self._hz = np.ascontiguousarray(hz, np.float64)
        self.N, self.M = G.shape[0], 0
        self.inst = None
        self.A = self.y = None
        self._x = None if x_true is None else np.ascontiguousarray(x_true, np.float64)
        self._xi = None if xi_true is None else np.ascontiguousarray(xi_true, np.int32)
        self.mode = EXPLICIT
        self._p = _Problem()
        if lib().orc_problem_init_gram(C.byref(self._p), self.N, _p(G), _p(self._hz)):
            raise InputError("problem init failed")
        self._p.x_true = _p(self._x)
        self._p.xi_true = _p(self._xi)
        return self

    @property
    def has_truth(self):
        return self._x is not None

    def _vec(self, ptr, n):
        return np.ctypeslib.as_array((C.c_double * n).from_address(ptr)).copy()

    @property
    def hz(self):
        return self._vec(self._p.hz, self.N)

    @property
    def gram_diag(self):
        return self._vec(self._p.D, self.N)

    @property
    def G(self):
        if not self._p.G:
            return None
        return self._vec(self._p.G, self.N * self.N).reshape(self.N, self.N)

    def apply_gram(self, w):
        w = np.ascontiguousarray(w, np.float64)
        out = np.zeros(self.N)
        lib().orc_gram_apply(C.byref(self._p), _p(w), _p(out))
        return out

    def apply_coupling(self, w):
        w = np.ascontiguousarray(w, np.float64)
        out = np.zeros(self.N)
        lib().orc_coupling_apply(C.byref(self._p), _p(w), _p(out))
        return out

    def local_field_cn(self, R, c, tau):
        R, c = (np.ascontiguousarray(v, np.float64) for v in (R, c))
        h = np.zeros(self.N)
        lib().orc_local_field_cn(C.byref(self._p), _p(R), _p(c), tau, _p(h))
        return h

    def local_field_bn(self, R, sigma, tau):
        R = np.ascontiguousarray(R, np.float64)
        s = np.ascontiguousarray(sigma, np.int32)
        h = np.zeros(self.N)
        lib().orc_local_field_bn(C.byref(self._p), _p(R), _p(s), tau, _p(h))
        return h

    def run_mfz(self, R, hp: HyperParams, eta, backend, rng: Rng, trace_mode=0):
        """run_mfz solver_mfz.cpp:90-124.  Returns dict (raises DivergenceError)."""
        R = np.ascontiguousarray(R, np.float64)
        c = np.zeros(self.N)
        e = np.zeros(self.N)
        s = np.zeros(self.N, np.int32)
        me = C.c_double()
        h = hp.to_c()
        cap = hp.n_steps + 1 if trace_mode else 0
        tsteps = np.zeros(max(cap, 1), np.int32)
        tc = np.zeros((max(cap, 1), self.N))
        te = np.zeros((max(cap, 1), self.N))
        cnt = C.c_int(0)
        rc = lib().orc_run_mfz(C.byref(self._p), _p(R), C.byref(h), eta, backend, rng.ptr,
                               _p(c), _p(e), _p(s), C.byref(me), trace_mode, C.byref(cnt),
                               _p(tsteps), _p(tc), _p(te), cap)
        if rc >= 0:
            raise DivergenceError(f"mfz_step: non-finite amplitude at spin {rc}", rc)
        if rc == -2:
            raise InputError("mfz_step: non-finite pump")
        if rc == -3:
            raise ConfigError("invalid hyper-parameters")
        out = dict(c=c, e=e, sigma=s, min_e=me.value)
        if trace_mode:
            n = cnt.value
            out["trace_steps"] = tsteps[:n].copy()
            out["trace_c"] = tc[:n].copy()
            out["trace_e"] = te[:n].copy()
        return out

    def local_field_pp(self, R, mt, tau):
        """local_field_pp solver_pp.cpp:31-38."""
        out = np.zeros(self.N)
        lib().orc_local_field_pp(C.byref(self._p), _p(np.ascontiguousarray(R, np.float64)),
                                 _p(np.ascontiguousarray(mt, np.float64)), tau, _p(out))
        return out

    def run_pp(self, R, hp: HyperParams, eta, rng: Rng):
        """run_pp solver_pp.cpp:100-132.  Returns dict (raises DivergenceError)."""
        R = np.ascontiguousarray(R, np.float64)
        N = self.N
        mu, n, m, e, mt = (np.zeros(N) for _ in range(5))
        s = np.zeros(N, np.int32)
        me = C.c_double()
        kind = C.c_int(0)
        h = hp.to_c()
        rc = lib().orc_run_pp(C.byref(self._p), _p(R), C.byref(h), eta, rng.ptr, _p(mu), _p(n),
                              _p(m), _p(e), _p(mt), _p(s), C.byref(me), C.byref(kind))
        if rc == -3:
            raise ConfigError("invalid hyper-parameters")
        if rc >= 0:
            if kind.value:
                raise DivergenceError(f"run_pp: |mu| exceeded {hp.mu_abort:f} at spin {rc}", rc)
            raise DivergenceError(f"pp_step: non-finite value at spin {rc}", rc)
        return dict(mu=mu, n=n, m=m, e=e, mu_tilde=mt, sigma=s, min_e=me.value)

    def cdp(self, sigma, R_prev, method=CDP_JACOBI, hp: HyperParams | None = None):
        hp = hp or HyperParams()
        s = np.ascontiguousarray(sigma, np.int32)
        Rp = np.ascontiguousarray(R_prev, np.float64)
        out = np.zeros(self.N)
        bad = C.c_int(-1)
        h = hp.to_c()
        rc = lib().orc_cdp_minimize(C.byref(self._p), _p(s), _p(Rp), method, C.byref(h),
                                    _p(out), C.byref(bad))
        if rc:
            raise InputError(f"jacobi_solve: singular diagonal at active index {bad.value}")
        return out

    def objective_at(self, R, sigma, lam):
        R = np.ascontiguousarray(R, np.float64)
        s = np.ascontiguousarray(sigma, np.int32)
        return lib().orc_objective_at(C.byref(self._p), _p(R), _p(s), lam)

    def hamiltonian_at(self, R, sigma, lam):
        R = np.ascontiguousarray(R, np.float64)
        s = np.ascontiguousarray(sigma, np.int32)
        return lib().orc_hamiltonian_at(C.byref(self._p), _p(R), _p(s), lam)

    def alternating_minimize(self, backend, hp: HyperParams, rng: Rng, R_init=None,
                             cdp=CDP_JACOBI, track_best=False, keep=False):
        R0 = self.hz if R_init is None else np.ascontiguousarray(R_init, np.float64)
        N = self.N
        Rout = np.zeros(N)
        sout = np.zeros(N, np.int32)
        hist = (_Record * (hp.velo + 1))()
        nh, fa, fi = C.c_int(), C.c_int(), C.c_int()
        hR = np.zeros((hp.velo + 1, N)) if keep else None
        hS = np.zeros((hp.velo + 1, N), np.int32) if keep else None
        h = hp.to_c()
        rc = lib().orc_alternating_minimize(C.byref(self._p), backend, C.byref(h), _p(R0),
                                            rng.ptr, cdp, int(track_best), _p(Rout), _p(sout),
                                            hist, C.byref(nh), _p(hR), _p(hS), C.byref(fa),
                                            C.byref(fi))
        if rc == 2:
            raise ConfigError("invalid hyper-parameters")
        if rc == 1:
            raise InputError(f"input error (index {fi.value})")
        H = [dict(i=r.i, eta=r.eta, hamiltonian=r.hamiltonian, rmse=r.rmse, hamming=r.hamming,
                  min_e=r.min_e, median_e=r.median_e, support=r.support)
             for r in hist[: nh.value]]
        res = dict(R=Rout, sigma=sout, history=H, failed=fa.value >= 0,
                   fail_alternation=fa.value, fail_index=fi.value,
                   fail_reason=((f"pp: divergence at spin {fi.value}" if backend == PP else
                                 f"mfz_step: non-finite amplitude at spin {fi.value}")
                                if fa.value >= 0 else ""))
        res["min_hamiltonian"] = min((r["hamiltonian"] for r in H), default=math.nan)
        res["final_rmse"] = H[-1]["rmse"] if H else math.nan
        res["final_hamming"] = H[-1]["hamming"] if H else math.nan
        if keep:
            res["hist_R"] = hR[: nh.value]
            res["hist_sigma"] = hS[: nh.value]
        return res


class DivergenceError(RuntimeError):
    def __init__(self, msg, index):
        super().__init__(msg)
        self.offending_index = index


def mfz_step(c, e, p, hp: HyperParams, eta, R, h):
    c, e, R, h = (np.ascontiguousarray(v, np.float64) for v in (c, e, R, h))
    N = c.size
    co, eo = np.zeros(N), np.zeros(N)
    hc = hp.to_c()
    rc = lib().orc_mfz_step(N, _p(c), _p(e), p, C.byref(hc), eta, _p(R), _p(h), _p(co), _p(eo))
    if rc == -2:
        raise InputError("mfz_step: non-finite pump")
    if rc >= 0:
        raise DivergenceError(f"mfz_step: non-finite amplitude at spin {rc}", rc)
    return co, eo


def measured_amplitude(mu, noise, hp: HyperParams):
    """measured_amplitude solver_pp.cpp:22-29."""
    mu = np.ascontiguousarray(mu, np.float64)
    out = np.zeros_like(mu)
    h = hp.to_c()
    if lib().orc_measured_amplitude(len(mu), _p(mu), _p(np.ascontiguousarray(noise, np.float64)),
                                    C.byref(h), _p(out)):
        raise ConfigError("measured_amplitude: j must be positive")
    return out


def pp_step(mu, n, m, e, p, hp: HyperParams, eta, R, h, noise):
    """pp_step solver_pp.cpp:45-98 -> (mu, n, m, e); raises DivergenceError."""
    arrs = [np.ascontiguousarray(x, np.float64) for x in (mu, n, m, e, R, h, noise)]
    N = len(arrs[0])
    if any(len(x) != N for x in arrs):
        raise InputError("pp_step: length mismatch")
    outs = [np.zeros(N) for _ in range(4)]
    hh = hp.to_c()
    rc = lib().orc_pp_step(N, _p(arrs[0]), _p(arrs[1]), _p(arrs[2]), _p(arrs[3]), p, C.byref(hh),
                           eta, _p(arrs[4]), _p(arrs[5]), _p(arrs[6]), *[_p(o) for o in outs])
    if rc >= 0:
        raise DivergenceError(f"pp_step: non-finite value at spin {rc}", rc)
    return tuple(outs)


def canon_dot(g, v, nseg=8, gran=8):
    g, v = (np.ascontiguousarray(a, np.float64) for a in (g, v))
    return lib().orc_canon_dot(_p(g), _p(v), g.size, nseg, gran)


def rmse(R, sigma, x, xi):
    R, x = (np.ascontiguousarray(a, np.float64) for a in (R, x))
    s, t = (np.ascontiguousarray(a, np.int32) for a in (sigma, xi))
    return lib().orc_rmse(R.size, _p(R), _p(s), _p(x), _p(t))


def hamming_loss(sigma, xi):
    s, t = (np.ascontiguousarray(a, np.int32) for a in (sigma, xi))
    return lib().orc_hamming(s.size, _p(s), _p(t))


def median(v):
    v = np.ascontiguousarray(v, np.float64)
    return lib().orc_median(v.size, _p(v))


def hamiltonian(inst: Instance, R, sigma, lam):
    A = np.asfortranarray(inst.A, np.float64)
    y = np.ascontiguousarray(inst.y, np.float64)
    R = np.ascontiguousarray(R, np.float64)
    s = np.ascontiguousarray(sigma, np.int32)
    return lib().orc_hamiltonian(A.shape[1], A.shape[0], _p(A), _p(y), _p(R), _p(s), lam)


def objective(inst: Instance, R, sigma, lam):
    A = np.asfortranarray(inst.A, np.float64)
    y = np.ascontiguousarray(inst.y, np.float64)
    R = np.ascontiguousarray(R, np.float64)
    s = np.ascontiguousarray(sigma, np.int32)
    return lib().orc_objective(A.shape[1], A.shape[0], _p(A), _p(y), _p(R), _p(s), lam)


def solve(inst: Instance, backend="mfz-bn", params: HyperParams | None = None, seed=1,
          cdp="jacobi", track_best=False, mode=CANON, nseg=8, gran=8):
    """Mirror of the reference's python ``cimcs.solve`` (bindings/module.cpp:127-141)."""
    if backend not in BACKENDS:
        raise ConfigError(f"unknown backend '{backend}' (use mfz-bn, mfz-cn or pp)")
    if cdp not in ("jacobi", "cg"):
        raise ConfigError("cdp must be 'jacobi' or 'cg'")
    params = params or HyperParams()
    prob = Problem(inst, mode, nseg, gran)
    return prob.alternating_minimize(BACKENDS[backend], params, Rng(seed),
                                     cdp=CDP_JACOBI if cdp == "jacobi" else CDP_CG,
                                     track_best=track_best)


def solve_batch_limited(instances, seeds, hp: HyperParams, nthreads, alt_limit=1,
                        backend=MFZ_BN, mode=LITERAL):
    """Bounded multi-threaded CPU sample (run_jobs model). Returns (wall_s, R, sigma)."""
    n = len(instances)
    N = instances[0].N
    As = [np.asfortranarray(i.A, np.float64) for i in instances]
    ys = [np.ascontiguousarray(i.y, np.float64) for i in instances]
    Ms = np.array([i.M for i in instances], np.int32)
    Ap = (C.c_void_p * n)(*[a.ctypes.data for a in As])
    yp = (C.c_void_p * n)(*[a.ctypes.data for a in ys])
    sd = np.ascontiguousarray(seeds, np.uint64)
    R = np.zeros((n, N))
    S = np.zeros((n, N), np.int32)
    h = hp.to_c()
    wall = lib().orc_solve_batch_limited(n, nthreads, alt_limit, N, _p(Ms), Ap, yp, mode,
                                         backend, C.byref(h), _p(sd), _p(R), _p(S))
    return wall, R, S


def solve_batch(instances, seeds, hp: HyperParams, nthreads, backend=MFZ_BN, mode=CANON,
                nseg=8, gran=8, cdp=CDP_JACOBI):
    """Full multi-threaded batch of trials. Returns (wall_s, R, sigma, fail_alt)."""
    n = len(instances)
    N = instances[0].N
    As = [np.asfortranarray(i.A, np.float64) for i in instances]
    ys = [np.ascontiguousarray(i.y, np.float64) for i in instances]
    xs = [np.ascontiguousarray(i.x_true, np.float64) for i in instances]
    xis = [np.ascontiguousarray(i.xi_true, np.int32) for i in instances]
    Ms = np.array([i.M for i in instances], np.int32)
    P = lambda arrs: (C.c_void_p * n)(*[a.ctypes.data for a in arrs])  # noqa: E731
    sd = np.ascontiguousarray(seeds, np.uint64)
    R = np.zeros((n, N))
    S = np.zeros((n, N), np.int32)
    FA = np.zeros(n, np.int32)
    h = hp.to_c()
    wall = lib().orc_solve_batch(n, nthreads, N, _p(Ms), P(As), P(ys), P(xs), P(xis), mode,
                                 nseg, gran, backend, C.byref(h), _p(sd), cdp, _p(R), _p(S),
                                 _p(FA))
    return wall, R, S, FA
