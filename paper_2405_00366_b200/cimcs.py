"""Python host mirror of the reference's ``cimcs`` module, on the B200 path.

Same names, argument meaning and error behaviour as the reference's pybind
module (bindings/module.cpp:57-160, python/cimcs/__init__.py):

    inst = gen_instance(N, alpha, a, nu, seed)
    res  = solve(inst, backend="mfz-bn", params=HyperParams(), seed=1,
                 cdp="jacobi", track_best=False)

``solve`` runs ONE trial (one instance, one replica) through the CUDA path.
``solve_batch`` and :class:`Context` expose the batched multi-instance /
multi-replica driver (B instances x R replicas per call) that replaces the
reference's ``run_jobs`` thread pool (tools/main.cpp:305-321).

Every compute call goes through libcimcs_gpu.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, fields
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import load

BACKENDS = {"mfz-cn": _lib.MFZ_CN, "mfz-bn": _lib.MFZ_BN, "pp": _lib.PP}
DTYPES = {"f32": _lib.F32, "fp32": _lib.F32, "float32": _lib.F32,
          "f64": _lib.F64, "fp64": _lib.F64, "float64": _lib.F64}


# ---------------------------------------------------------------- errors
class ConfigError(RuntimeError):
    """types.hpp:22-26 config_error."""


class InputError(ValueError):
    """types.hpp:16-20 input_error."""


class DivergenceError(RuntimeError):
    """types.hpp:28-33 divergence_error (offending_index = first bad spin)."""

    def __init__(self, msg, offending_index=-1):
        super().__init__(msg)
        self.offending_index = offending_index


class CudaError(RuntimeError):
    pass


def _check(rc: int):
    if rc == _lib.OK:
        return
    msg = _lib.last_error()
    if rc == _lib.INPUT_ERROR:
        raise InputError(msg)
    if rc == _lib.CONFIG_ERROR:
        raise ConfigError(msg)
    if rc == _lib.DIVERGENCE:
        raise DivergenceError(msg)
    raise CudaError(msg)


# ------------------------------------------------------------ parameters
@dataclass
class HyperParams:
    """HyperParams, types.hpp:77-96, plus the BASELINE pump extension."""
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
    pump_kind: int = _lib.PUMP_SIGMOID
    pump_end: float = 1.2

    def to_c(self) -> _lib.Hyper:
        h = _lib.Hyper()
        for f in fields(self):
            setattr(h, f.name, type(getattr(h, f.name))(getattr(self, f.name)))
        return h

    def validate(self):
        h = self.to_c()
        _check(load().cimcs_hyper_validate(C.byref(h)))


def baseline_params(velo: int = 19, n_steps: int = 1000, **kw) -> HyperParams:
    """BASELINE.json configs 0-2: dt 0.01, linear pump 0 -> 1.2, 20 outer iterations."""
    return HyperParams(dt=0.01, n_steps=n_steps, velo=velo, pump_kind=_lib.PUMP_LINEAR,
                       pump_end=1.2, **kw)


def pump_schedule(t: float, p_thr: float, d: float) -> float:
    """orchestrator.cpp:12-14 (host scalar; the GPU path reads a host-built table)."""
    return (p_thr - d) + 2.0 * d / (1.0 + math.exp(-(t - 4.0) / 2.0))


def eta_schedule(i: int, eta_init: float, eta_end: float, velo: int) -> float:
    """orchestrator.cpp:16-20."""
    if velo < 1:
        raise ConfigError("eta_schedule: velo must be >= 1")
    linear = eta_init * (1.0 - float(i) / velo)
    return eta_end if linear < eta_end else linear


def nccl_unique_id() -> bytes:
    """128-byte NCCL id for cimcs_create_sharded (broadcast it to all ranks)."""
    buf = (C.c_uint8 * 128)()
    _check(load().cimcs_nccl_unique_id(buf, 128))
    return bytes(buf)


def mix_seed(base: int, salt: int) -> int:
    return load().cimcs_mix_seed(base, salt)


def gemv_order(dtype="f64"):
    ns, gr = C.c_int32(), C.c_int32()
    load().cimcs_gemv_order(DTYPES[dtype], C.byref(ns), C.byref(gr))
    return ns.value, gr.value


# ------------------------------------------------------------- instances
@dataclass
class Instance:
    """ProblemInstance, types.hpp:41-54 (A is M x N, column-major)."""
    A: np.ndarray
    y: np.ndarray
    x_true: np.ndarray | None = None
    xi_true: np.ndarray | None = None
    a: float = 0.0
    alpha: float = 0.0
    nu: float = 0.0
    seed: int = 0

    @property
    def N(self) -> int:
        return int(self.A.shape[1])

    @property
    def M(self) -> int:
        return int(self.A.shape[0])

    def has_truth(self) -> bool:
        return self.x_true is not None and self.xi_true is not None


def gen_dims(N, alpha, a):
    M, K = C.c_int32(), C.c_int32()
    _check(load().cimcs_gen_dims(N, alpha, a, C.byref(M), C.byref(K)))
    return M.value, K.value


def gen_instance(N: int, alpha: float, a: float, nu: float, seed: int) -> Instance:
    """gen_instance, datagen.cpp:15-55 (host, same stream and draw order)."""
    if nu < 0:
        raise InputError("gen_instance: need nu >= 0")
    M, _ = gen_dims(N, alpha, a)
    A = np.zeros((M, N), order="F")
    y = np.zeros(M)
    x = np.zeros(N)
    xi = np.zeros(N, np.int32)
    _check(load().cimcs_gen_instance(N, alpha, a, nu, seed, A.ctypes.data, y.ctypes.data,
                                     x.ctypes.data, xi.ctypes.data))
    return Instance(A, y, x, xi, a, alpha, nu, seed)


def gen_instances(N, params: Sequence[tuple], threads: int = 0) -> list[Instance]:
    """Many instances on host threads; params = [(alpha, a, nu, seed), ...]."""
    B = len(params)
    al = np.array([p[0] for p in params], np.float64)
    aa = np.array([p[1] for p in params], np.float64)
    nu = np.array([p[2] for p in params], np.float64)
    sd = np.array([p[3] for p in params], np.uint64)
    out = []
    for p in params:
        M, _ = gen_dims(N, p[0], p[1])
        out.append(Instance(np.zeros((M, N), order="F"), np.zeros(M), np.zeros(N),
                            np.zeros(N, np.int32), p[1], p[0], p[2], int(p[3])))
    P = lambda xs: (C.c_void_p * B)(*[x.ctypes.data for x in xs])  # noqa: E731
    _check(load().cimcs_gen_instances(
        B, N, al.ctypes.data, aa.ctypes.data, nu.ctypes.data, sd.ctypes.data,
        P([o.A for o in out]), P([o.y for o in out]), P([o.x_true for o in out]),
        P([o.xi_true for o in out]), threads))
    return out


# --------------------------------------------------------------- context
def _traj(a, B, R, N, dtype=np.float64):
    a = np.ascontiguousarray(a, dtype=dtype)
    if a.size != B * R * N:
        raise InputError(f"expected {B}x{R}x{N} values, got shape {a.shape}")
    return a.reshape(B, R, N)


class Context:
    """One device context: B problems of equal N, device-resident coupling."""

    def __init__(self, device: int = 0, dtype: str = "f32", shard=None):
        """shard = (world, rank, nccl_id_bytes) for a row-sharded context."""
        self._lib = load()
        self.dtype = dtype
        self._ctx = C.c_void_p()
        if shard is None:
            _check(self._lib.cimcs_create(device, DTYPES[dtype], C.byref(self._ctx)))
        else:
            world, rank, nid = shard
            buf = (C.c_uint8 * 128).from_buffer_copy(bytes(nid))
            _check(self._lib.cimcs_create_sharded(device, DTYPES[dtype], world, rank, buf,
                                                  C.byref(self._ctx)))
        self.B = self.N = 0
        self._keep = None

    def close(self):
        if self._ctx:
            self._lib.cimcs_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key: str, value: int):
        _check(self._lib.cimcs_set_option(self._ctx, key.encode(), int(value)))

    def set_problems(self, instances: Sequence[Instance]):
        B = len(instances)
        if B < 1:
            raise InputError("no instances")
        N = instances[0].N
        if any(inst.N != N for inst in instances):
            raise InputError("all instances of a context must share N")
        As = [np.asfortranarray(i.A, np.float64) for i in instances]
        ys = [np.ascontiguousarray(i.y, np.float64) for i in instances]
        truth = all(getattr(i, "x_true", None) is not None and
                    getattr(i, "xi_true", None) is not None for i in instances)
        xs = [np.ascontiguousarray(i.x_true, np.float64) for i in instances] if truth else None
        xis = [np.ascontiguousarray(i.xi_true, np.int32) for i in instances] if truth else None
        Ms = np.array([i.M for i in instances], np.int32)
        P = lambda arrs: (C.c_void_p * B)(*[a.ctypes.data for a in arrs])  # noqa: E731
        _check(self._lib.cimcs_set_problems(
            self._ctx, B, N, Ms.ctypes.data, P(As), P(ys), P(xs) if truth else None,
            P(xis) if truth else None))
        self.B, self.N = B, N

    def set_mri_problem(self, target_image, mask, gamma: float, x_true=None):
        """MriTransform(target_image, mask, gamma) + make_problem(t, &truth)
        (mri.hpp:46-99, mri.cpp:393-411): the matrix-free transform-chain
        problem (one instance, fp32 contexts)."""
        img = np.ascontiguousarray(target_image, np.float64)
        H, W = img.shape
        m = np.ascontiguousarray(mask, np.int32)
        x = None if x_true is None else np.ascontiguousarray(x_true, np.float64).reshape(-1)
        if x is not None and x.size != H * W:
            raise InputError("make_problem: truth length mismatch")
        _check(self._lib.cimcs_set_mri_problem(self._ctx, H, W, img.ctypes.data, m.size,
                                               m.ctypes.data, float(gamma),
                                               None if x is None else x.ctypes.data))
        self.B, self.N = 1, H * W

    def set_dct_problem(self, n: int, levels: int, freqs, y, x_true=None):
        """BASELINE config 3 as the matrix-free DCT o Haar^-1 chain (one instance,
        fp32 contexts): the dense instance's A = S C2 Psi_levels^-1 with rows in
        the order of `freqs` (u * n + v) and observations `y`."""
        f = np.ascontiguousarray(freqs, np.int32).reshape(-1)
        yy = np.ascontiguousarray(y, np.float64).reshape(-1)
        if yy.size != f.size:
            raise InputError("dct problem: one observation per frequency")
        x = None if x_true is None else np.ascontiguousarray(x_true, np.float64).reshape(-1)
        if x is not None and x.size != n * n:
            raise InputError("dct problem: truth length mismatch")
        _check(self._lib.cimcs_set_dct_problem(self._ctx, int(n), int(levels), f.size,
                                               f.ctypes.data, yy.ctypes.data,
                                               None if x is None else x.ctypes.data))
        self.B, self.N = 1, n * n

    def mri_lasso(self, lambda_l1: float = 3e-4, max_iters: int = 5000, tol: float = 1e-8,
                  step: float = 1.0):
        """lasso_init(t, lambda) (mri.cpp:372-377): FISTA warm start of the
        built MRI problem -> (x, iterations, objective)."""
        x = np.zeros(self.N)
        it, f = C.c_int32(), C.c_double()
        _check(self._lib.cimcs_mri_lasso(self._ctx, float(lambda_l1), int(max_iters), float(tol),
                                         float(step), x.ctypes.data, C.byref(it), C.byref(f)))
        return x, it.value, f.value

    def set_generated_problems(self, N: int, params: Sequence[tuple]):
        """Instances generated ON THE GPU from counter-based Philox streams
        (gen_instance's recipe, NOT the reference's mt19937_64 stream: a documented
        deviation for config-4-scale runs); params = [(alpha, a, nu, seed), ...]."""
        B = len(params)
        al = np.array([p[0] for p in params], np.float64)
        aa = np.array([p[1] for p in params], np.float64)
        nu = np.array([p[2] for p in params], np.float64)
        sd = np.array([p[3] for p in params], np.uint64)
        _check(self._lib.cimcs_set_generated_problems(self._ctx, B, N, al.ctypes.data,
                                                      aa.ctypes.data, nu.ctypes.data,
                                                      sd.ctypes.data))
        self.B, self.N = B, N
        self._gen_params = [tuple(p) for p in params]

    def get_instance(self, b: int) -> Instance:
        """The resident instance b (e.g. a generated one) back on the host."""
        al, a, nu, seed = self._gen_params[b] if hasattr(self, "_gen_params") else (0, 0, 0, 0)
        M, _ = gen_dims(self.N, al, a) if al else (None, None)
        if M is None:
            raise InputError("get_instance: only for generated problem sets")
        A = np.zeros((M, self.N), order="F")
        y = np.zeros(M)
        x = np.zeros(self.N)
        xi = np.zeros(self.N, np.int32)
        _check(self._lib.cimcs_get_instance(self._ctx, b, A.ctypes.data, y.ctypes.data,
                                            x.ctypes.data, xi.ctypes.data))
        return Instance(A, y, x, xi, a, al, nu, int(seed))

    def canon_order(self):
        """(nseg, gran) of the fp64 contraction order of the resident problems
        (the oracle's ORC_CANON parameters, cimcs_canon_order)."""
        ns, gr = C.c_int32(), C.c_int32()
        _check(self._lib.cimcs_canon_order(self._ctx, C.byref(ns), C.byref(gr)))
        return ns.value, gr.value

    def build_coupling(self):
        _check(self._lib.cimcs_build_coupling(self._ctx))

    def get_coupling(self, b: int, gram: bool = True):
        G = np.zeros((self.N, self.N)) if gram else None
        hz = np.zeros(self.N)
        D = np.zeros(self.N)
        _check(self._lib.cimcs_get_coupling(self._ctx, b, None if G is None else G.ctypes.data,
                                            hz.ctypes.data, D.ctypes.data))
        return G, hz, D

    def _need(self, R: int):
        """The reference raises input_error for an empty problem / replica set (types.hpp:16-33);
        checked here before any host array is shaped."""
        if getattr(self, "B", 0) < 1:
            raise InputError("no problems set (set_problems / set_mri_problem first)")
        if not 1 <= int(R) <= 16:
            raise InputError("R must be in [1, 16]")

    def mfz_step(self, R: int, backend: str, hp: HyperParams, eta: float, p: float, Rsig, c, e):
        self._need(R)
        B, N = self.B, self.N
        Rs, cc, ee = (_traj(x, B, R, N) for x in (Rsig, c, e))
        co, eo, ho = (np.zeros((B, R, N)) for _ in range(3))
        fi = np.zeros((B, R), np.int32)
        h = hp.to_c()
        rc = self._lib.cimcs_mfz_step(self._ctx, R, BACKENDS[backend], C.byref(h), eta, p,
                                      Rs.ctypes.data, cc.ctypes.data, ee.ctypes.data,
                                      co.ctypes.data, eo.ctypes.data, ho.ctypes.data,
                                      fi.ctypes.data)
        if rc not in (_lib.OK, _lib.DIVERGENCE):
            _check(rc)
        return dict(c=co, e=eo, h=ho, fail_index=fi)

    def run_cim(self, R: int, backend: str, hp: HyperParams, eta: float, Rsig, c0):
        self._need(R)
        B, N = self.B, self.N
        Rs, c0 = _traj(Rsig, B, R, N), _traj(c0, B, R, N)
        co, eo = np.zeros((B, R, N)), np.zeros((B, R, N))
        so = np.zeros((B, R, N), np.int32)
        me = np.zeros((B, R))
        fi = np.zeros((B, R), np.int32)
        h = hp.to_c()
        rc = self._lib.cimcs_run_cim(self._ctx, R, BACKENDS[backend], C.byref(h), eta,
                                     Rs.ctypes.data, c0.ctypes.data, co.ctypes.data,
                                     eo.ctypes.data, so.ctypes.data, me.ctypes.data,
                                     fi.ctypes.data)
        if rc not in (_lib.OK, _lib.DIVERGENCE):
            _check(rc)
        return dict(c=co, e=eo, sigma=so, min_e=me, fail_index=fi)

    def run_pp(self, R: int, hp: HyperParams, eta: float, Rsig, seeds):
        """run_pp (solver_pp.cpp:100-132) for every trajectory from its stream seed."""
        self._need(R)
        B, N = self.B, self.N
        Rs = _traj(Rsig, B, R, N)
        sd = np.ascontiguousarray(seeds, np.uint64).reshape(B * R)
        mu, e, mt = (np.zeros((B, R, N)) for _ in range(3))
        so = np.zeros((B, R, N), np.int32)
        me = np.zeros((B, R))
        fi = np.zeros((B, R), np.int32)
        h = hp.to_c()
        rc = self._lib.cimcs_run_pp(self._ctx, R, C.byref(h), eta, Rs.ctypes.data, sd.ctypes.data,
                                    mu.ctypes.data, e.ctypes.data, mt.ctypes.data, so.ctypes.data,
                                    me.ctypes.data, fi.ctypes.data)
        if rc not in (_lib.OK, _lib.DIVERGENCE):
            _check(rc)
        return dict(mu=mu, e=e, mu_tilde=mt, sigma=so, min_e=me, fail_index=fi)

    def refit(self, R: int, sigma, R_prev, hp: HyperParams | None = None,
              cdp: str = "jacobi", return_iterations: bool = False):
        """cdp_minimize (cdp.cpp:132-139) of every trajectory on its support:
        the damped Jacobi refit or (cdp="cg") conjugate gradient."""
        if cdp not in ("jacobi", "cg"):
            raise ConfigError("cdp must be 'jacobi' or 'cg'")
        hp = hp or HyperParams()
        self._need(R)
        B, N = self.B, self.N
        s = _traj(sigma, B, R, N, np.int32)
        rp = _traj(R_prev, B, R, N)
        out = np.zeros((B, R, N))
        its = np.zeros((B, R), np.int32)
        h = hp.to_c()
        method = _lib.CDP_JACOBI if cdp == "jacobi" else _lib.CDP_CG
        _check(self._lib.cimcs_cdp_minimize(self._ctx, R, s.ctypes.data, rp.ctypes.data, method,
                                            C.byref(h), out.ctypes.data, its.ctypes.data))
        return (out, its) if return_iterations else out

    def score(self, R: int, Rsig, sigma, lam: float):
        self._need(R)
        B, N = self.B, self.N
        rs = _traj(Rsig, B, R, N)
        s = _traj(sigma, B, R, N, np.int32)
        obj, rm, hm = np.zeros((B, R)), np.zeros((B, R)), np.zeros((B, R))
        _check(self._lib.cimcs_score(self._ctx, R, rs.ctypes.data, s.ctypes.data, lam,
                                     obj.ctypes.data, rm.ctypes.data, hm.ctypes.data))
        return dict(objective=obj, rmse=rm, hamming=hm)

    def solve(self, R: int, backend: str, hp: HyperParams, seeds, R_init=None,
              track_best: bool = False, cdp: str = "jacobi") -> dict:
        if backend not in BACKENDS:
            raise ConfigError(f"unknown backend '{backend}' (use mfz-bn, mfz-cn or pp)")
        if cdp not in ("jacobi", "cg"):
            raise ConfigError("cdp must be 'jacobi' or 'cg'")
        self._need(R)
        B, N = self.B, self.N
        sd = np.ascontiguousarray(seeds, np.uint64).reshape(B * R)
        ri = None if R_init is None else _traj(R_init, B, R, N)
        nalt = hp.velo + 1
        Ro = np.zeros((B, R, N))
        So = np.zeros((B, R, N), np.int32)
        hist = (_lib.Record * (nalt * B * R))()
        nh = np.zeros((B, R), np.int32)
        fa = np.zeros((B, R), np.int32)
        fi = np.zeros((B, R), np.int32)
        h = hp.to_c()
        _check(self._lib.cimcs_solve(
            self._ctx, R, BACKENDS[backend], C.byref(h),
            _lib.CDP_JACOBI if cdp == "jacobi" else _lib.CDP_CG, sd.ctypes.data,
            None if ri is None else ri.ctypes.data, int(track_best), Ro.ctypes.data,
            So.ctypes.data, hist, nh.ctypes.data, fa.ctypes.data, fi.ctypes.data))
        H = np.ctypeslib.as_array(hist).view(np.dtype([
            ("i", np.int32), ("support", np.int32), ("eta", np.float64),
            ("hamiltonian", np.float64), ("rmse", np.float64), ("hamming", np.float64),
            ("min_e", np.float64), ("median_e", np.float64)])).reshape(B, R, nalt).copy()
        return dict(R=Ro, sigma=So, history=H, n_hist=nh, fail_alt=fa, fail_index=fi,
                    backend=backend)

    def timeline(self) -> np.ndarray:
        """%globaltimer stamps [CTA][4] of the last tile / update launch pair (option
        "timeline" = 1; rows 0..255 tile CTAs, rows 256..8191 update CTAs b * gridDim.x + x,
        rows 8192.. tile CTA 0's per-tile stamps)."""
        out = np.zeros((8192 + 256, 4), np.uint64)
        n = C.c_int64(0)
        _check(self._lib.cimcs_get_timeline(self._ctx, out.ctypes.data, out.size, C.byref(n)))
        return out

    def timing(self) -> dict:
        t = _lib.Timing()
        _check(self._lib.cimcs_get_timing(self._ctx, C.byref(t)))
        return {f: getattr(t, f) for f, _ in _lib.Timing._fields_}


# ------------------------------------------------------------ public API
def trial_dict(res, b, r, n_steps):
    nh = int(res["n_hist"][b, r])
    H = res["history"][b, r, :nh]
    hist = [dict(i=int(h["i"]), eta=float(h["eta"]), hamiltonian=float(h["hamiltonian"]),
                 rmse=float(h["rmse"]), hamming=float(h["hamming"]), seconds=math.nan,
                 min_e=float(h["min_e"]), median_e=float(h["median_e"]),
                 support=int(h["support"])) for h in H]
    failed = int(res["fail_alt"][b, r]) >= 0
    out = dict(R=res["R"][b, r].copy(), sigma=res["sigma"][b, r].copy(), failed=failed,
               fail_reason=((f"pp: divergence at spin {int(res['fail_index'][b, r])}"
                             if res.get("backend") == "pp" else
                             f"mfz_step: non-finite amplitude at spin {int(res['fail_index'][b, r])}")
                            if failed else ""),
               fail_alternation=int(res["fail_alt"][b, r]), history=hist)
    out["min_hamiltonian"] = min((h["hamiltonian"] for h in hist), default=math.nan)
    out["final_rmse"] = hist[-1]["rmse"] if hist else math.nan
    out["final_hamming"] = hist[-1]["hamming"] if hist else math.nan
    return out


def solve(instance: Instance, backend: str = "mfz-bn", params: HyperParams | None = None,
          seed: int = 1, cdp: str = "jacobi", track_best: bool = False, dtype: str = "f64",
          device: int = 0) -> dict:
    """cimcs.solve (bindings/module.cpp:127-141) on the B200 path: one trial."""
    params = params or HyperParams()
    if backend not in BACKENDS:
        raise ConfigError(f"unknown backend '{backend}' (use mfz-bn, mfz-cn or pp)")
    if cdp not in ("jacobi", "cg"):
        raise ConfigError("cdp must be 'jacobi' or 'cg'")
    params.validate()
    with Context(device, dtype) as ctx:
        ctx.set_problems([instance])
        ctx.build_coupling()
        res = ctx.solve(1, backend, params, [seed], track_best=track_best, cdp=cdp)
    return trial_dict(res, 0, 0, params.n_steps)


def replica_seeds(instances: Sequence[Instance], R: int, backend: str) -> np.ndarray:
    """⊕ replica rho of instance s uses mix_seed(s, backend + 3 rho); rho = 0 is the
    reference's cmd_run stream (tools/main.cpp:423)."""
    be = BACKENDS[backend]
    return np.array([[mix_seed(inst.seed, be + 3 * r) for r in range(R)] for inst in instances],
                    np.uint64)


def solve_batch(instances: Sequence[Instance], R: int = 1, backend: str = "mfz-bn",
                params: HyperParams | None = None, seeds=None, dtype: str = "f32",
                device: int = 0, track_best: bool = False) -> dict:
    """Batched multi-instance / multi-replica driver (replaces run_jobs)."""
    params = params or HyperParams()
    params.validate()
    if seeds is None:
        seeds = replica_seeds(instances, R, backend)
    with Context(device, dtype) as ctx:
        ctx.set_problems(instances)
        ctx.build_coupling()
        res = ctx.solve(R, backend, params, seeds, track_best=track_best)
        res["timing"] = ctx.timing()
    return res
