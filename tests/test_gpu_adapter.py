"""The reference-side adapter (integration/gpu_adapter.cpp), compiled against the
reference's real headers into oracle/_ref/libref_adapter.so, on the GPU:

* its alternating_minimize_gpu (the reference's own signature, orchestrator.hpp:139-141,
  over the C ABI) returns bitwise what the product's Python API returns and what
  the oracle's canonical order predicts;
* against the reference's OWN CPU solver (oracle/_ref/libref_solver.so, the
  reference's alternating_minimize compiled from /root/reference) on the same
  instance and seed -- north_star's fp64 bar: identical supports, RMSE within 1e-6
  relative.  Runs use the reference's own schedule (sigmoid pump, dt 0.02),
  shortened.
"""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import ref_solver as RS

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "oracle", "_ref", "libref_adapter.so")


@pytest.fixture(scope="module")
def adapter(gpu, O):
    if not os.path.exists(SO):
        pytest.skip("oracle/_ref/libref_adapter.so not built (needs /root/reference)")
    L = C.CDLL(SO)
    vp, i = C.c_void_p, C.c_int
    L.adapter_alternating_minimize_gpu.argtypes = [i, i, vp, vp, vp, vp, i,
                                                   C.POINTER(O._Hyper), C.c_uint64, i, i, i,
                                                   vp, vp, vp, vp, vp]
    return L


def _run(L, O, inst, backend, hp, seed, dtype=1):
    A = np.asfortranarray(inst.A)
    y = np.ascontiguousarray(inst.y)
    x = np.ascontiguousarray(inst.x_true)
    xi = np.ascontiguousarray(inst.xi_true, np.int32)
    M, N = A.shape
    R = np.zeros(N)
    s = np.zeros(N, np.int32)
    hist = np.zeros((hp.velo + 1, 7))
    nh, fa = C.c_int(), C.c_int()
    h = hp.to_c()
    rc = L.adapter_alternating_minimize_gpu(N, M, A.ctypes.data, y.ctypes.data, x.ctypes.data,
                                            xi.ctypes.data, backend, C.byref(h), seed, 0, 0,
                                            dtype, R.ctypes.data, s.ctypes.data,
                                            hist.ctypes.data, C.byref(nh), C.byref(fa))
    assert rc == 0
    return R, s, hist[: nh.value], fa.value


@pytest.mark.parametrize("N,velo", [(500, 5), (2000, 1)])
def test_adapter_vs_product_oracle_and_reference(adapter, gpu, O, N, velo):
    inst = (O.gen_instance(500, 0.6, 0.2, 0.01, 0) if N == 500
            else O.gen_instance(2000, 0.5, 0.1, 0.01, 1))
    hp = O.HyperParams(velo=velo)  # the reference's own schedule (types.hpp:77-96)
    seed = O.mix_seed(inst.seed, 1)
    R, s, hist, fa = _run(adapter, O, inst, O.MFZ_BN, hp, seed)
    assert fa == -1 and len(hist) == velo + 1
    # the product's own API: same bits
    pres = gpu.solve(inst, "mfz-bn", gpu.HyperParams(velo=velo), seed=seed)
    assert np.array_equal(R, pres["R"]) and np.array_equal(s, pres["sigma"])
    # the oracle in the GPU's canonical order: same bits
    with gpu.Context(0, "f64") as ctx:
        ctx.set_problems([inst])
        order = ctx.canon_order()
    ref = O.Problem(inst, O.CANON, *order).alternating_minimize(O.MFZ_BN, hp, O.Rng(seed))
    assert np.array_equal(R, ref["R"]) and np.array_equal(s, ref["sigma"])
    # the reference's own solver (compiled from /root/reference): north_star's bar
    if RS.available():
        rr = RS.alternating_minimize(inst, O.MFZ_BN, hp, seed)
        assert np.array_equal(s, rr["sigma"])
        rm_g = O.rmse(R, s, inst.x_true, inst.xi_true)
        rm_r = O.rmse(rr["R"], rr["sigma"], inst.x_true, inst.xi_true)
        assert abs(rm_g - rm_r) <= 1e-6 * rm_r
