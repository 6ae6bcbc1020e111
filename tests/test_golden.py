"""Committed golden fixtures (tests/golden/make_golden.py) -- no /root/reference
needed at run time.

* ref_rng / ref_instances: produced by the reference's own rng.hpp and
  datagen.cpp; the oracle and the product's host generator must match them
  bit for bit.
* oracle_config0: the oracle's fp64 solve of BASELINE config 0; the oracle must
  keep reproducing it (CPU) and the GPU fp64 path must match it (GPU test).
"""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    return np.load(os.path.join(GOLD, name))


def test_oracle_rng_matches_reference_golden(O):
    z = _load("ref_rng.npz")
    for s in z["seeds"]:
        s = int(s)
        r = O.Rng(s)
        assert [r.raw() for _ in range(1000)] == [int(v) for v in z[f"raw_{s}"]]
        r = O.Rng(s)
        assert np.array_equal(np.array([r.gauss() for _ in range(1000)]), z[f"gauss_{s}"])


@pytest.mark.parametrize("gen", ["oracle", "product"])
def test_instances_match_reference_golden(O, gen):
    z = _load("ref_instances.npz")
    for k in range(int(z["n"])):
        N, al, a, nu, s = z[f"args_{k}"]
        args = (int(N), float(al), float(a), float(nu), int(s))
        if gen == "oracle":
            inst = O.gen_instance(*args)
        else:
            from paper_2405_00366_b200 import cimcs as P
            inst = P.gen_instance(*args)
        assert np.array_equal(inst.A, z[f"A_{k}"])
        assert np.array_equal(inst.y, z[f"y_{k}"])
        assert np.array_equal(inst.x_true, z[f"x_{k}"])
        assert np.array_equal(inst.xi_true, z[f"xi_{k}"])


@pytest.mark.slow
def test_oracle_config0_reproduces_golden(O):
    z = _load("oracle_config0.npz")
    inst = O.gen_instance(500, 0.6, 0.2, 0.01, 0)
    res = O.Problem(inst, O.CANON).alternating_minimize(O.MFZ_BN, O.baseline_params(),
                                                         O.Rng(int(z["seed"][0])))
    assert np.array_equal(res["R"], z["canon_R"])
    assert np.array_equal(res["sigma"], z["canon_sigma"])
    assert np.array_equal(np.array([h["hamiltonian"] for h in res["history"]]),
                          z["canon_hamiltonian"])


def test_golden_literal_and_canon_agree():
    """The reference-literal (A^T(A w)) and canonical orders give the same
    config-0 supports and RMSE to rounding."""
    z = _load("oracle_config0.npz")
    assert np.array_equal(z["canon_sigma"], z["literal_sigma"])
    assert np.allclose(z["canon_rmse"], z["literal_rmse"], rtol=1e-12, atol=0)
    assert np.array_equal(z["canon_support"], z["literal_support"])


@pytest.mark.gpu
def test_gpu_config0_matches_golden(gpu):
    """GPU fp64 solve of config 0 (through the C ABI) == committed oracle golden."""
    z = _load("oracle_config0.npz")
    inst = gpu.gen_instance(500, 0.6, 0.2, 0.01, 0)
    with gpu.Context(0, "f64") as ctx:
        ctx.set_problems([inst])
        ctx.build_coupling()
        res = ctx.solve(1, "mfz-bn", gpu.baseline_params(), [int(z["seed"][0])])
    assert np.array_equal(res["R"][0, 0], z["canon_R"])
    assert np.array_equal(res["sigma"][0, 0], z["canon_sigma"])
    assert np.array_equal(res["history"][0, 0]["support"], z["canon_support"])
    assert np.array_equal(res["history"][0, 0]["median_e"], z["canon_median_e"])
    assert np.allclose(res["history"][0, 0]["hamiltonian"], z["canon_hamiltonian"], rtol=1e-12)
