"""The oracle's LITERAL restatement against the reference's OWN solver.

oracle/Makefile.ref compiles the reference's model.cpp, solver_mfz.cpp,
solver_pp.cpp, cdp.cpp and orchestrator.cpp unmodified from /root/reference
against a sequential Eigen shim (oracle/refshim/Eigen/Dense; Eigen3 is absent
here).  With the shim's fixed reduction order the reference's own
alternating_minimize / run_cim / cdp_minimize / objective_at must equal the
oracle's LITERAL mode BIT FOR BIT: this pins the restated control flow,
elementwise arithmetic, schedules, RNG consumption and refit of
oracle/oracle.c to the reference code itself (Eigen's own SIMD reduction order
remains unpinnable).  The reference has only its sigmoid
pump, so these runs use its own schedule (types.hpp:77-96).  CPU only.
"""
import numpy as np
import pytest

from oracle import ref_solver as RS

pytestmark = pytest.mark.skipif(not RS.available(), reason="oracle/_ref/libref_solver.so absent")


def _same_history(ref, orc):
    assert len(ref["history"]) == len(orc["history"])
    for h, o in zip(ref["history"], orc["history"]):
        assert int(h[0]) == o["i"]
        assert h[1] == o["eta"]
        assert h[2] == o["hamiltonian"]
        assert h[3] == o["rmse"] or (np.isnan(h[3]) and np.isnan(o["rmse"]))
        assert h[4] == o["hamming"] or (np.isnan(h[4]) and np.isnan(o["hamming"]))
        assert h[5] == o["min_e"]
        assert h[6] == o["median_e"]


@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn", "pp"])
@pytest.mark.parametrize("cdp", ["jacobi", "cg"])
def test_alternating_minimize_bitwise(O, backend, cdp):
    """alternating_minimize (orchestrator.cpp:170-235) at BASELINE config 0's instance,
    the reference's own schedule shortened to 4 alternations."""
    inst = O.gen_instance(500, 0.6, 0.2, 0.01, 0)
    hp = O.HyperParams(velo=3)
    be = O.BACKENDS[backend]
    cd = O.CDP_JACOBI if cdp == "jacobi" else O.CDP_CG
    seed = O.mix_seed(0, be)
    ref = RS.alternating_minimize(inst, be, hp, seed, cdp=cd)
    orc = O.Problem(inst, O.LITERAL).alternating_minimize(be, hp, O.Rng(seed), cdp=cd)
    assert np.array_equal(ref["R"], orc["R"])
    assert np.array_equal(ref["sigma"], orc["sigma"])
    assert ref["failed"] == orc["failed"]
    _same_history(ref, orc)


def test_track_best_and_r_init(O):
    inst = O.gen_instance(300, 0.5, 0.1, 0.01, 3)
    hp = O.HyperParams(velo=4, n_steps=300)
    r0 = np.random.default_rng(0).normal(size=300)
    ref = RS.alternating_minimize(inst, O.MFZ_BN, hp, 77, R_init=r0, track_best=True)
    orc = O.Problem(inst, O.LITERAL).alternating_minimize(O.MFZ_BN, hp, O.Rng(77), R_init=r0,
                                                          track_best=True)
    assert np.array_equal(ref["R"], orc["R"])
    assert np.array_equal(ref["sigma"], orc["sigma"])
    _same_history(ref, orc)


def test_config1_shape_bitwise(O):
    """BASELINE config-1 shape (N=2000, M=1000): one alternation of 200 steps."""
    inst = O.gen_instance(2000, 0.5, 0.1, 0.01, 1)
    hp = O.HyperParams(velo=1, n_steps=200)
    seed = O.mix_seed(1, 1)
    ref = RS.alternating_minimize(inst, O.MFZ_BN, hp, seed)
    orc = O.Problem(inst, O.LITERAL).alternating_minimize(O.MFZ_BN, hp, O.Rng(seed))
    assert np.array_equal(ref["R"], orc["R"])
    assert np.array_equal(ref["sigma"], orc["sigma"])
    _same_history(ref, orc)


def test_divergence_matches(O):
    """divergence_error -> failed at the same alternation with the same message
    (solver_mfz.cpp:75-85, orchestrator.cpp:222-227)."""
    inst = O.gen_instance(200, 0.6, 0.2, 0.01, 5)
    hp = O.HyperParams(velo=2, dt=5.0, n_steps=50)
    ref = RS.alternating_minimize(inst, O.MFZ_BN, hp, 9)
    orc = O.Problem(inst, O.LITERAL).alternating_minimize(O.MFZ_BN, hp, O.Rng(9))
    assert ref["failed"] and orc["failed"]
    assert ref["fail_alternation"] == orc["fail_alternation"]
    assert ref["fail_reason"] == orc["fail_reason"]


@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn", "pp"])
def test_run_cim_bitwise(O, backend):
    inst = O.gen_instance(400, 0.5, 0.15, 0.01, 11)
    hp = O.HyperParams(n_steps=400)
    be = O.BACKENDS[backend]
    p = O.Problem(inst, O.LITERAL)
    R = p.hz.copy()
    ref = RS.run_cim(inst, be, hp, 0.6, 21, R)
    if be == O.PP:
        orc = p.run_pp(R, hp, 0.6, O.Rng(21))
        amp = orc["mu_tilde"]
    else:
        orc = p.run_mfz(R, hp, 0.6, be, O.Rng(21))
        amp = orc["c"]
    assert np.array_equal(ref["sigma"], orc["sigma"])
    assert np.array_equal(ref["e"], orc["e"])
    assert np.array_equal(ref["amplitude"], amp)
    assert ref["min_e"] == orc["min_e"]


@pytest.mark.parametrize("cdp", [0, 1])
def test_cdp_minimize_and_score_bitwise(O, cdp):
    inst = O.gen_instance(600, 0.5, 0.1, 0.01, 4)
    rng = np.random.default_rng(1)
    sigma = (rng.random(600) < 0.2).astype(np.int32)
    R0 = rng.normal(size=600)
    hp = O.HyperParams()
    p = O.Problem(inst, O.LITERAL)
    out = RS.cdp_minimize(inst, sigma, R0, hp, cdp)
    assert np.array_equal(out, p.cdp(sigma, R0, cdp, hp))
    obj, rm, hm = RS.score(inst, out, sigma, 0.05)
    assert obj == p.objective_at(out, sigma, 0.05)
    assert rm == O.rmse(out, sigma, inst.x_true, inst.xi_true)
    assert hm == O.hamming_loss(sigma, inst.xi_true)


def test_random_small_problems_bitwise(O):
    """40 random small problems (N 8-150, random alpha / a / nu, BN / CN / Positive-P,
    Jacobi / CG, track_best, dt 0.01-0.1, 2-5 alternations of 10-200 steps, divergent
    ones included): the reference's own alternating_minimize and the oracle's LITERAL
    restatement agree bit for bit on R, sigma and the failure flag."""
    rng = np.random.default_rng(3)
    for _ in range(40):
        N = int(rng.choice([8, 20, 33, 64, 100, 150]))
        inst = O.gen_instance(N, float(rng.uniform(0.3, 0.95)), float(rng.uniform(0.05, 0.5)),
                              float(rng.choice([0.0, 0.01, 0.1])), int(rng.integers(0, 10 ** 6)))
        be = O.BACKENDS[str(rng.choice(["mfz-bn", "mfz-cn", "pp"]))]
        cd = int(rng.choice([O.CDP_JACOBI, O.CDP_CG]))
        hp = O.HyperParams(velo=int(rng.integers(1, 5)), n_steps=int(rng.integers(10, 200)),
                           dt=float(rng.choice([0.01, 0.02, 0.1])))
        tb = bool(rng.integers(0, 2))
        seed = int(rng.integers(0, 2 ** 62))
        ref = RS.alternating_minimize(inst, be, hp, seed, cdp=cd, track_best=tb)
        orc = O.Problem(inst, O.LITERAL).alternating_minimize(be, hp, O.Rng(seed), cdp=cd,
                                                              track_best=tb)
        assert ref["failed"] == orc["failed"]
        assert np.array_equal(ref["R"], orc["R"]) and np.array_equal(ref["sigma"], orc["sigma"])
