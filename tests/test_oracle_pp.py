"""Oracle Positive-P backend (solver_pp.cpp) -- known answers ported from the
reference's tests/test_solver_pp.cpp (each test cites its TEST_CASE line)."""
import math

import numpy as np
import pytest


def _vac(N):
    return np.zeros(N), np.zeros(N), np.zeros(N), np.ones(N)


def test_measurement_exact_without_saturation(O):
    """test_solver_pp.cpp:34-42: g2 = 0 -> mu_tilde == mu exactly."""
    mu = np.array([1.5, -0.25, 1e-10])
    noise = O.Rng(1).gauss_vector(3)
    assert np.array_equal(O.measured_amplitude(mu, noise, O.HyperParams(g2=0.0)), mu)


def test_measurement_rejects_bad_j(O):
    """test_solver_pp.cpp:44-56."""
    with pytest.raises(O.ConfigError):
        O.measured_amplitude(np.zeros(3), np.zeros(3), O.HyperParams(j=0.0))
    with pytest.raises(O.ConfigError):
        O.measured_amplitude(np.zeros(3), np.zeros(3), O.HyperParams(j=-1.0))


def test_measurement_noise_variance(O):
    """test_solver_pp.cpp:58-73: g2/(4 j dt) = 1 -> unit-variance deviation."""
    N = 100000
    mt = O.measured_amplitude(np.full(N, 5.0), O.Rng(77).gauss_vector(N),
                              O.HyperParams(g2=0.4, j=1.0, dt=0.1))
    dev = mt - 5.0
    var = dev @ dev / N
    assert abs(var - 1.0) < 3.0 * math.sqrt(2.0 / (N - 1))
    assert abs(dev.mean()) < 3.0 / math.sqrt(N)


def test_one_pump_step_fills_anomalous_moment_only(O):
    """test_solver_pp.cpp:75-87 (default dt 0.02)."""
    hp = O.HyperParams(K=0.0)
    mu, n, m, e = O.pp_step(*_vac(5), 1.0, hp, 0.3, np.ones(5), np.zeros(5),
                            O.Rng(3).gauss_vector(5))
    assert np.array_equal(mu, np.zeros(5)) and np.array_equal(n, np.zeros(5))
    assert np.array_equal(m, np.full(5, 0.02))


def test_fluctuations_feed_photon_number(O):
    """test_solver_pp.cpp:89-101."""
    hp = O.HyperParams(K=0.0, g2=0.0)
    st = _vac(2)
    g = O.Rng(3)
    for _ in range(2):
        st = O.pp_step(*st, 1.0, hp, 0.3, np.ones(2), np.zeros(2), g.gauss_vector(2))
    assert st[1][0] > 0.0 and np.array_equal(st[0], np.zeros(2))


def test_below_threshold_stays_vacuum(O):
    """test_solver_pp.cpp:103-115."""
    hp = O.HyperParams(K=0.0)
    st = _vac(3)
    g = O.Rng(9)
    for _ in range(100):
        st = O.pp_step(*st, 0.0, hp, 0.4, np.ones(3), np.zeros(3), g.gauss_vector(3))
    for a in st[:3]:
        assert np.array_equal(a, np.zeros(3))


def test_mean_field_saturates_when_g2_zero(O):
    """test_solver_pp.cpp:117-133: (p - 1 - j) mu - mu^3 = 0 at p = 2.4."""
    hp = O.HyperParams(K=0.0, g2=0.0, j=1.0)
    st = (np.array([0.3, -0.3]), np.zeros(2), np.zeros(2), np.ones(2))
    g = O.Rng(5)
    for _ in range(1500):
        st = O.pp_step(*st, 2.4, hp, 0.3, np.zeros(2), np.zeros(2), g.gauss_vector(2))
    t = math.sqrt(0.4)
    assert abs(st[0][0] - t) < 1e-4 and abs(st[0][1] + t) < 1e-4
    assert np.isfinite(st[1][0]) and np.isfinite(st[2][0])


def test_feedback_gain_exact_noiseless(O):
    """test_solver_pp.cpp:135-145."""
    hp = O.HyperParams(g2=0.0, K=0.0)
    out = O.pp_step(*_vac(1), 1.0, hp, 0.3, np.ones(1), np.zeros(1), O.Rng(2).gauss_vector(1))
    assert out[3][0] == 1.0 + hp.dt * (-hp.beta * (0.0 - hp.tau) * 1.0)


def test_full_call_consumes_one_deviate_per_mode_per_step(O):
    """test_solver_pp.cpp:147-156."""
    inst = O.gen_instance(7, 0.6, 0.2, 0.0, 13)
    p = O.Problem(inst, O.EXPLICIT)
    g = O.Rng(21)
    before = g.gauss_count
    p.run_pp(p.hz, O.HyperParams(n_steps=50), 0.4, g)
    assert g.gauss_count - before == 50 * 7


def test_local_field_reduces_to_scaled_bias(O):
    """test_solver_pp.cpp:158-173: mu_tilde == -sqrt(tau) zeroes the coupled term."""
    inst = O.gen_instance(8, 0.75, 0.25, 0.0, 17)
    p = O.Problem(inst, O.EXPLICIT)
    tau = 0.15
    h = p.local_field_pp(np.ones(8), np.full(8, -math.sqrt(tau)), tau)
    assert np.array_equal(h, math.sqrt(tau) * p.hz)


def test_matrix_free_and_dense_local_fields_agree(O):
    """test_solver_pp.cpp:175-183 (literal A^T(A w) vs explicit J, 1e-12)."""
    inst = O.gen_instance(12, 0.7, 0.3, 0.05, 23)
    g = O.Rng(4)
    R, mt = g.gauss_vector(12), g.gauss_vector(12)
    a = O.Problem(inst, O.LITERAL).local_field_pp(R, mt, 0.21)
    b = O.Problem(inst, O.EXPLICIT).local_field_pp(R, mt, 0.21)
    assert np.allclose(a, b, rtol=0, atol=1e-12)


def test_step_flags_blowups_by_spin(O):
    """test_solver_pp.cpp:185-202."""
    mu, n, m, e = _vac(4)
    mu[3] = 1e200
    with pytest.raises(O.DivergenceError) as ex:
        O.pp_step(mu, n, m, e, 1.0, O.HyperParams(), 0.3, np.zeros(4), np.zeros(4),
                  O.Rng(6).gauss_vector(4))
    assert ex.value.offending_index == 3
    with pytest.raises(O.InputError):
        O.pp_step(mu, n, m, e, 1.0, O.HyperParams(), 0.3, np.zeros(3), np.zeros(4), np.zeros(4))


def test_runaway_trajectories_abort(O):
    """test_solver_pp.cpp:204-212 (mu_abort guard)."""
    inst = O.gen_instance(6, 0.8, 0.5, 0.0, 3)
    p = O.Problem(inst, O.EXPLICIT)
    with pytest.raises(O.DivergenceError, match="exceeded"):
        p.run_pp(np.ones(6), O.HyperParams(mu_abort=1e-6, n_steps=10), 0.0, O.Rng(8))


def test_full_calls_reproducible_sigma_from_measurement(O):
    """test_solver_pp.cpp:214-238."""
    inst = O.gen_instance(10, 0.6, 0.2, 0.05, 29)
    p = O.Problem(inst, O.EXPLICIT)
    hp = O.HyperParams(n_steps=120, tau=0.21, K=0.01)
    a = p.run_pp(p.hz, hp, 0.4, O.Rng(14))
    b = p.run_pp(p.hz, hp, 0.4, O.Rng(14))
    assert np.array_equal(a["mu"], b["mu"]) and np.array_equal(a["sigma"], b["sigma"])
    assert np.array_equal(a["sigma"], (a["mu_tilde"] > 0).astype(np.int32))
    assert a["min_e"] <= 1.0


def test_alternation_with_pp_backend(O):
    """alternating_minimize with Backend::PositiveP (orchestrator.cpp:140-161, 170-235)."""
    inst = O.gen_instance(40, 0.7, 0.2, 0.01, 9)
    res = O.solve(inst, "pp", O.HyperParams(velo=4, n_steps=200), seed=3)
    assert not res["failed"] and len(res["history"]) == 5
    again = O.solve(inst, "pp", O.HyperParams(velo=4, n_steps=200), seed=3)
    assert np.array_equal(res["R"], again["R"])
