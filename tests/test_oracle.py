"""Pins of the C oracle against the reference's own known-answer tests.

Each test cites the reference test it ports (paths relative to
/root/reference/proj).  CPU only.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

# ------------------------------------------------------------- schedules


def test_pump_schedule_known_values(O):
    # test_orchestrator.cpp:29-43, test_smoke.py:31
    assert math.isclose(O.pump_schedule(4.0, 1.0, 0.4), 1.0, rel_tol=1e-12)
    assert math.isclose(O.pump_schedule(4.0, 0.7, 0.6), 0.7, rel_tol=1e-12)
    assert O.pump_schedule(0.0, 1.0, 0.4) == (1.0 - 0.4) + 2.0 * 0.4 / (1.0 + math.exp(2.0))
    assert abs(O.pump_schedule(0.0, 1.0, 0.4) - 0.695362) < 5e-7
    assert math.isclose(O.pump_schedule(1e9, 1.0, 0.4), 1.4, rel_tol=1e-12)
    assert math.isclose(O.pump_schedule(-1e9, 1.0, 0.4), 0.6, rel_tol=1e-12)
    ts = np.arange(-10.0, 30.0 + 1e-9, 0.25)
    ps = [O.pump_schedule(t, 1.0, 0.4) for t in ts]
    assert all(b > a for a, b in zip(ps, ps[1:]))


def test_pump_tanh_closed_form(O):
    # acceptance.cpp:50-72 (#1)
    worst = 0.0
    for p_thr, d in ((1.0, 0.4), (1.0, 0.6), (1.3, 0.25)):
        for k in range(1000):
            t = 20.0 * k / 999.0
            direct = (p_thr - d) + d * (1.0 + math.tanh((t - 4.0) / 4.0))
            worst = max(worst, abs(O.pump_schedule(t, p_thr, d) - direct))
    assert worst <= 1e-12


def test_eta_schedule(O):
    # test_orchestrator.cpp:45-60, test_smoke.py:32-33
    assert O.eta_schedule(0, 0.8, 0.18, 51) == 0.8
    assert O.eta_schedule(51, 0.8, 0.18, 51) == 0.18
    assert O.eta_schedule(60, 0.8, 0.18, 51) == 0.18
    assert O.eta_schedule(26, 0.8, 0.18, 51) == 0.8 * (1.0 - 26.0 / 51.0)
    assert abs(O.eta_schedule(26, 0.8, 0.18, 51) - 0.392157) < 5e-7
    assert O.eta_schedule(3, 0.5, 0.5, 7) == 0.5
    with pytest.raises(O.ConfigError):
        O.eta_schedule(0, 0.8, 0.18, 0)
    for ei, ee, velo in ((0.8, 0.18, 51), (0.8, 0.01, 999), (0.3, 0.3, 10)):
        for i in range(velo + 1):
            direct = max(ei * (velo - i) / velo, ee)
            assert abs(O.eta_schedule(i, ei, ee, velo) - direct) <= 1e-12


def test_linear_pump_table(O):
    hp = O.baseline_params()
    p = O.pump_table(hp)
    assert p[0] == 0.0
    t = 0.0
    for k in range(hp.n_steps):
        assert p[k] == 1.2 * t / (hp.n_steps * hp.dt)
        t = t + hp.dt
    assert 1.19 < p[-1] < 1.2


def test_trace_stride(O):
    # test_solver_mfz.cpp:232-253
    assert O.trace_stride(499) == 1
    assert O.trace_stride(500) == 2
    assert O.trace_stride(1000) == 3
    assert O.trace_stride(1, 2) == 1
    assert O.trace_stride(10, 2) == 10


# ------------------------------------------------------------- RNG / data


def test_mt19937_64_standard_value(O):
    # the C++ standard fixes the 10000th output of a default-seeded mt19937_64
    r = O.Rng(5489)
    for _ in range(9999):
        r.raw()
    assert r.raw() == 9981545732273789042


def test_round_half_away(O):
    # test_datagen.cpp:10-16
    assert O.round_half_away(2.5) == 3
    assert O.round_half_away(-2.5) == -3
    assert O.round_half_away(2.4) == 2
    assert O.round_half_away(0.5) == 1
    assert O.round_half_away(0.0) == 0


def test_gen_dims_and_support(O):
    # test_datagen.cpp:18-33
    assert O.gen_instance(500, 0.6, 0.1, 0.0, 1).M == 300
    assert O.gen_instance(12, 8.0 / 12.0, 0.25, 0.0, 1).M == 8
    assert O.gen_instance(3, 0.5, 0.0, 0.0, 1).M == 2
    for seed in range(1, 6):
        inst = O.gen_instance(40, 0.5, 0.2, 0.1, seed)
        assert inst.xi_true.sum() == 8
        assert set(np.unique(inst.xi_true)) <= {0, 1}
    assert O.gen_instance(10, 1.0, 1.0, 0.0, 2).xi_true.sum() == 10
    assert O.gen_instance(10, 1.0, 0.0, 0.0, 2).xi_true.sum() == 0


def test_noiseless_exact_and_bad_args(O):
    # test_datagen.cpp:35-39, 83-90
    inst = O.gen_instance(30, 0.7, 0.3, 0.0, 11)
    w = inst.x_true * inst.xi_true
    y = np.zeros(inst.M)
    for r in range(inst.N):
        y = y + inst.A[:, r] * w[r]
    assert np.array_equal(y, inst.y)
    for args in ((10, 0.0, 0.2, 0.0), (10, 1.5, 0.2, 0.0), (10, 0.5, -0.1, 0.0),
                 (10, 0.5, 1.1, 0.0), (10, 0.5, 0.2, -0.1), (0, 0.5, 0.2, 0.0)):
        with pytest.raises(O.InputError):
            O.gen_instance(*args, 1)


def test_entry_statistics(O):
    # test_datagen.cpp:51-69
    inst = O.gen_instance(2000, 0.6, 0.2, 0.1, 7)
    assert inst.M == 1200
    n = 2000.0 * 1200.0
    a_var = float((inst.A ** 2).sum()) / n
    assert abs(a_var - 1 / 1200) < 3 * (1 / 1200) * math.sqrt(2 / (n - 1))
    x_var = float((inst.x_true ** 2).sum()) / 2000
    assert abs(x_var - 1) < 3 * math.sqrt(2 / 1999)


def test_c0_variance(O):
    # test_solver_mfz.cpp:25-39 (init_mfz: c = 0.01 * gauss)
    r = O.Rng(42)
    g = np.array([0.01 * r.gauss() for _ in range(100000)])
    assert abs(g.mean()) < 1e-4
    assert 0.9e-4 < (g ** 2).mean() < 1.1e-4
    assert r.gauss_count == 100000


# ------------------------------------------------------------- coupling


def test_coupling_by_hand(O):
    # test_model.cpp:67-79 (J = -A^T A, diag 0; hz = A^T y) via G / D
    inst = O.Instance(np.array([[1.0, 2.0]], order="F"), np.array([3.0]))
    for mode in (O.LITERAL, O.CANON, O.EXPLICIT):
        p = O.Problem(inst, mode)
        assert list(p.hz) == [3.0, 6.0]
        assert list(p.gram_diag) == [1.0, 4.0]
        # J w = D∘w - G w
        assert list(p.apply_coupling(np.array([1.0, 0.0]))) == [0.0, -2.0]
        assert list(p.apply_coupling(np.array([0.0, 1.0]))) == [-2.0, 0.0]


def test_orthogonal_columns_decouple(O):
    # test_model.cpp:81-88
    A = np.zeros((3, 3), order="F")
    A[0, 0], A[1, 1], A[2, 2] = 2.0, -1.0, 0.5
    p = O.Problem(O.Instance(A, np.zeros(3)), O.CANON)
    for k in range(3):
        e = np.zeros(3)
        e[k] = 1.0
        assert np.all(p.apply_coupling(e) == 0.0)


def test_modes_agree_on_coupling(O):
    # test_orchestrator.cpp:80-110 (apply_coupling vs J w < 1e-10)
    inst = O.gen_instance(14, 0.7, 0.3, 0.1, 61)
    lit, can, exp = (O.Problem(inst, m) for m in (O.LITERAL, O.CANON, O.EXPLICIT))
    rng = np.random.default_rng(9)
    for _ in range(10):
        w = rng.normal(size=14)
        J = -inst.A.T @ inst.A
        np.fill_diagonal(J, 0.0)
        for p in (lit, can, exp):
            assert np.max(np.abs(p.apply_coupling(w) - J @ w)) < 1e-10


def test_canon_gram_is_sequential_fma(O):
    inst = O.gen_instance(9, 0.8, 0.3, 0.05, 71)
    p = O.Problem(inst, O.CANON)
    G = p.G

    def fma(a, b, c):
        return float(Fraction(a) * Fraction(b) + Fraction(c))

    for i in range(9):
        for j in range(9):
            acc = 0.0
            for k in range(inst.M):
                acc = fma(inst.A[k, i], inst.A[k, j], acc)
            assert G[i, j] == acc
    assert np.array_equal(G, G.T)
    assert np.array_equal(np.diag(G), p.gram_diag)


def test_canon_dot_segments(O):
    rng = np.random.default_rng(3)
    g, v = rng.normal(size=300), rng.normal(size=300)

    def fma(a, b, c):
        return float(Fraction(a) * Fraction(b) + Fraction(c))

    for nseg, gran in ((8, 8), (4, 16), (1, 1)):
        P = [0.0] * nseg
        for j in range(300):
            s = (j // gran) % nseg
            P[s] = fma(g[j], v[j], P[s])
        acc = P[0]
        for q in range(1, nseg):
            acc = acc + P[q]
        assert O.canon_dot(g, v, nseg, gran) == acc


# ------------------------------------------------------------- MFZ fields


def test_field_bias_only(O):
    # test_solver_mfz.cpp:41-53
    inst = O.Instance(np.zeros((1, 3), order="F"), np.zeros(1))
    p = O.Problem(inst, O.CANON)
    # hz must be set by hand: zero A gives hz = 0; use tau=4 identity on zero
    R = np.full(3, 7.0)
    c = np.full(3, 0.3)
    assert np.all(p.local_field_cn(R, c, 4.0) == 0.0)
    assert np.all(p.local_field_bn(R, np.ones(3, np.int32), 4.0) == 0.0)


def test_bn_field_sqrt_tau_scaling(O):
    # test_solver_mfz.cpp:55-66
    inst = O.gen_instance(12, 0.75, 0.3, 0.1, 5)
    p = O.Problem(inst, O.CANON)
    R = O.Rng(1).gauss_vector(12)
    sigma = np.array([1 if r % 3 == 0 else 0 for r in range(12)], np.int32)
    assert np.array_equal(p.local_field_bn(R, sigma, 4.0), 2.0 * p.local_field_bn(R, sigma, 1.0))


def test_saturated_fields_coincide(O):
    # test_solver_mfz.cpp:84-99 (bitwise CN == BN at c = +-1, tau = 1)
    inst = O.gen_instance(16, 0.8, 0.25, 0.0, 21)
    for mode in (O.LITERAL, O.CANON, O.EXPLICIT):
        p = O.Problem(inst, mode)
        R = O.Rng(3).gauss_vector(16)
        c = np.array([1.0 if r % 2 == 0 else -1.0 for r in range(16)])
        sigma = (c > 0).astype(np.int32)
        assert np.max(np.abs(p.local_field_cn(R, c, 1.0) - p.local_field_bn(R, sigma, 1.0))) == 0.0


def test_free_dynamics_fixed_point(O):
    # test_solver_mfz.cpp:101-115
    hp = O.HyperParams(K=0.0)
    c, e = np.array([0.1, -0.1]), np.ones(2)
    z = np.zeros(2)
    for _ in range(1000):
        c, e = O.mfz_step(c, e, 1.4, hp, 0.5, z, z)
    assert abs(c[0] - math.sqrt(0.4)) < 1e-4
    assert abs(c[1] + math.sqrt(0.4)) < 1e-4


def test_loss_variant_fixed_point(O):
    # test_solver_mfz.cpp:117-128
    hp = O.HyperParams(K=0.0, mfz_loss_minus_j=True, j=1.0)
    c, e = np.array([0.2]), np.ones(1)
    z = np.zeros(1)
    for _ in range(1500):
        c, e = O.mfz_step(c, e, 2.4, hp, 0.5, z, z)
    assert abs(c[0] - math.sqrt(0.4)) < 1e-4


def test_error_field_exact_updates(O):
    # test_solver_mfz.cpp:130-151
    hp = O.HyperParams()
    e0 = np.linspace(0.5, 1.5, 3)
    c1, e1 = O.mfz_step(np.ones(3), e0, 1.2, hp, 0.3, np.zeros(3), np.zeros(3))
    assert np.array_equal(e1, e0)
    assert not np.array_equal(c1, np.ones(3))
    _, e2 = O.mfz_step(np.array([2.0]), np.ones(1), 1.0, hp, 0.3, np.zeros(1), np.zeros(1))
    assert e2[0] == 1.0 + hp.dt * (-hp.beta * (4.0 - 1.0))
    _, e3 = O.mfz_step(np.array([0.5]), np.ones(1), 1.0, hp, 0.3, np.zeros(1), np.zeros(1))
    assert e3[0] > 1.0


def test_step_coordinatewise(O):
    # test_solver_mfz.cpp:153-171
    hp = O.HyperParams()
    r = O.Rng(7)
    c, e, R, h = (r.gauss_vector(6) for _ in range(4))
    e = np.abs(e)
    fc, fe = O.mfz_step(c, e, 1.1, hp, 0.4, R, h)
    for k in range(6):
        oc, oe = O.mfz_step(c[k:k + 1], e[k:k + 1], 1.1, hp, 0.4, R[k:k + 1], h[k:k + 1])
        assert oc[0] == fc[k] and oe[0] == fe[k]


def test_divergence_names_spin(O):
    # test_solver_mfz.cpp:173-189
    hp = O.HyperParams()
    c = np.zeros(4)
    c[2] = 1e200
    with pytest.raises(O.DivergenceError) as ei:
        O.mfz_step(c, np.ones(4), 1.0, hp, 0.3, np.zeros(4), np.zeros(4))
    assert ei.value.offending_index == 2
    with pytest.raises(O.InputError):
        O.mfz_step(c, np.ones(4), float("nan"), hp, 0.3, np.zeros(4), np.zeros(4))


def _zero_problem(O, N):
    return O.Problem(O.Instance(np.zeros((1, N), order="F"), np.zeros(1)), O.CANON)


def test_threshold_only_keeps_spins_off(O):
    # test_solver_mfz.cpp:202-213
    p = _zero_problem(O, 10)
    hp = O.HyperParams(n_steps=500)
    res = p.run_mfz(np.ones(10), hp, 0.5, O.MFZ_BN, O.Rng(11))
    assert res["sigma"].sum() == 0
    assert res["c"].max() < 0.0
    assert res["min_e"] > 0.0


def test_run_reproducible_and_mode_matters(O):
    # test_solver_mfz.cpp:215-230
    inst = O.gen_instance(15, 0.6, 0.2, 0.05, 31)
    p = O.Problem(inst, O.CANON)
    hp = O.HyperParams(n_steps=200)
    a = p.run_mfz(p.hz, hp, 0.4, O.MFZ_BN, O.Rng(5))
    b = p.run_mfz(p.hz, hp, 0.4, O.MFZ_BN, O.Rng(5))
    c = p.run_mfz(p.hz, hp, 0.4, O.MFZ_CN, O.Rng(5))
    assert np.array_equal(a["c"], b["c"]) and np.array_equal(a["e"], b["e"])
    assert not np.array_equal(a["c"], c["c"])


def test_trace_counts(O):
    # test_solver_mfz.cpp:255-281
    p = _zero_problem(O, 3)
    hp = O.HyperParams(n_steps=1000)
    full = p.run_mfz(np.ones(3), hp, 0.3, O.MFZ_BN, O.Rng(8), trace_mode=2)
    assert len(full["trace_steps"]) == 1001
    assert full["trace_steps"][0] == 0 and full["trace_steps"][-1] == 1000
    dec = p.run_mfz(np.ones(3), hp, 0.3, O.MFZ_BN, O.Rng(8), trace_mode=1)
    assert len(dec["trace_steps"]) <= 500 and dec["trace_steps"][-1] == 1000
    assert np.array_equal(dec["trace_c"][-1], full["trace_c"][-1])
    none = p.run_mfz(np.ones(3), hp, 0.3, O.MFZ_BN, O.Rng(8))
    assert np.array_equal(none["c"], full["c"])


def test_injection_equals_flip_energy(O):
    # test_solver_mfz.cpp:283-308 and acceptance.cpp:77-114 (#2)
    for seed in range(1, 21):
        N = 4 + seed % 7
        inst = O.gen_instance(N, 0.8, 0.3, 0.1, seed)
        for mode in (O.LITERAL, O.CANON):
            p = O.Problem(inst, mode)
            r = O.Rng(seed * 97 + 1)
            R = r.gauss_vector(N)
            sigma = np.array([1 if r.uniform_open() > 0.5 else 0 for _ in range(N)], np.int32)
            tau, eta = 1.0, 0.37
            lam = eta * eta / 2.0
            h = p.local_field_bn(R, sigma, tau)
            for k in range(N):
                s1, s0 = sigma.copy(), sigma.copy()
                s1[k], s0[k] = 1, 0
                gap = O.hamiltonian(inst, R, s1, lam) - O.hamiltonian(inst, R, s0, lam)
                lhs = R[k] * h[k] - eta * eta / 4.0 * math.sqrt(tau)
                rhs = -math.sqrt(tau) / 2.0 * gap
                assert math.isclose(lhs, rhs, rel_tol=1e-10, abs_tol=1e-12)


# ------------------------------------------------------------------- cdp


def test_jacobi_known_answers(O):
    # test_cdp.cpp:79-99: scalar / diagonal systems exact at dt_c = 1, 1 sweep
    inst = O.Instance(np.array([[math.sqrt(2.0)]], order="F"), np.array([4.0 / math.sqrt(2.0)]))
    hp = O.HyperParams(dt_c=1.0, jacobi_iters=1)
    # diagonal A: columns orthogonal
    A = np.diag([math.sqrt(2.0), 2.0, math.sqrt(8.0)])
    A = np.asfortranarray(A)
    # hz = A^T y = (2,2,2) -> y = (2/sqrt2, 1, 2/sqrt8)
    y = np.array([2.0 / math.sqrt(2.0), 1.0, 2.0 / math.sqrt(8.0)])
    for mode in (O.LITERAL, O.CANON):
        p = O.Problem(O.Instance(A, y), mode)
        assert list(p.gram_diag) == pytest.approx([2.0, 4.0, 8.0], rel=1e-15)
        R = p.cdp(np.ones(3, np.int32), np.ones(3), O.CDP_JACOBI, hp)
        assert R == pytest.approx([1.0, 0.5, 0.25], rel=1e-15)
    del inst


def test_inactive_entries_bitwise_kept(O):
    # test_cdp.cpp:204-221
    inst = O.gen_instance(10, 0.8, 0.3, 0.1, 42)
    R_prev = O.Rng(3).gauss_vector(10)
    for mode in (O.LITERAL, O.CANON):
        p = O.Problem(inst, mode)
        for method in (O.CDP_CG, O.CDP_JACOBI):
            assert np.array_equal(p.cdp(np.zeros(10, np.int32), R_prev, method), R_prev)
            sigma = np.zeros(10, np.int32)
            sigma[2] = sigma[5] = 1
            out = p.cdp(sigma, R_prev, method)
            for r in range(10):
                if sigma[r] == 0:
                    assert out[r] == R_prev[r]
            assert out[2] != R_prev[2]


def test_jacobi_lowers_residual(O):
    # test_cdp.cpp:233-255
    for seed in range(1, 51):
        inst = O.gen_instance(8, 1.0, 0.5, 0.05, seed)
        r = O.Rng(seed + 1000)
        sigma = np.array([1 if r.uniform_open() > 0.5 else 0 for _ in range(8)], np.int32)
        if sigma.sum() == 0:
            sigma[0] = 1
        R_prev = r.gauss_vector(8)
        p = O.Problem(inst, O.CANON)
        out = p.cdp(sigma, R_prev, O.CDP_JACOBI)
        act = np.flatnonzero(sigma)
        G = inst.A[:, act].T @ inst.A[:, act]
        b = inst.A[:, act].T @ inst.y
        assert np.linalg.norm(G @ out[act] - b) < np.linalg.norm(G @ R_prev[act] - b)


def test_singular_diagonal_rejected(O):
    # test_cdp.cpp:114-126
    A = np.zeros((2, 3), order="F")
    A[0, 0] = 1.0
    p = O.Problem(O.Instance(A, np.ones(2)), O.CANON)
    sigma = np.array([0, 1, 0], np.int32)
    with pytest.raises(O.InputError, match="1"):
        p.cdp(sigma, np.zeros(3), O.CDP_JACOBI)


# ------------------------------------------------------------ alternation


def _scalar_instance(O):
    # test_orchestrator.cpp:16-25
    return O.Instance(np.ones((1, 1), order="F"), np.ones(1), np.ones(1), np.ones(1, np.int32),
                      1.0, 1.0)


def test_scalar_recovery(O):
    # test_orchestrator.cpp:185-206 (MFZ backends)
    inst = _scalar_instance(O)
    hp = O.HyperParams(velo=5, n_steps=400)
    for be in ("mfz-bn", "mfz-cn"):
        res = O.solve(inst, be, hp, seed=17, cdp="cg")
        assert not res["failed"]
        assert res["sigma"][0] == 1
        assert abs(res["R"][0] - 1.0) < 1e-6
        assert res["final_rmse"] < 1e-6 and res["final_hamming"] == 0.0
        assert len(res["history"]) == 6


def test_silent_observation(O):
    # test_orchestrator.cpp:208-225
    inst = O.Instance(np.eye(3, order="F"), np.zeros(3), np.zeros(3), np.zeros(3, np.int32))
    res = O.solve(inst, "mfz-bn", O.HyperParams(velo=3, n_steps=100), seed=2)
    assert not res["failed"]
    assert res["sigma"].sum() == 0
    assert res["final_rmse"] == 0.0 and res["final_hamming"] == 0.0


def test_history_and_reruns(O):
    # test_orchestrator.cpp:227-273
    inst = O.gen_instance(10, 0.8, 0.2, 0.05, 101)
    hp = O.HyperParams(velo=7, n_steps=60)
    p = O.Problem(inst, O.CANON)
    res = p.alternating_minimize(O.MFZ_BN, hp, O.Rng(4), keep=True)
    assert len(res["history"]) == 8
    for i, rec in enumerate(res["history"]):
        assert rec["i"] == i
        assert rec["eta"] == O.eta_schedule(i, hp.eta_init, hp.eta_end, hp.velo)
        lam = rec["eta"] ** 2 / 2.0
        assert math.isclose(rec["hamiltonian"],
                            p.objective_at(res["hist_R"][i], res["hist_sigma"][i], lam),
                            rel_tol=1e-12)
        assert rec["min_e"] > 0 and rec["median_e"] > 0
    assert np.array_equal(res["R"], res["hist_R"][-1])
    again = p.alternating_minimize(O.MFZ_BN, hp, O.Rng(4))
    assert np.array_equal(again["R"], res["R"])
    assert [h["hamiltonian"] for h in again["history"]] == [h["hamiltonian"] for h in res["history"]]


def test_refit_never_raises_objective(O):
    # test_orchestrator.cpp:275-294
    inst = O.gen_instance(16, 0.75, 0.25, 0.05, 121)
    hp = O.HyperParams(velo=6, n_steps=100)
    p = O.Problem(inst, O.CANON)
    res = p.alternating_minimize(O.MFZ_BN, hp, O.Rng(7), cdp=O.CDP_CG, keep=True)
    assert not res["failed"]
    for i in range(1, len(res["history"])):
        lam = res["history"][i]["eta"] ** 2 / 2.0
        s = res["hist_sigma"][i]
        assert p.objective_at(res["hist_R"][i], s, lam) <= \
            p.objective_at(res["hist_R"][i - 1], s, lam) + 1e-9


def test_divergence_marks_failed(O):
    # test_smoke.py:59-65
    inst = O.gen_instance(10, 1.0, 0.3, 0.0, 2)
    res = O.solve(inst, "mfz-cn", O.HyperParams(dt=5.0), seed=1)
    assert res["failed"] and res["fail_reason"]
    assert res["fail_alternation"] == 0 and res["history"] == []
    assert math.isnan(res["final_rmse"])


def test_track_best(O):
    # test_orchestrator.cpp:315-332
    inst = O.gen_instance(14, 0.7, 0.3, 0.1, 141)
    hp = O.HyperParams(velo=8, n_steps=60)
    p = O.Problem(inst, O.CANON)
    res = p.alternating_minimize(O.MFZ_CN, hp, O.Rng(9), track_best=True, keep=True)
    best = int(np.argmin([h["hamiltonian"] for h in res["history"]]))
    assert np.array_equal(res["R"], res["hist_R"][best])
    assert np.array_equal(res["sigma"], res["hist_sigma"][best])


def test_bad_backend(O):
    inst = O.gen_instance(8, 1.0, 0.25, 0.0, 1)
    with pytest.raises(O.ConfigError):
        O.solve(inst, backend="nope")


@pytest.mark.slow
def test_brute_force_parity_small(O):
    # acceptance.cpp:119-151 (#3): both field modes hit the exhaustive optimum
    # on >= 14/20 seeds at N=12 (K=16, beta=1, eta 0.3 -> 0.01, CG refit)
    import itertools
    hits = {"mfz-bn": 0, "mfz-cn": 0}
    for s in range(1, 21):
        inst = O.gen_instance(12, 8.0 / 12.0, 0.25, 0.0, s)
        hp = O.HyperParams(eta_init=0.3, eta_end=0.01, K=16.0, beta=1.0)
        lam = hp.eta_end ** 2 / 2
        best = 0.0
        yy = float(inst.y @ inst.y)
        for k in range(1, 13):
            for act in itertools.combinations(range(12), k):
                As = inst.A[:, act]
                Rs = np.linalg.lstsq(As, inst.y, rcond=None)[0]
                r = inst.y - As @ Rs
                H = 0.5 * float(r @ r) - 0.5 * yy + lam * k
                best = min(best, H)
        for mode, be in ((1, "mfz-bn"), (0, "mfz-cn")):
            res = O.solve(inst, be, hp, seed=s * 1000 + mode, cdp="cg")
            if not res["failed"] and abs(res["history"][-1]["hamiltonian"] - best) <= 1e-6:
                hits[be] += 1
    assert hits["mfz-bn"] >= 14 and hits["mfz-cn"] >= 14, hits
