"""GPU parity: the CUDA path (through the C ABI) against the C oracle.

fp64: bitwise against the oracle's ORC_CANON mode, which restates the GPU's
documented summation order (gram: one sequential fma chain per entry; G*v:
8 segments of 8-wide granules, fma chains, segments added left to right).
Scalars that the GPU reduces in a different order (objective, rmse) are
compared at 1e-12 relative.  fp32: the stated tolerances below.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_SCALAR = 1e-12


def _ctx(P, insts, dtype="f64"):
    ctx = P.Context(0, dtype)
    ctx.set_problems(insts)
    ctx.build_coupling()
    return ctx


def _probs(O, insts):
    nseg, gran = 8, 8
    return [O.Problem(i, O.CANON, nseg, gran) for i in insts]


@pytest.fixture(scope="module")
def small(O):
    # two instances of equal N, different M (phase-grid style)
    return [O.gen_instance(200, 0.6, 0.2, 0.01, 3), O.gen_instance(200, 0.4, 0.1, 0.01, 4)]


def test_gemv_order_matches_oracle_params(gpu):
    assert gpu.gemv_order("f64") == (8, 8)


def test_gram_build_bitwise(gpu, O, small):
    ctx = _ctx(gpu, small)
    for b, (inst, p) in enumerate(zip(small, _probs(O, small))):
        G, hz, D = ctx.get_coupling(b)
        assert np.array_equal(G, p.G)
        assert np.array_equal(hz, p.hz)
        assert np.array_equal(D, p.gram_diag)
    ctx.close()


@pytest.mark.parametrize("N", [37, 128, 300])
def test_gram_build_ragged_sizes(gpu, O, N):
    insts = [O.gen_instance(N, 0.5, 0.2, 0.01, 11)]
    ctx = _ctx(gpu, insts)
    G, hz, D = ctx.get_coupling(0)
    p = _probs(O, insts)[0]
    assert np.array_equal(G, p.G) and np.array_equal(hz, p.hz) and np.array_equal(D, p.gram_diag)
    ctx.close()


@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
@pytest.mark.parametrize("R", [1, 3, 16])
def test_single_step_bitwise(gpu, O, small, backend, R):
    """L1: identical (c, e, R) -> bitwise (h, c', e')."""
    ctx = _ctx(gpu, small)
    probs = _probs(O, small)
    B, N = len(small), small[0].N
    rng = np.random.default_rng(R)
    Rs = rng.normal(size=(B, R, N))
    c = rng.normal(scale=0.5, size=(B, R, N))
    e = np.abs(rng.normal(size=(B, R, N))) + 0.1
    hp = O.baseline_params()
    ghp = gpu.baseline_params()
    eta, p = 0.37, 0.83
    out = ctx.mfz_step(R, backend, ghp, eta, p, Rs, c, e)
    for b in range(B):
        for r in range(R):
            if backend == "mfz-bn":
                h = probs[b].local_field_bn(Rs[b, r], (c[b, r] > 0).astype(np.int32), hp.tau)
            else:
                h = probs[b].local_field_cn(Rs[b, r], c[b, r], hp.tau)
            co, eo = O.mfz_step(c[b, r], e[b, r], p, hp, eta, Rs[b, r], h)
            assert np.array_equal(out["h"][b, r], h)
            assert np.array_equal(out["c"][b, r], co)
            assert np.array_equal(out["e"][b, r], eo)
    assert (out["fail_index"] == -1).all()
    ctx.close()


def test_step_divergence_index(gpu, O):
    """test_solver_mfz.cpp:173-189: a blown-up amplitude names the spin."""
    inst = O.Instance(np.zeros((1, 4), order="F"), np.zeros(1))
    ctx = _ctx(gpu, [inst])
    c = np.zeros((1, 1, 4))
    c[0, 0, 2] = 1e200
    out = ctx.mfz_step(1, "mfz-bn", gpu.HyperParams(), 0.3, 1.0, np.zeros((1, 1, 4)), c,
                       np.ones((1, 1, 4)))
    assert out["fail_index"][0, 0] == 2
    with pytest.raises(gpu.InputError):
        ctx.mfz_step(1, "mfz-bn", gpu.HyperParams(), 0.3, float("nan"), np.zeros((1, 1, 4)), c,
                     np.ones((1, 1, 4)))
    ctx.close()


@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
def test_run_cim_bitwise(gpu, O, small, backend):
    """L2: a whole CIM call from identical c0 / R."""
    R = 4
    ctx = _ctx(gpu, small)
    probs = _probs(O, small)
    B, N = len(small), small[0].N
    hp = O.baseline_params(n_steps=300)
    seeds = [[O.mix_seed(inst.seed, 1 + 3 * r) for r in range(R)] for inst in small]
    c0 = np.zeros((B, R, N))
    for b in range(B):
        for r in range(R):
            g = O.Rng(seeds[b][r])
            c0[b, r] = [0.01 * g.gauss() for _ in range(N)]
    Rs = np.stack([np.stack([p.hz] * R) for p in probs])
    out = ctx.run_cim(R, backend, gpu.baseline_params(n_steps=300), 0.5, Rs, c0)
    be = O.MFZ_BN if backend == "mfz-bn" else O.MFZ_CN
    for b in range(B):
        for r in range(R):
            ref = probs[b].run_mfz(Rs[b, r], hp, 0.5, be, O.Rng(seeds[b][r]))
            assert np.array_equal(out["c"][b, r], ref["c"])
            assert np.array_equal(out["e"][b, r], ref["e"])
            assert np.array_equal(out["sigma"][b, r], ref["sigma"])
            assert out["min_e"][b, r] == ref["min_e"]
    ctx.close()


def test_refit_bitwise(gpu, O, small):
    """cdp_minimize (Jacobi): active entries bitwise, inactive untouched."""
    R = 3
    ctx = _ctx(gpu, small)
    probs = _probs(O, small)
    B, N = len(small), small[0].N
    rng = np.random.default_rng(5)
    sigma = (rng.random((B, R, N)) < 0.3).astype(np.int32)
    sigma[0, 0] = 0  # empty support: returned unchanged
    Rp = rng.normal(size=(B, R, N))
    hp = O.HyperParams()
    out = ctx.refit(R, sigma, Rp, gpu.HyperParams())
    for b in range(B):
        for r in range(R):
            ref = probs[b].cdp(sigma[b, r], Rp[b, r], O.CDP_JACOBI, hp)
            assert np.array_equal(out[b, r], ref)
    assert np.array_equal(out[0, 0], Rp[0, 0])
    ctx.close()


def test_refit_singular_diagonal(gpu, O):
    A = np.zeros((2, 3), order="F")
    A[0, 0] = 1.0
    ctx = _ctx(gpu, [O.Instance(A, np.ones(2))])
    with pytest.raises(gpu.InputError, match="1"):
        ctx.refit(1, np.array([[[0, 1, 0]]], np.int32), np.zeros((1, 1, 3)))
    ctx.close()


def test_score(gpu, O, small):
    R = 2
    ctx = _ctx(gpu, small)
    probs = _probs(O, small)
    B, N = len(small), small[0].N
    rng = np.random.default_rng(8)
    Rs = rng.normal(size=(B, R, N))
    sigma = (rng.random((B, R, N)) < 0.4).astype(np.int32)
    out = ctx.score(R, Rs, sigma, 0.05)
    for b in range(B):
        for r in range(R):
            obj = probs[b].objective_at(Rs[b, r], sigma[b, r], 0.05)
            assert math.isclose(out["objective"][b, r], obj, rel_tol=TOL_SCALAR)
            rm = O.rmse(Rs[b, r], sigma[b, r], small[b].x_true, small[b].xi_true)
            assert math.isclose(out["rmse"][b, r], rm, rel_tol=TOL_SCALAR)
            assert out["hamming"][b, r] == O.hamming_loss(sigma[b, r], small[b].xi_true)
    ctx.close()


def _oracle_solve(O, inst, be, hp, seed, track_best=False):
    p = O.Problem(inst, O.CANON)
    return p.alternating_minimize(be, hp, O.Rng(seed), track_best=track_best)


def test_solve_config0_bitwise(gpu, O):
    """L3 on BASELINE config 0 (N=500, M=300, K=100, 1 replica, 20 x 1000, fp64)."""
    inst = O.gen_instance(500, 0.6, 0.2, 0.01, 0)
    hp = O.baseline_params()
    seed = O.mix_seed(0, 1)
    ref = _oracle_solve(O, inst, O.MFZ_BN, hp, seed)
    ctx = _ctx(gpu, [inst])
    res = ctx.solve(1, "mfz-bn", gpu.baseline_params(), [seed])
    assert res["fail_alt"][0, 0] == -1 and not ref["failed"]
    assert np.array_equal(res["sigma"][0, 0], ref["sigma"])
    assert np.array_equal(res["R"][0, 0], ref["R"])
    H = res["history"][0, 0]
    assert res["n_hist"][0, 0] == len(ref["history"]) == 20
    for h, g in zip(ref["history"], H):
        assert g["i"] == h["i"] and g["eta"] == h["eta"] and g["support"] == h["support"]
        assert g["min_e"] == h["min_e"] and g["median_e"] == h["median_e"]
        assert math.isclose(g["hamiltonian"], h["hamiltonian"], rel_tol=TOL_SCALAR)
        assert math.isclose(g["rmse"], h["rmse"], rel_tol=TOL_SCALAR)
        assert g["hamming"] == h["hamming"]
    ctx.close()


@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
def test_solve_batch_replicas_bitwise(gpu, O, backend):
    """Multi-instance x multi-replica driver: every trajectory equals its own
    independent reference trial (replica seeds mix_seed(s, backend + 3 rho))."""
    insts = [O.gen_instance(160, 0.5, 0.1, 0.01, s) for s in (1, 2)]
    R = 3
    hp = O.baseline_params(velo=4, n_steps=250)
    ghp = gpu.baseline_params(velo=4, n_steps=250)
    be = O.MFZ_BN if backend == "mfz-bn" else O.MFZ_CN
    seeds = np.array([[O.mix_seed(i.seed, be + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    ctx = _ctx(gpu, insts)
    res = ctx.solve(R, backend, ghp, seeds, track_best=True)
    for b, inst in enumerate(insts):
        for r in range(R):
            ref = _oracle_solve(O, inst, be, hp, int(seeds[b, r]), track_best=True)
            assert np.array_equal(res["R"][b, r], ref["R"])
            assert np.array_equal(res["sigma"][b, r], ref["sigma"])
            assert res["n_hist"][b, r] == len(ref["history"])
    ctx.close()


def test_python_solve_mirrors_reference_api(gpu, O):
    """cimcs.solve signature and result dict (bindings/module.cpp:15-39, 127-141)."""
    inst = gpu.gen_instance(12, 1.0, 0.25, 0.0, 11)
    params = gpu.HyperParams(eta_end=0.01)
    res = gpu.solve(inst, backend="mfz-bn", params=params, seed=5)
    assert not res["failed"]
    assert len(res["history"]) == params.velo + 1
    ref = O.solve(O.gen_instance(12, 1.0, 0.25, 0.0, 11), "mfz-bn", O.HyperParams(eta_end=0.01),
                  seed=5)
    assert np.array_equal(res["R"], ref["R"]) and np.array_equal(res["sigma"], ref["sigma"])
    with pytest.raises(gpu.ConfigError):
        gpu.solve(inst, backend="nope")


def test_divergence_marks_trial_failed(gpu, O):
    """test_smoke.py:59-65: dt=5 fails the trial, history empty, NaN metrics."""
    inst = gpu.gen_instance(10, 1.0, 0.3, 0.0, 2)
    res = gpu.solve(inst, backend="mfz-cn", params=gpu.HyperParams(dt=5.0), seed=1)
    ref = O.solve(O.gen_instance(10, 1.0, 0.3, 0.0, 2), "mfz-cn", O.HyperParams(dt=5.0), seed=1)
    assert res["failed"] and ref["failed"]
    assert res["fail_alternation"] == ref["fail_alternation"] == 0
    assert res["fail_reason"] == ref["fail_reason"]
    assert res["history"] == [] and math.isnan(res["final_rmse"])


def test_silent_and_scalar_instances(gpu, O):
    """test_orchestrator.cpp:185-225 (MFZ backends, Jacobi refit on the GPU path)."""
    silent = gpu.Instance(np.eye(3, order="F"), np.zeros(3), np.zeros(3), np.zeros(3, np.int32))
    res = gpu.solve(silent, "mfz-bn", gpu.HyperParams(velo=3, n_steps=100), seed=2)
    assert not res["failed"] and res["sigma"].sum() == 0 and res["final_rmse"] == 0.0
    scal = gpu.Instance(np.ones((1, 1), order="F"), np.ones(1), np.ones(1), np.ones(1, np.int32))
    for be in ("mfz-bn", "mfz-cn"):
        hp = gpu.HyperParams(velo=5, n_steps=400, jacobi_iters=400)
        res = gpu.solve(scal, be, hp, seed=17)
        assert res["sigma"][0] == 1 and abs(res["R"][0] - 1.0) < 1e-6
        assert len(res["history"]) == 6


def test_fp32_path_tolerance(gpu, O):
    """fp32 mode vs the fp64 oracle on config-0 shaped instances.

    Stated fp32 tolerance: supports identical on >= 90% of trials and the
    mean |dRMSE| / RMSE <= 5e-2 (fp32 rounding perturbs near-zero spins)."""
    insts = [O.gen_instance(300, 0.6, 0.2, 0.01, s) for s in range(1, 7)]
    hp = O.baseline_params(velo=9)
    seeds = np.array([[O.mix_seed(i.seed, 1)] for i in insts], np.uint64)
    ctx = _ctx(gpu, insts, "f32")
    res = ctx.solve(1, "mfz-bn", gpu.baseline_params(velo=9), seeds)
    same, rel = 0, []
    for b, inst in enumerate(insts):
        ref = _oracle_solve(O, inst, O.MFZ_BN, hp, int(seeds[b, 0]))
        same += np.array_equal(res["sigma"][b, 0], ref["sigma"])
        g = O.rmse(res["R"][b, 0], res["sigma"][b, 0], inst.x_true, inst.xi_true)
        rel.append(abs(g - ref["final_rmse"]) / ref["final_rmse"])
    assert same >= 0.9 * len(insts)
    assert np.mean(rel) <= 5e-2
    ctx.close()


# ------------------------------------------------ fp32 tensor-core (tcgen05) path

def _ctx_opts(P, insts, dtype, **opts):
    ctx = P.Context(0, dtype)
    for k, v in opts.items():
        ctx.set_option(k, v)
    ctx.set_problems(insts)
    ctx.build_coupling()
    return ctx


@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
@pytest.mark.parametrize("R", [3, 8, 16])
def test_tc_step_field_accuracy(gpu, O, backend, R):
    """fp32 contraction on tcgen05 (symmetric fp16 hi/lo tiles, N > 512): local
    field within 2e-5 (relative to the field's scale) of the fp64 oracle; the
    CUDA-core fp32 kernel is held to the same bound."""
    insts = [O.gen_instance(640, 0.6, 0.2, 0.01, 3), O.gen_instance(640, 0.4, 0.1, 0.01, 4)]
    probs = _probs(O, insts)
    B, N = 2, 640
    rng = np.random.default_rng(R)
    Rs = rng.normal(size=(B, R, N))
    c = rng.normal(scale=0.5, size=(B, R, N))
    e = np.abs(rng.normal(size=(B, R, N))) + 0.1
    hp = gpu.baseline_params()
    out = {}
    for tc in (1, 0):
        ctx = _ctx_opts(gpu, insts, "f32", tensor_cores=tc)
        out[tc] = ctx.mfz_step(R, backend, hp, 0.37, 0.83, Rs, c, e)
        ctx.close()
    ohp = O.baseline_params()
    for b in range(B):
        for r in range(R):
            if backend == "mfz-bn":
                h = probs[b].local_field_bn(Rs[b, r], (c[b, r] > 0).astype(np.int32), ohp.tau)
            else:
                h = probs[b].local_field_cn(Rs[b, r], c[b, r], ohp.tau)
            scale = np.max(np.abs(h))
            err_tc = np.max(np.abs(out[1]["h"][b, r] - h)) / scale
            err_cc = np.max(np.abs(out[0]["h"][b, r] - h)) / scale
            assert err_tc < 2e-5, (err_tc, err_cc)
            assert err_cc < 2e-5, (err_tc, err_cc)


def test_tc_refit_and_score_accuracy(gpu, O):
    insts = [O.gen_instance(640, 0.6, 0.2, 0.01, 7)]
    p = _probs(O, insts)[0]
    R = 16
    rng = np.random.default_rng(2)
    sigma = (rng.random((1, R, 640)) < 0.3).astype(np.int32)
    Rp = rng.normal(size=(1, R, 640))
    ctx = _ctx_opts(gpu, insts, "f32", tensor_cores=1)
    out = ctx.refit(R, sigma, Rp, gpu.HyperParams())
    sc = ctx.score(R, Rp, sigma, 0.05)
    ctx.close()
    for r in range(R):
        ref = p.cdp(sigma[0, r], Rp[0, r], O.CDP_JACOBI, O.HyperParams())
        assert np.max(np.abs(out[0, r] - ref)) < 1e-4 * max(1.0, np.max(np.abs(ref)))
        keep = sigma[0, r] == 0  # untouched (fp32-rounded on upload)
        assert np.array_equal(out[0, r][keep], Rp[0, r][keep].astype(np.float32))
        obj = p.objective_at(Rp[0, r], sigma[0, r], 0.05)
        assert math.isclose(sc["objective"][0, r], obj, rel_tol=1e-5, abs_tol=1e-6)


@pytest.mark.parametrize("N,cluster", [(600, 0), (256, 0), (256, 1)])
def test_tc_solve_matches_fp64_supports(gpu, O, N, cluster):
    """fp32 solve vs the fp64 oracle (stated short-schedule fp32 tolerance:
    >= 90% identical supports, mean |dRMSE|/RMSE <= 5e-2): N=600 runs the
    tcgen05 symmetric path, N=256 the CUDA-core grid kernel (cluster=0) or the
    small-N cluster loop (cluster=1)."""
    insts = [O.gen_instance(N, 0.5, 0.1, 0.01, s) for s in range(1, 5)]
    R = 4
    hp = O.baseline_params(velo=9)
    seeds = np.array([[O.mix_seed(i.seed, 1 + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    ctx = _ctx_opts(gpu, insts, "f32", tensor_cores=1, cluster_loop=cluster)
    res = ctx.solve(R, "mfz-bn", gpu.baseline_params(velo=9), seeds)
    ctx.close()
    same, rel = 0, []
    for b, inst in enumerate(insts):
        for r in range(R):
            ref = _oracle_solve(O, inst, O.MFZ_BN, hp, int(seeds[b, r]))
            same += np.array_equal(res["sigma"][b, r], ref["sigma"])
            g = O.rmse(res["R"][b, r], res["sigma"][b, r], inst.x_true, inst.xi_true)
            rel.append(abs(g - ref["final_rmse"]) / ref["final_rmse"])
    assert same >= 0.9 * len(insts) * R, same
    assert np.mean(rel) <= 5e-2


def test_solve_matches_reference_literal_order(gpu, O):
    """fp64 GPU solve vs the oracle in the reference's own coupling form
    (matrix-free A^T(A w), orchestrator.cpp:86-88): identical supports and
    RMSE within 1e-12 relative on config-0 instances (4 seeds)."""
    for s in range(4):
        inst = O.gen_instance(500, 0.6, 0.2, 0.01, s)
        hp = O.baseline_params()
        seed = O.mix_seed(s, 1)
        ref = O.Problem(inst, O.LITERAL).alternating_minimize(O.MFZ_BN, hp, O.Rng(seed))
        ctx = _ctx(gpu, [inst])
        res = ctx.solve(1, "mfz-bn", gpu.baseline_params(), [seed])
        ctx.close()
        assert np.array_equal(res["sigma"][0, 0], ref["sigma"])
        g = O.rmse(res["R"][0, 0], res["sigma"][0, 0], inst.x_true, inst.xi_true)
        assert math.isclose(g, ref["final_rmse"], rel_tol=1e-12)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_row_sharded_context_world1(gpu, O, dtype):
    """The row-sharded context (padded 128-row slices, NCCL communicator) at
    world size 1 reproduces the plain context: bitwise in fp64."""
    insts = [O.gen_instance(300, 0.6, 0.2, 0.01, s) for s in (5, 6)]
    R = 3
    hp = gpu.baseline_params(velo=3, n_steps=300)
    seeds = np.array([[O.mix_seed(i.seed, 1 + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    plain = _ctx(gpu, insts, dtype)
    a = plain.solve(R, "mfz-bn", hp, seeds)
    plain.close()
    sh = gpu.Context(0, dtype, shard=(1, 0, gpu.nccl_unique_id()))
    sh.set_problems(insts)
    sh.build_coupling()
    b = sh.solve(R, "mfz-bn", hp, seeds)
    sh.close()
    if dtype == "f64":
        assert np.array_equal(a["R"], b["R"]) and np.array_equal(a["sigma"], b["sigma"])
    else:
        assert (a["sigma"] == b["sigma"]).mean() > 0.99


def test_phase_grid_mixed_M_bitwise(gpu, O):
    """Config-2 style batch: instances of different M (alpha) in one context,
    seeded in instance_grid order; every trajectory bitwise equal to its own
    fp64 oracle trial."""
    from paper_2405_00366_b200 import workloads as W
    grid = [g for g in W.config2_grid(trials=1)][::7][:4]  # 4 cells, alphas differ
    insts = [O.gen_instance(128, al, a, nu, s) for al, a, nu, s in grid]
    assert len({i.M for i in insts}) > 1
    R = 2
    hp = O.baseline_params(velo=2, n_steps=250)
    seeds = np.array([[O.mix_seed(i.seed, 1 + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    ctx = _ctx(gpu, insts)
    res = ctx.solve(R, "mfz-bn", gpu.baseline_params(velo=2, n_steps=250), seeds)
    ctx.close()
    for b, inst in enumerate(insts):
        for r in range(R):
            ref = _oracle_solve(O, inst, O.MFZ_BN, hp, int(seeds[b, r]))
            assert np.array_equal(res["R"][b, r], ref["R"])
            assert np.array_equal(res["sigma"][b, r], ref["sigma"])


@pytest.mark.parametrize("N,cluster", [(600, 0), (256, 1)])
def test_tc_cn_mode_and_track_best(gpu, O, N, cluster):
    """fp32 paths (tcgen05 symmetric at N=600, cluster loop at N=256),
    continuous-field mode with track_best."""
    insts = [O.gen_instance(N, 0.5, 0.1, 0.01, s) for s in (11, 12)]
    R = 4
    hp = O.baseline_params(velo=5)
    seeds = np.array([[O.mix_seed(i.seed, 0 + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    ctx = _ctx_opts(gpu, insts, "f32", tensor_cores=1, cluster_loop=cluster)
    res = ctx.solve(R, "mfz-cn", gpu.baseline_params(velo=5), seeds, track_best=True)
    ctx.close()
    same = 0
    for b, inst in enumerate(insts):
        for r in range(R):
            ref = _oracle_solve(O, inst, O.MFZ_CN, hp, int(seeds[b, r]), track_best=True)
            same += np.array_equal(res["sigma"][b, r], ref["sigma"])
    assert same >= 0.9 * len(insts) * R


def test_solve_config0_reference_literal_schedule_bitwise(gpu, O):
    """SURVEY §8(d) "c0-ref" control: config 0's instance with the reference's OWN
    schedule and defaults (HyperParams(), types.hpp:77-96: sigmoid pump p_thr 1,
    d 0.4, dt 0.02, velo 51 -> 52 alternations x 1000 steps, Jacobi refit), no
    builder extension: fp64 GPU solve bitwise equal to the oracle."""
    inst = O.gen_instance(500, 0.6, 0.2, 0.01, 0)
    hp = O.HyperParams()
    seed = O.mix_seed(0, 1)
    ref = _oracle_solve(O, inst, O.MFZ_BN, hp, seed)
    ctx = _ctx(gpu, [inst])
    res = ctx.solve(1, "mfz-bn", gpu.HyperParams(), [seed])
    assert not ref["failed"] and res["fail_alt"][0, 0] == -1
    assert res["n_hist"][0, 0] == len(ref["history"]) == 52
    assert np.array_equal(res["sigma"][0, 0], ref["sigma"])
    assert np.array_equal(res["R"][0, 0], ref["R"])
    for h, g in zip(ref["history"], res["history"][0, 0]):
        assert g["eta"] == h["eta"] and g["support"] == h["support"] and g["min_e"] == h["min_e"]
        assert math.isclose(g["rmse"], h["rmse"], rel_tol=TOL_SCALAR)
    ctx.close()
