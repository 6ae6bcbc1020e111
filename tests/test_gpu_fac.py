"""Factored fp32 path (fac_kernels.cuh): G w = A^T (A w) from fp16 hi/lo tiles of
A, phase 1 (u = A w) and phase 2 (A^T u + fused update) in one cooperative
launch per step.  factored=1 forces it (auto picks it when A's tiles are fewer
than the gram triangle's and the instances fill the SMs, e.g. config 1).

Stated fp32 tolerances, the same as the symmetric path: local field within
2e-5 of the field scale vs the fp64 oracle; refit within 1e-4; objective
rel 1e-5; solve supports identical on >= 90 % of the trajectories with mean
|dRMSE|/RMSE <= 5e-2.  Every output block is summed by one task in a fixed
tile order, so two runs are bitwise identical whatever the scheduling.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ctx(P, insts, **opts):
    ctx = P.Context(0, "f32")
    opts.setdefault("factored", 1)
    for k, v in opts.items():
        ctx.set_option(k, v)
    ctx.set_problems(insts)
    ctx.build_coupling()
    return ctx


def _field(O, p, backend, Rs, c, tau):
    if backend == "mfz-bn":
        return p.local_field_bn(Rs, (c > 0).astype(np.int32), tau)
    return p.local_field_cn(Rs, c, tau)


# (N, alpha): M = round(alpha N) -- M a multiple of 128, ragged M, nRB odd
# (a 1-column last phase-2 task), nRB < 2 nMB (one column per task)
@pytest.mark.parametrize("N,alpha", [(1024, 0.25), (700, 0.3), (1300, 0.45), (600, 0.9)])
@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
def test_fac_step_field_accuracy(gpu, O, N, alpha, backend):
    insts = [O.gen_instance(N, alpha, 0.2, 0.01, 3), O.gen_instance(N, alpha, 0.1, 0.01, 4),
             O.gen_instance(N, alpha, 0.1, 0.01, 5)]
    probs = [O.Problem(i, O.CANON) for i in insts]
    B, R = 3, 16
    rng = np.random.default_rng(N)
    Rs = rng.normal(size=(B, R, N))
    Rs[0, 0, :50] *= 1e-4
    c = rng.normal(scale=0.5, size=(B, R, N))
    e = np.abs(rng.normal(size=(B, R, N))) + 0.1
    ctx = _ctx(gpu, insts)
    out = ctx.mfz_step(R, backend, gpu.baseline_params(), 0.37, 0.83, Rs, c, e)
    ctx.close()
    tau = O.baseline_params().tau
    for b in range(B):
        for r in range(R):
            h = _field(O, probs[b], backend, Rs[b, r], c[b, r], tau)
            err = np.max(np.abs(out["h"][b, r] - h)) / np.max(np.abs(h))
            assert err < 2e-5, (b, r, err)


@pytest.mark.parametrize("skew", [0, 1, 10])
def test_fac_skew_and_replicas(gpu, O, skew):
    """R = 3 (padded to 8 replica slots) and task layouts with skew 0 (phase 2
    right after phase 1: CTAs wait on the counters) give the same bits."""
    insts = [O.gen_instance(900, 0.4, 0.1, 0.01, s) for s in range(1, 6)]
    R = 3
    rng = np.random.default_rng(3)
    Rs = rng.normal(size=(5, R, 900))
    c = rng.normal(scale=0.5, size=(5, R, 900))
    e = np.ones((5, R, 900))
    ref = _ctx(gpu, insts, fac_skew=10)
    a = ref.mfz_step(R, "mfz-cn", gpu.baseline_params(), 0.4, 0.9, Rs, c, e)
    ref.close()
    ctx = _ctx(gpu, insts, fac_skew=skew)
    b = ctx.mfz_step(R, "mfz-cn", gpu.baseline_params(), 0.4, 0.9, Rs, c, e)
    ctx.close()
    for k in ("h", "c", "e"):
        assert np.array_equal(a[k], b[k])
    p = O.Problem(insts[4], O.CANON)
    h = p.local_field_cn(Rs[4, 2], c[4, 2], 1.0)
    assert np.max(np.abs(b["h"][4, 2] - h)) < 2e-5 * np.max(np.abs(h))


def test_fac_refit_cg_and_score(gpu, O):
    insts = [O.gen_instance(640, 0.3, 0.2, 0.01, 7), O.gen_instance(640, 0.3, 0.1, 0.01, 8)]
    R = 16
    rng = np.random.default_rng(2)
    sigma = (rng.random((2, R, 640)) < 0.2).astype(np.int32)
    Rp = rng.normal(size=(2, R, 640))
    ctx = _ctx(gpu, insts)
    out = ctx.refit(R, sigma, Rp, gpu.HyperParams())
    outc = ctx.refit(R, sigma, Rp, gpu.HyperParams(), cdp="cg")
    sc = ctx.score(R, Rp, sigma, 0.05)
    ctx.close()
    for b in range(2):
        p = O.Problem(insts[b], O.CANON)
        for r in range(R):
            for res, m in ((out, O.CDP_JACOBI), (outc, O.CDP_CG)):
                ref = p.cdp(sigma[b, r], Rp[b, r], m, O.HyperParams())
                assert np.max(np.abs(res[b, r] - ref)) < 1e-4 * max(1.0, np.max(np.abs(ref)))
            obj = p.objective_at(Rp[b, r], sigma[b, r], 0.05)
            assert math.isclose(sc["objective"][b, r], obj, rel_tol=1e-5, abs_tol=1e-6)


@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
def test_fac_solve_matches_fp64_and_is_deterministic(gpu, O, backend):
    insts = [O.gen_instance(600, 0.3, 0.1, 0.01, s) for s in range(1, 4)]
    R = 4
    hp = O.baseline_params(velo=7)
    be = O.MFZ_BN if backend == "mfz-bn" else O.MFZ_CN
    seeds = np.array([[O.mix_seed(i.seed, be + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    runs = []
    for _ in range(2):
        ctx = _ctx(gpu, insts)
        runs.append(ctx.solve(R, backend, gpu.baseline_params(velo=7), seeds))
        ctx.close()
    assert np.array_equal(runs[0]["R"], runs[1]["R"])
    assert np.array_equal(runs[0]["sigma"], runs[1]["sigma"])
    res = runs[0]
    same, rel = 0, []
    for b, inst in enumerate(insts):
        for r in range(R):
            ref = O.Problem(inst, O.CANON).alternating_minimize(be, hp, O.Rng(int(seeds[b, r])))
            same += np.array_equal(res["sigma"][b, r], ref["sigma"])
            g = O.rmse(res["R"][b, r], res["sigma"][b, r], inst.x_true, inst.xi_true)
            rel.append(abs(g - ref["final_rmse"]) / ref["final_rmse"])
    assert same >= 0.9 * len(insts) * R, same
    assert np.mean(rel) <= 5e-2


def test_fac_matches_symmetric_path(gpu, O):
    insts = [O.gen_instance(1000, 0.5, 0.1, 0.01, 9), O.gen_instance(1000, 0.5, 0.1, 0.01, 10)]
    R = 16
    rng = np.random.default_rng(4)
    Rs = rng.normal(size=(2, R, 1000))
    c = rng.normal(scale=0.5, size=(2, R, 1000))
    e = np.ones((2, R, 1000))
    outs = []
    for fac in (1, 0):
        ctx = _ctx(gpu, insts, factored=fac)
        outs.append(ctx.mfz_step(R, "mfz-bn", gpu.baseline_params(), 0.4, 0.9, Rs, c, e)["h"])
        ctx.close()
    assert np.max(np.abs(outs[0] - outs[1])) <= 4e-5 * np.max(np.abs(outs[1]))


def test_fac_get_coupling_and_graph_replay(gpu, O):
    """get_coupling returns the fp64 A^T A; a second solve on the same context
    (graph replay, self-reset counters) repeats the first bit for bit."""
    insts = [O.gen_instance(520, 0.4, 0.1, 0.01, 11)]
    ctx = _ctx(gpu, insts)
    G, hz, D = ctx.get_coupling(0)
    ref = O.Problem(insts[0], O.CANON)
    assert np.max(np.abs(G - ref.G)) <= 1e-12 * np.max(np.abs(ref.G))
    assert np.allclose(hz, ref.hz, rtol=0, atol=1e-6)
    R = 8
    seeds = np.array([[O.mix_seed(11, 1 + 3 * r) for r in range(R)]], np.uint64)
    hp = gpu.baseline_params(velo=2, n_steps=200)
    a = ctx.solve(R, "mfz-bn", hp, seeds)
    b = ctx.solve(R, "mfz-bn", hp, seeds)
    ctx.close()
    assert np.array_equal(a["R"], b["R"]) and np.array_equal(a["sigma"], b["sigma"])
