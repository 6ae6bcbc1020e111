"""Small-N cluster loop (cluster_kernels.cuh): a whole CIM call / Jacobi refit
in one thread-block-cluster launch with G register-resident.

fp64: bitwise against the oracle (ORC_CANON) at the eligibility edges
(N = 1, 33, 256, 500, 512) and bitwise against the per-step grid kernels
(cluster_loop=0), including divergence, mixed M, CN mode and N = 513 (grid
path).  fp32 CUDA-core: cluster == grid bitwise (same canonical FFMA chains).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ctx(P, insts, dtype="f64", **opts):
    ctx = P.Context(0, dtype)
    for k, v in opts.items():
        ctx.set_option(k, v)
    ctx.set_problems(insts)
    ctx.build_coupling()
    return ctx


def _c0(O, insts, R, salt=1):
    N = insts[0].N
    seeds = [[O.mix_seed(i.seed, salt + 3 * r) for r in range(R)] for i in insts]
    c0 = np.zeros((len(insts), R, N))
    for b in range(len(insts)):
        for r in range(R):
            g = O.Rng(seeds[b][r])
            c0[b, r] = [0.01 * g.gauss() for _ in range(N)]
    return seeds, c0


@pytest.mark.parametrize("N", [1, 33, 256, 512])
@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
def test_cluster_run_cim_bitwise(gpu, O, N, backend):
    insts = [O.gen_instance(N, 0.6, 0.2, 0.01, 5), O.gen_instance(N, 0.5, 0.2, 0.01, 6)]
    R = 3
    probs = [O.Problem(i, O.CANON) for i in insts]
    seeds, c0 = _c0(O, insts, R)
    Rs = np.stack([np.stack([p.hz] * R) for p in probs])
    hp = O.baseline_params(n_steps=300)
    ctx = _ctx(gpu, insts)
    out = ctx.run_cim(R, backend, gpu.baseline_params(n_steps=300), 0.5, Rs, c0)
    ctx.close()
    be = O.MFZ_BN if backend == "mfz-bn" else O.MFZ_CN
    for b in range(len(insts)):
        for r in range(R):
            ref = probs[b].run_mfz(Rs[b, r], hp, 0.5, be, O.Rng(seeds[b][r]))
            assert np.array_equal(out["c"][b, r], ref["c"]), (b, r)
            assert np.array_equal(out["e"][b, r], ref["e"])
            assert np.array_equal(out["sigma"][b, r], ref["sigma"])
            assert out["min_e"][b, r] == ref["min_e"]


@pytest.mark.parametrize("N", [33, 500])
def test_cluster_refit_bitwise(gpu, O, N):
    insts = [O.gen_instance(N, 0.6, 0.2, 0.01, 8)]
    p = O.Problem(insts[0], O.CANON)
    R = 4
    rng = np.random.default_rng(3)
    sigma = (rng.random((1, R, N)) < 0.3).astype(np.int32)
    Rp = rng.normal(size=(1, R, N))
    ctx = _ctx(gpu, insts)
    out = ctx.refit(R, sigma, Rp, gpu.HyperParams())
    ctx.close()
    for r in range(R):
        assert np.array_equal(out[0, r], p.cdp(sigma[0, r], Rp[0, r], O.CDP_JACOBI,
                                               O.HyperParams()))


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
def test_cluster_equals_grid_solve(gpu, O, dtype, backend):
    """Whole solves, mixed M, 3 instances x 4 replicas: cluster loop == grid kernels."""
    insts = [O.gen_instance(300, a, 0.15, 0.01, s) for s, a in ((1, 0.4), (2, 0.6), (3, 0.8))]
    R = 4
    hp = gpu.baseline_params(velo=5, n_steps=400)
    be = 1 if backend == "mfz-bn" else 0
    seeds = np.array([[O.mix_seed(i.seed, be + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    out = []
    for cl in (1, 0):
        ctx = _ctx(gpu, insts, dtype, cluster_loop=cl, tensor_cores=0)
        out.append(ctx.solve(R, backend, hp, seeds, track_best=True))
        ctx.close()
    a, b = out
    for k in ("R", "sigma", "n_hist", "fail_alt"):
        assert np.array_equal(a[k], b[k]), k
    for f in ("eta", "support", "min_e", "median_e", "hamming"):
        assert np.array_equal(a["history"][f], b["history"][f]), f


def test_cluster_divergence_matches_grid(gpu, O):
    """dt = 5 diverges in alternation 0: same fail step, index and frozen state."""
    insts = [O.gen_instance(100, 0.8, 0.3, 0.0, 2)]
    R = 2
    seeds, c0 = _c0(O, insts, R, salt=0)
    p = O.Problem(insts[0], O.CANON)
    Rs = np.stack([np.stack([p.hz] * R)])
    outs = []
    for cl in (1, 0):
        ctx = _ctx(gpu, insts, cluster_loop=cl)
        outs.append(ctx.run_cim(R, "mfz-cn", gpu.HyperParams(dt=5.0), 0.5, Rs, c0))
        ctx.close()
    assert (outs[0]["fail_index"] >= 0).all()
    for k in ("c", "e", "fail_index", "min_e", "sigma"):
        assert np.array_equal(outs[0][k], outs[1][k], equal_nan=True), k
    sol = []
    for cl in (1, 0):
        ctx = _ctx(gpu, insts, cluster_loop=cl)
        sol.append(ctx.solve(R, "mfz-cn", gpu.HyperParams(dt=5.0, velo=2),
                             np.array([seeds[0]], np.uint64)))
        ctx.close()
    assert np.array_equal(sol[0]["fail_alt"], sol[1]["fail_alt"])
    assert np.array_equal(sol[0]["fail_index"], sol[1]["fail_index"])
    ref = O.solve(O.gen_instance(100, 0.8, 0.3, 0.0, 2), "mfz-cn", O.HyperParams(dt=5.0, velo=2),
                  seed=int(seeds[0][0]))
    assert ref["failed"] and sol[0]["fail_alt"][0, 0] == ref["fail_alternation"]


def test_grid_path_beyond_cluster_limit(gpu, O):
    """N = 513 is outside the cluster loop: the fp64 DMMA symmetric path (in its
    own canonical order, cimcs_canon_order) still matches the oracle."""
    inst = O.gen_instance(513, 0.5, 0.2, 0.01, 4)
    hp = O.baseline_params(velo=2, n_steps=200)
    seed = O.mix_seed(4, 1)
    ctx = _ctx(gpu, [inst])
    order = ctx.canon_order()
    res = ctx.solve(1, "mfz-bn", gpu.baseline_params(velo=2, n_steps=200), [seed])
    ctx.close()
    ref = O.Problem(inst, O.CANON, *order).alternating_minimize(O.MFZ_BN, hp, O.Rng(seed))
    assert np.array_equal(res["R"][0, 0], ref["R"])
    assert np.array_equal(res["sigma"][0, 0], ref["sigma"])
