"""GPU conjugate-gradient refit (cdp="cg", cdp.cpp:66-105) against the oracle.

fp64: bitwise against the oracle's ORC_CANON CG (G*p in the canonical
contraction order, dot products summed left to right over the active set),
both from the graph path (conditional WHILE node) and the host-polled path.
fp32: the CG recursion stays in fp64 while G*p runs on the tensor cores;
stated tolerance 1e-4 of the solution scale.
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


@pytest.fixture(scope="module")
def insts(O):
    return [O.gen_instance(200, 0.6, 0.2, 0.01, 3), O.gen_instance(200, 0.4, 0.1, 0.01, 4)]


def _supports(B, R, N, seed, density=0.2):
    rng = np.random.default_rng(seed)
    sigma = (rng.random((B, R, N)) < density).astype(np.int32)
    sigma[0, 0] = 0  # empty support: R_prev returned unchanged
    return sigma, rng.normal(size=(B, R, N))


def test_cg_refit_bitwise(gpu, O, insts):
    R = 3
    B, N = len(insts), insts[0].N
    sigma, Rp = _supports(B, R, N, 11)
    ctx = _ctx(gpu, insts)
    out, its = ctx.refit(R, sigma, Rp, gpu.HyperParams(), cdp="cg", return_iterations=True)
    ctx.close()
    for b in range(B):
        p = O.Problem(insts[b], O.CANON)
        for r in range(R):
            ref = p.cdp(sigma[b, r], Rp[b, r], O.CDP_CG, O.HyperParams())
            assert np.array_equal(out[b, r], ref), (b, r)
    assert np.array_equal(out[0, 0], Rp[0, 0]) and its[0, 0] == 0
    assert np.all(its[sigma.sum(axis=2) > 0] > 0)


def test_cg_iteration_cap_and_tolerance(gpu, O, insts):
    """cg_max_iters caps the loop; a loose cg_tol stops earlier (cdp.cpp:77)."""
    R = 2
    B, N = len(insts), insts[0].N
    sigma, Rp = _supports(B, R, N, 12, density=0.35)
    ctx = _ctx(gpu, insts)
    for hp_kw in ({"cg_max_iters": 3}, {"cg_tol": 1e-3}, {"cg_max_iters": 0}):
        out, its = ctx.refit(R, sigma, Rp, gpu.HyperParams(**hp_kw), cdp="cg",
                             return_iterations=True)
        for b in range(B):
            p = O.Problem(insts[b], O.CANON)
            for r in range(R):
                ref = p.cdp(sigma[b, r], Rp[b, r], O.CDP_CG, O.HyperParams(**hp_kw))
                assert np.array_equal(out[b, r], ref), (hp_kw, b, r)
        if "cg_max_iters" in hp_kw:
            assert its.max() <= hp_kw["cg_max_iters"]
    ctx.close()


def test_cg_host_loop_matches_graph(gpu, O, insts):
    """use_graphs=0 (host-polled loop) equals the conditional-node graph."""
    R = 4
    B, N = len(insts), insts[0].N
    hp = gpu.baseline_params(velo=3, n_steps=200)
    seeds = np.array([[O.mix_seed(i.seed, 1 + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    a = _ctx(gpu, insts)
    ra = a.solve(R, "mfz-bn", hp, seeds, cdp="cg")
    a.close()
    b = _ctx(gpu, insts, use_graphs=0)
    rb = b.solve(R, "mfz-bn", hp, seeds, cdp="cg")
    b.close()
    assert np.array_equal(ra["R"], rb["R"]) and np.array_equal(ra["sigma"], rb["sigma"])


@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
def test_cg_solve_bitwise(gpu, O, backend):
    """alternating_minimize with cdp=cg: every trajectory equals the oracle's."""
    insts = [O.gen_instance(160, 0.5, 0.1, 0.01, s) for s in (1, 2)]
    R = 2
    hp = O.baseline_params(velo=4, n_steps=250)
    be = O.MFZ_BN if backend == "mfz-bn" else O.MFZ_CN
    seeds = np.array([[O.mix_seed(i.seed, be + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    ctx = _ctx(gpu, insts)
    res = ctx.solve(R, backend, gpu.baseline_params(velo=4, n_steps=250), seeds, cdp="cg")
    ctx.close()
    for b, inst in enumerate(insts):
        p = O.Problem(inst, O.CANON)
        for r in range(R):
            ref = p.alternating_minimize(be, hp, O.Rng(int(seeds[b, r])), cdp=O.CDP_CG)
            assert np.array_equal(res["R"][b, r], ref["R"]), (b, r)
            assert np.array_equal(res["sigma"][b, r], ref["sigma"])


def test_cg_python_solve(gpu, O):
    """cimcs.solve(..., cdp="cg") mirrors the reference binding (module.cpp:127-141)."""
    inst = gpu.gen_instance(40, 0.7, 0.2, 0.01, 9)
    res = gpu.solve(inst, backend="mfz-bn", params=gpu.HyperParams(velo=5), seed=3, cdp="cg")
    ref = O.solve(O.gen_instance(40, 0.7, 0.2, 0.01, 9), "mfz-bn", O.HyperParams(velo=5),
                  seed=3, cdp="cg")
    assert np.array_equal(res["R"], ref["R"]) and np.array_equal(res["sigma"], ref["sigma"])


def test_cg_fp32_tensor_cores(gpu, O):
    insts = [O.gen_instance(640, 0.6, 0.2, 0.01, 7)]
    p = O.Problem(insts[0], O.CANON)
    R = 16
    sigma, Rp = _supports(1, R, 640, 13)
    ctx = _ctx(gpu, insts, "f32", tensor_cores=1)
    out, its = ctx.refit(R, sigma, Rp, gpu.HyperParams(), cdp="cg", return_iterations=True)
    ctx.close()
    assert its.max() < 10000  # the fp64 recursion converges on the fp16 hi/lo operator
    for r in range(R):
        ref = p.cdp(sigma[0, r], Rp[0, r], O.CDP_CG, O.HyperParams())
        assert np.max(np.abs(out[0, r] - ref)) < 1e-4 * max(1.0, np.max(np.abs(ref)))
        keep = sigma[0, r] == 0
        assert np.array_equal(out[0, r][keep], Rp[0, r][keep].astype(np.float32))


def test_cg_on_world1_sharded_context(gpu, O):
    """A row-sharded context of world 1 (no collective) runs CG; world > 1
    contexts reject cdp=cg with ConfigError (the all-gathered dots are not built)."""
    import paper_2405_00366_b200 as P
    uid = P.nccl_unique_id()
    inst = O.gen_instance(64, 0.5, 0.2, 0.01, 1)
    ctx = gpu.Context(0, "f64", shard=(1, 0, uid))
    ctx.set_problems([inst])
    ctx.build_coupling()
    sigma, Rp = _supports(1, 1, 64, 4, density=0.4)
    sigma[0, 0, :8] = 1
    out = ctx.refit(1, sigma, Rp, cdp="cg")
    ctx.close()
    ref = O.Problem(inst, O.CANON).cdp(sigma[0, 0], Rp[0, 0], O.CDP_CG, O.HyperParams())
    assert np.array_equal(out[0, 0], ref)
