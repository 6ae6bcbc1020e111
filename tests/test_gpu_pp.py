"""GPU Positive-P backend (cimcs_run_pp / solve(backend="pp")) against the oracle.

fp64: bitwise against the oracle's ORC_CANON run_pp / alternating_minimize
(same unit normals: each trajectory's reference stream is drawn on the host and
streamed to the device in 64-step chunks, so n_steps around the chunk edges is
tested) -- on the CUDA-core kernels (N <= 512, sym64 = 0) and on the DMMA
symmetric-tile path.  fp32 (CUDA cores and the tcgen05 symmetric-tile path): stated
tolerance on the measured amplitude.
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


@pytest.mark.parametrize("n_steps", [1, 64, 65, 200])
def test_run_pp_bitwise(gpu, O, n_steps):
    insts = [O.gen_instance(150, 0.6, 0.2, 0.01, 5), O.gen_instance(150, 0.5, 0.2, 0.01, 6)]
    R = 3
    seeds = np.array([[O.mix_seed(i.seed, 2 + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    hp = O.HyperParams(n_steps=n_steps, g2=0.01, K=0.5)
    ctx = _ctx(gpu, insts)
    probs = [O.Problem(i, O.CANON) for i in insts]
    Rs = np.stack([np.stack([p.hz] * R) for p in probs])
    out = ctx.run_pp(R, gpu.HyperParams(n_steps=n_steps, g2=0.01, K=0.5), 0.5, Rs, seeds)
    ctx.close()
    for b in range(2):
        for r in range(R):
            ref = probs[b].run_pp(Rs[b, r], hp, 0.5, O.Rng(int(seeds[b, r])))
            assert np.array_equal(out["mu"][b, r], ref["mu"]), (b, r)
            assert np.array_equal(out["e"][b, r], ref["e"])
            assert np.array_equal(out["mu_tilde"][b, r], ref["mu_tilde"])
            assert np.array_equal(out["sigma"][b, r], ref["sigma"])
            assert out["min_e"][b, r] == ref["min_e"]


def test_pp_solve_bitwise(gpu, O):
    """alternating_minimize(Backend::PositiveP): R, sigma and the history."""
    insts = [O.gen_instance(120, 0.7, 0.2, 0.01, s) for s in (1, 2)]
    R = 2
    hp = O.HyperParams(velo=3, n_steps=150, g2=0.01)
    seeds = np.array([[O.mix_seed(i.seed, 2 + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    ctx = _ctx(gpu, insts)
    res = ctx.solve(R, "pp", gpu.HyperParams(velo=3, n_steps=150, g2=0.01), seeds)
    ctx.close()
    for b, inst in enumerate(insts):
        for r in range(R):
            ref = O.Problem(inst, O.CANON).alternating_minimize(O.PP, hp, O.Rng(int(seeds[b, r])))
            assert np.array_equal(res["R"][b, r], ref["R"]), (b, r)
            assert np.array_equal(res["sigma"][b, r], ref["sigma"])
            assert res["n_hist"][b, r] == len(ref["history"])
            for g, h in zip(res["history"][b, r], ref["history"]):
                assert g["min_e"] == h["min_e"] and g["median_e"] == h["median_e"]


def test_pp_divergence_and_abort(gpu, O):
    """|mu| > mu_abort fails the trial at the same alternation and spin as the oracle."""
    inst = O.gen_instance(30, 0.8, 0.3, 0.0, 3)
    hp = O.HyperParams(velo=2, n_steps=40, mu_abort=1e-3)
    ref = O.solve(inst, "pp", hp, seed=8)
    res = gpu.solve(gpu.gen_instance(30, 0.8, 0.3, 0.0, 3), "pp",
                    gpu.HyperParams(velo=2, n_steps=40, mu_abort=1e-3), seed=8)
    assert ref["failed"] and res["failed"]
    assert res["fail_alternation"] == ref["fail_alternation"]
    assert res["fail_reason"] == f"pp: divergence at spin {ref['fail_index']}"


def test_pp_fp32_cuda_cores(gpu, O):
    insts = [O.gen_instance(300, 0.6, 0.2, 0.01, 7)]
    R = 4
    seeds = np.array([[O.mix_seed(7, 2 + 3 * r) for r in range(R)]], np.uint64)
    p = O.Problem(insts[0], O.CANON)
    Rs = np.stack([np.stack([p.hz] * R)])
    hp = O.HyperParams(n_steps=100, g2=0.01)
    ctx = _ctx(gpu, insts, "f32", tensor_cores=0)
    out = ctx.run_pp(R, gpu.HyperParams(n_steps=100, g2=0.01), 0.5, Rs, seeds)
    ctx.close()
    for r in range(R):
        ref = p.run_pp(Rs[0, r], hp, 0.5, O.Rng(int(seeds[0, r])))
        assert np.max(np.abs(out["mu_tilde"][0, r] - ref["mu_tilde"])) < 1e-4


def test_pp_on_tcgen05_context(gpu, O):
    """Positive-P on the fp32 tcgen05 symmetric-tile path (N > 512): the update kernel
    runs the same element update (pp_elem) on the tensor-core G w; measured amplitude
    within the fp32 tolerance of the oracle, and equal supports after 100 steps."""
    N = 640
    insts = [O.gen_instance(N, 0.6, 0.2, 0.01, 1), O.gen_instance(N, 0.5, 0.2, 0.01, 2)]
    R = 4
    seeds = np.array([[O.mix_seed(i.seed, 2 + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    probs = [O.Problem(i, O.CANON) for i in insts]
    Rs = np.stack([np.stack([p.hz] * R) for p in probs])
    hp = O.HyperParams(n_steps=100, g2=0.01)
    ctx = _ctx(gpu, insts, "f32")
    out = ctx.run_pp(R, gpu.HyperParams(n_steps=100, g2=0.01), 0.5, Rs, seeds)
    ctx.close()
    for b in range(2):
        for r in range(R):
            ref = probs[b].run_pp(Rs[b, r], hp, 0.5, O.Rng(int(seeds[b, r])))
            assert np.max(np.abs(out["mu_tilde"][b, r] - ref["mu_tilde"])) < 1e-4
            assert np.max(np.abs(out["e"][b, r] - ref["e"])) < 1e-4 * np.max(np.abs(ref["e"]))


@pytest.mark.parametrize("N,n_steps", [(600, 70), (1100, 130)])
def test_pp_on_dmma_path_bitwise(gpu, O, N, n_steps):
    """fp64 contexts with N > 512 run Positive-P on the DMMA symmetric-tile path (the
    default): bitwise against the oracle in that path's canonical order, chunk edges of
    the host noise stream included; with sym64=0 the CUDA-core kernel gives the (8, 8)
    order's bits."""
    insts = [O.gen_instance(N, 0.6, 0.2, 0.01, 2), O.gen_instance(N, 0.5, 0.1, 0.01, 3)]
    R = 3
    seeds = np.array([[O.mix_seed(i.seed, 2 + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    for opts in ({}, {"sym64": 0}):
        ctx = _ctx(gpu, insts, **opts)
        order = ctx.canon_order()
        assert order == ((-(-N // 512), 512) if not opts else (8, 8))
        probs = [O.Problem(i, O.CANON, *order) for i in insts]
        Rs = np.stack([np.stack([p.hz] * R) for p in probs])
        out = ctx.run_pp(R, gpu.HyperParams(n_steps=n_steps, g2=0.01), 0.5, Rs, seeds)
        ctx.close()
        for b in range(2):
            for r in range(R):
                ref = probs[b].run_pp(Rs[b, r], O.HyperParams(n_steps=n_steps, g2=0.01), 0.5,
                                      O.Rng(int(seeds[b, r])))
                assert np.array_equal(out["mu"][b, r], ref["mu"]), (opts, b, r)
                assert np.array_equal(out["e"][b, r], ref["e"])
                assert np.array_equal(out["mu_tilde"][b, r], ref["mu_tilde"])
                assert np.array_equal(out["sigma"][b, r], ref["sigma"])
                assert out["min_e"][b, r] == ref["min_e"]


def test_pp_solve_on_dmma_path_bitwise(gpu, O):
    """alternating_minimize(Backend::PositiveP) on the DMMA path: R, sigma, history."""
    insts = [O.gen_instance(600, 0.7, 0.2, 0.01, s) for s in (1, 2)]
    R = 2
    hp = O.HyperParams(velo=2, n_steps=120, g2=0.01)
    seeds = np.array([[O.mix_seed(i.seed, 2 + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    ctx = _ctx(gpu, insts)
    order = ctx.canon_order()
    res = ctx.solve(R, "pp", gpu.HyperParams(velo=2, n_steps=120, g2=0.01), seeds)
    ctx.close()
    for b, inst in enumerate(insts):
        for r in range(R):
            ref = O.Problem(inst, O.CANON, *order).alternating_minimize(
                O.PP, hp, O.Rng(int(seeds[b, r])))
            assert np.array_equal(res["R"][b, r], ref["R"]), (b, r)
            assert np.array_equal(res["sigma"][b, r], ref["sigma"])
            assert res["n_hist"][b, r] == len(ref["history"])
            for g, h in zip(res["history"][b, r], ref["history"]):
                assert g["min_e"] == h["min_e"] and g["median_e"] == h["median_e"]
