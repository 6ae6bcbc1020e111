"""fp64 DMMA symmetric-tile path (sym64_kernels.cuh) against the oracle, BITWISE.

Unsharded fp64 contexts with N > 512 store the gram as upper-triangle 64 x 64
fp64 tiles and contract on the FP64 tensor cores (mma.sync m8n8k4, which the
B200 evaluates as a sequential fma chain, tools/peaks_probe.cu).  Their order
is the oracle's ORC_CANON with (nseg, gran) = (ceil(N/512), 512), reported by
cimcs_canon_order; every quantity below is compared bit for bit with the oracle
in that order, except reduced scalars (objective, rmse: 1e-12 relative).
"""
import math

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


def _probs(O, insts, order):
    return [O.Problem(i, O.CANON, *order) for i in insts]


@pytest.mark.parametrize("N", [600, 1100, 2000])
def test_order_and_gram_tiles(gpu, O, N):
    insts = [O.gen_instance(N, 0.5, 0.1, 0.01, 5)]
    ctx = _ctx(gpu, insts)
    order = ctx.canon_order()
    assert order == (-(-N // 512), 512)
    G, hz, D = ctx.get_coupling(0)
    p = _probs(O, insts, order)[0]
    assert np.array_equal(G, p.G) and np.array_equal(hz, p.hz) and np.array_equal(D, p.gram_diag)
    ctx.close()
    ctx = _ctx(gpu, insts, sym64=0)  # the CUDA-core grid kernel keeps the (8, 8) order
    assert ctx.canon_order() == (8, 8)
    ctx.close()


@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
@pytest.mark.parametrize("N,R", [(600, 3), (1100, 16), (2000, 8)])
def test_single_step_bitwise(gpu, O, backend, N, R):
    insts = [O.gen_instance(N, 0.6, 0.2, 0.01, 3), O.gen_instance(N, 0.4, 0.1, 0.01, 4)]
    ctx = _ctx(gpu, insts)
    probs = _probs(O, insts, ctx.canon_order())
    B = len(insts)
    rng = np.random.default_rng(R)
    Rs = rng.normal(size=(B, R, N))
    c = rng.normal(scale=0.5, size=(B, R, N))
    e = np.abs(rng.normal(size=(B, R, N))) + 0.1
    hp, ghp = O.baseline_params(), gpu.baseline_params()
    out = ctx.mfz_step(R, backend, ghp, 0.37, 0.83, Rs, c, e)
    for b in range(B):
        for r in range(R):
            if backend == "mfz-bn":
                h = probs[b].local_field_bn(Rs[b, r], (c[b, r] > 0).astype(np.int32), hp.tau)
            else:
                h = probs[b].local_field_cn(Rs[b, r], c[b, r], hp.tau)
            co, eo = O.mfz_step(c[b, r], e[b, r], 0.83, hp, 0.37, Rs[b, r], h)
            assert np.array_equal(out["h"][b, r], h)
            assert np.array_equal(out["c"][b, r], co)
            assert np.array_equal(out["e"][b, r], eo)
    ctx.close()


@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
def test_run_cim_bitwise(gpu, O, backend):
    """A whole CIM call (300 steps) from identical c0 / R."""
    insts = [O.gen_instance(700, 0.5, 0.1, 0.01, s) for s in (1, 2)]
    R, N = 5, 700
    ctx = _ctx(gpu, insts)
    probs = _probs(O, insts, ctx.canon_order())
    hp = O.baseline_params(n_steps=300)
    seeds = [[O.mix_seed(inst.seed, 1 + 3 * r) for r in range(R)] for inst in insts]
    c0 = np.zeros((2, R, N))
    for b in range(2):
        for r in range(R):
            g = O.Rng(seeds[b][r])
            c0[b, r] = [0.01 * g.gauss() for _ in range(N)]
    Rs = np.stack([np.stack([p.hz] * R) for p in probs])
    out = ctx.run_cim(R, backend, gpu.baseline_params(n_steps=300), 0.6, Rs, c0)
    be = O.BACKENDS[backend]
    for b in range(2):
        for r in range(R):
            ref = probs[b].run_mfz(Rs[b, r], hp, 0.6, be, O.Rng(seeds[b][r]))
            assert np.array_equal(out["c"][b, r], ref["c"])
            assert np.array_equal(out["e"][b, r], ref["e"])
            assert np.array_equal(out["sigma"][b, r], ref["sigma"])
            assert out["min_e"][b, r] == ref["min_e"]
    ctx.close()


@pytest.mark.parametrize("cdp", ["jacobi", "cg"])
def test_refit_bitwise(gpu, O, cdp):
    insts = [O.gen_instance(900, 0.5, 0.1, 0.01, 8)]
    R = 8
    ctx = _ctx(gpu, insts)
    p = _probs(O, insts, ctx.canon_order())[0]
    rng = np.random.default_rng(2)
    sigma = (rng.random((1, R, 900)) < 0.25).astype(np.int32)
    Rp = rng.normal(size=(1, R, 900))
    out = ctx.refit(R, sigma, Rp, gpu.HyperParams(), cdp=cdp)
    sc = ctx.score(R, Rp, sigma, 0.05)
    ctx.close()
    m = O.CDP_JACOBI if cdp == "jacobi" else O.CDP_CG
    for r in range(R):
        ref = p.cdp(sigma[0, r], Rp[0, r], m, O.HyperParams())
        assert np.array_equal(out[0, r], ref)
        obj = p.objective_at(Rp[0, r], sigma[0, r], 0.05)
        assert math.isclose(sc["objective"][0, r], obj, rel_tol=1e-12, abs_tol=1e-14)


@pytest.mark.parametrize("cmp", [0, 1])
def test_compacted_refit_bitwise(gpu, O, cmp):
    """The segment-preserving compacted Jacobi refit (cmp_kernels.cuh, cmp64) is
    bitwise the oracle's: N=1700 (4 segments of 512, the last ragged), supports
    chosen so that segment 1 is empty in every instance (dropped), the union
    widths differ per instance and per segment, and one instance has a single
    active spin."""
    N, R = 1700, 8
    insts = [O.gen_instance(N, 0.5, 0.1, 0.01, s) for s in (41, 42, 43)]
    ctx = _ctx(gpu, insts, refit_compact=cmp)
    order = ctx.canon_order()
    assert order == (4, 512)
    rng = np.random.default_rng(7)
    sigma = np.zeros((3, R, N), np.int32)
    sigma[0, :, :512] = rng.random((R, 512)) < 0.3
    sigma[0, :, 1024:1536] = rng.random((R, 512)) < 0.05
    sigma[1, :, 1024:] = rng.random((R, N - 1024)) < 0.4
    sigma[2, 3, 1600] = 1
    Rp = rng.normal(size=(3, R, N))
    out = ctx.refit(R, sigma, Rp, gpu.HyperParams())
    ctx.close()
    for b, inst in enumerate(insts):
        p = O.Problem(inst, O.CANON, *order)
        for r in range(R):
            ref = p.cdp(sigma[b, r], Rp[b, r], O.CDP_JACOBI, O.HyperParams())
            assert np.array_equal(out[b, r], ref), (b, r)


def test_compacted_refit_solve_matches_full(gpu, O):
    """Whole solves with the compacted refit on and off: bitwise equal."""
    insts = [O.gen_instance(1300, 0.5, 0.1, 0.01, s) for s in (51, 52)]
    R = 8
    seeds = np.array([[O.mix_seed(i.seed, 1 + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    res = {}
    for cmp in (0, 1):
        ctx = _ctx(gpu, insts, refit_compact=cmp)
        res[cmp] = ctx.solve(R, "mfz-bn", gpu.baseline_params(velo=3, n_steps=200), seeds)
        ctx.close()
    assert np.array_equal(res[0]["R"], res[1]["R"])
    assert np.array_equal(res[0]["sigma"], res[1]["sigma"])
    for b in range(2):
        for r in range(R):
            for h0, h1 in zip(res[0]["history"][b, r], res[1]["history"][b, r]):
                assert h0 == h1


@pytest.mark.parametrize("backend,track_best", [("mfz-bn", False), ("mfz-cn", True)])
def test_solve_bitwise(gpu, O, backend, track_best):
    """Whole alternating solves: 2 instances x 3 replicas (NR padded to 8), N=600."""
    insts = [O.gen_instance(600, 0.5, 0.1, 0.01, s) for s in (11, 12)]
    R = 3
    be = O.BACKENDS[backend]
    seeds = np.array([[O.mix_seed(i.seed, be + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    ctx = _ctx(gpu, insts)
    order = ctx.canon_order()
    res = ctx.solve(R, backend, gpu.baseline_params(velo=3, n_steps=300), seeds,
                    track_best=track_best)
    ctx.close()
    hp = O.baseline_params(velo=3, n_steps=300)
    for b, inst in enumerate(insts):
        p = O.Problem(inst, O.CANON, *order)
        for r in range(R):
            ref = p.alternating_minimize(be, hp, O.Rng(int(seeds[b, r])), track_best=track_best)
            assert np.array_equal(res["R"][b, r], ref["R"])
            assert np.array_equal(res["sigma"][b, r], ref["sigma"])
            for h, g in zip(ref["history"], res["history"][b, r]):
                assert g["support"] == h["support"] and g["min_e"] == h["min_e"]
                assert g["median_e"] == h["median_e"]
                assert math.isclose(g["hamiltonian"], h["hamiltonian"], rel_tol=1e-12,
                                    abs_tol=1e-14)


def test_solve_config1_shape_bitwise(gpu, O):
    """BASELINE config-1 shape (N=2000, M=1000), 16 replicas, 2 x 200 steps:
    two replicas checked bitwise against the oracle."""
    insts = [O.gen_instance(2000, 0.5, 0.1, 0.01, 1)]
    R = 16
    seeds = np.array([[O.mix_seed(1, 1 + 3 * r) for r in range(R)]], np.uint64)
    ctx = _ctx(gpu, insts)
    order = ctx.canon_order()
    res = ctx.solve(R, "mfz-bn", gpu.baseline_params(velo=1, n_steps=200), seeds)
    ctx.close()
    p = O.Problem(insts[0], O.CANON, *order)
    for r in (0, 15):
        ref = p.alternating_minimize(O.MFZ_BN, O.baseline_params(velo=1, n_steps=200),
                                     O.Rng(int(seeds[0, r])))
        assert np.array_equal(res["R"][0, r], ref["R"])
        assert np.array_equal(res["sigma"][0, r], ref["sigma"])



def test_divergence_on_sym64_path(gpu, O):
    """A blown-up trajectory on the DMMA path fails at the same alternation and
    spin as the oracle (solver_mfz.cpp:75-85, orchestrator.cpp:222-227)."""
    inst = O.gen_instance(600, 0.6, 0.2, 0.01, 5)
    seed = O.mix_seed(5, 1)
    ctx = _ctx(gpu, [inst])
    order = ctx.canon_order()
    res = ctx.solve(1, "mfz-bn", gpu.HyperParams(velo=2, dt=5.0, n_steps=50), [seed])
    ctx.close()
    ref = O.Problem(inst, O.CANON, *order).alternating_minimize(
        O.MFZ_BN, O.HyperParams(velo=2, dt=5.0, n_steps=50), O.Rng(seed))
    assert ref["failed"] and res["fail_alt"][0, 0] == ref["fail_alternation"]
    assert res["fail_index"][0, 0] == ref["fail_index"]


@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
def test_item_flags_do_not_change_results(gpu, O, backend):
    """Item flags (option overlap_update: an instance's update CTAs run under the
    DMMA tile kernel as soon as its items are published) only change WHEN an update
    CTA runs: 12 instances x 16 replicas (more items than one wave of update CTAs
    can hold resident), N = 1100 (3 segments, 6 items per instance), whole solves --
    R, sigma and the histories are bitwise equal with the flags off and on, and
    equal to the oracle for one trajectory.  (Also the regression case of the compacted
    refit's dense-union fallback: with 12 x 16 supports the per-segment widths round up
    to 512 + 512 + 128 = 1152 rows > ldN = 1120, which used to overrun the state.)"""
    insts = [O.gen_instance(1100, 0.5, 0.1, 0.01, s) for s in range(21, 33)]
    R = 16
    be = O.BACKENDS[backend]
    seeds = np.array([[O.mix_seed(i.seed, be + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    res = []
    for ov in (0, 1):
        ctx = _ctx(gpu, insts, overlap_update=ov)
        order = ctx.canon_order()
        res.append(ctx.solve(R, backend, gpu.baseline_params(velo=2, n_steps=150), seeds))
        ctx.close()
    assert np.array_equal(res[0]["R"], res[1]["R"])
    assert np.array_equal(res[0]["sigma"], res[1]["sigma"])
    assert np.array_equal(res[0]["fail_alt"], res[1]["fail_alt"])
    for b in range(len(insts)):
        for r in range(R):
            for h0, h1 in zip(res[0]["history"][b, r], res[1]["history"][b, r]):
                assert h0 == h1
    ref = O.Problem(insts[5], O.CANON, *order).alternating_minimize(
        be, O.baseline_params(velo=2, n_steps=150), O.Rng(int(seeds[5, 7])))
    assert np.array_equal(res[1]["R"][5, 7], ref["R"])
    assert np.array_equal(res[1]["sigma"][5, 7], ref["sigma"])


def test_update_runs_under_the_tile_kernel(gpu, O):
    """The defining property of the item flags, from the per-CTA %globaltimer stamps
    (option timeline): with the flags on, update CTAs of early instances pass their
    wait while tile CTAs are still working (40 instances x 16 replicas, N = 1537: 400
    items on 148 CTAs, so a CTA's first item -- an early instance's -- ends well before the
    launch does; with a shape whose largest item spans the whole launch, e.g. N = 1100,
    every instance completes at the end and there is nothing to overlap); with the flags
    off every update CTA waits for the whole tile grid.  Stamps are ordered entry <= past
    the wait <= exit either way."""
    N, B, R = 1537, 40, 16
    insts = [O.gen_instance(N, 0.5, 0.1, 0.01, 100 + s) for s in range(B)]
    rng = np.random.default_rng(5)
    Rs = np.abs(rng.normal(size=(B, R, N))) * 0.1
    c0 = rng.normal(scale=1e-2, size=(B, R, N))
    first_pass, last_tile = {}, {}
    for ov in (0, 1):
        ctx = gpu.Context(0, "f64")
        ctx.set_option("timeline", 1)
        ctx.set_option("overlap_update", ov)
        ctx.set_problems(insts)
        ctx.build_coupling()
        ctx.run_cim(R, "mfz-bn", gpu.baseline_params(velo=1, n_steps=12), 0.5, Rs, c0)
        tl = ctx.timeline().astype(np.int64)
        ctx.close()
        tile = tl[:256]
        tile = tile[tile[:, 0] > 0]
        nupd = 2 * B * (-(-N // 64))  # step modes: two 32-row CTAs per 64-row block
        upd = tl[256:256 + nupd]
        assert len(tile) == 148 and np.all(upd[:, 0] > 0)
        assert np.all(upd[:, 0] <= upd[:, 1]) and np.all(upd[:, 1] <= upd[:, 2])
        first_pass[ov], last_tile[ov] = upd[:, 1].min(), tile[:, 2].max()
    assert first_pass[0] >= last_tile[0]  # no flags: after the whole tile grid
    assert first_pass[1] < last_tile[1] - 5000  # flags: >= 5 us before the last tile item
