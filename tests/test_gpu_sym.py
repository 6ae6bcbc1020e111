"""Symmetric-tile fp32 path (sym_kernels.cuh): the upper-triangle gram tiles
stored once as scaled fp16 hi/lo planes, each tile feeding G w and G^T w.

Stated fp32 tolerances: gram within
1e-6 of max |G|; local field within 2e-5 of the field scale vs the fp64
oracle; refit within 1e-4; solve supports identical on >= 90 % of the
trajectories with mean |dRMSE|/RMSE <= 5e-2.  The cross-CTA reduction runs
in a fixed order, so two runs are bitwise identical.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ctx(P, insts, **opts):
    ctx = P.Context(0, "f32")
    for k, v in opts.items():
        ctx.set_option(k, v)
    ctx.set_problems(insts)
    ctx.build_coupling()
    return ctx


@pytest.mark.parametrize("N", [513, 640, 1000])
def test_sym_gram(gpu, O, N):
    insts = [O.gen_instance(N, 0.5, 0.1, 0.01, 5), O.gen_instance(N, 0.7, 0.1, 0.01, 6)]
    ctx = _ctx(gpu, insts)
    for b, inst in enumerate(insts):
        G, hz, D = ctx.get_coupling(b)
        ref = O.Problem(inst, O.CANON).G
        assert np.max(np.abs(G - ref)) <= 1e-6 * np.max(np.abs(ref))
        assert np.array_equal(G, G.T)
    ctx.close()


@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
@pytest.mark.parametrize("R", [3, 16])
def test_sym_step_field_accuracy(gpu, O, backend, R):
    insts = [O.gen_instance(700, 0.6, 0.2, 0.01, 3), O.gen_instance(700, 0.4, 0.1, 0.01, 4)]
    probs = [O.Problem(i, O.CANON) for i in insts]
    B, N = 2, 700
    rng = np.random.default_rng(R)
    Rs = rng.normal(size=(B, R, N))
    Rs[0, 0, :50] *= 1e-4  # widely different magnitudes inside one replica
    c = rng.normal(scale=0.5, size=(B, R, N))
    e = np.abs(rng.normal(size=(B, R, N))) + 0.1
    ctx = _ctx(gpu, insts)
    out = ctx.mfz_step(R, backend, gpu.baseline_params(), 0.37, 0.83, Rs, c, e)
    ctx.close()
    ohp = O.baseline_params()
    for b in range(B):
        for r in range(R):
            if backend == "mfz-bn":
                h = probs[b].local_field_bn(Rs[b, r], (c[b, r] > 0).astype(np.int32), ohp.tau)
            else:
                h = probs[b].local_field_cn(Rs[b, r], c[b, r], ohp.tau)
            err = np.max(np.abs(out["h"][b, r] - h)) / np.max(np.abs(h))
            assert err < 2e-5, (b, r, err)


def test_sym_refit_cg_and_score(gpu, O):
    insts = [O.gen_instance(600, 0.6, 0.2, 0.01, 7)]
    p = O.Problem(insts[0], O.CANON)
    R = 16
    rng = np.random.default_rng(2)
    sigma = (rng.random((1, R, 600)) < 0.2).astype(np.int32)
    Rp = rng.normal(size=(1, R, 600))
    ctx = _ctx(gpu, insts)
    out = ctx.refit(R, sigma, Rp, gpu.HyperParams())
    outc = ctx.refit(R, sigma, Rp, gpu.HyperParams(), cdp="cg")
    sc = ctx.score(R, Rp, sigma, 0.05)
    ctx.close()
    for r in range(R):
        for res, m in ((out, O.CDP_JACOBI), (outc, O.CDP_CG)):
            ref = p.cdp(sigma[0, r], Rp[0, r], m, O.HyperParams())
            assert np.max(np.abs(res[0, r] - ref)) < 1e-4 * max(1.0, np.max(np.abs(ref)))
        obj = p.objective_at(Rp[0, r], sigma[0, r], 0.05)
        assert math.isclose(sc["objective"][0, r], obj, rel_tol=1e-5, abs_tol=1e-6)


@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
def test_sym_solve_matches_fp64_and_is_deterministic(gpu, O, backend):
    insts = [O.gen_instance(600, 0.5, 0.1, 0.01, s) for s in range(1, 4)]
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


def test_sym_matches_cuda_core_kernel(gpu, O):
    """tensor_cores=0 (fp32 CUDA-core FFMA kernel) and the symmetric tcgen05 path
    agree to fp32 accuracy."""
    insts = [O.gen_instance(800, 0.5, 0.1, 0.01, 9)]
    R = 8
    rng = np.random.default_rng(4)
    Rs = rng.normal(size=(1, R, 800))
    c = rng.normal(scale=0.5, size=(1, R, 800))
    e = np.ones((1, R, 800))
    outs = []
    for tc in (1, 0):
        ctx = _ctx(gpu, insts, tensor_cores=tc)
        outs.append(ctx.mfz_step(R, "mfz-cn", gpu.baseline_params(), 0.4, 0.9, Rs, c, e)["h"])
        ctx.close()
    assert np.max(np.abs(outs[0] - outs[1])) <= 4e-5 * np.max(np.abs(outs[1]))


@pytest.mark.parametrize("N", [1100, 2000, 8200])
def test_sym_gram_on_tensor_cores(gpu, O, N):
    """gram_tc=1 (forced below its N >= 8192 default): the large-N gram on tcgen05
    from fp16 hi/lo splits of A (gram_tc_kernels.cuh, no library GEMM) matches the
    oracle gram within 1e-6 of max |G| and drives the same local field."""
    insts = [O.gen_instance(N, 0.5, 0.1, 0.01, 21), O.gen_instance(N, 0.6, 0.1, 0.01, 22)]
    ctx = _ctx(gpu, insts, gram_tc=1)
    for b, inst in enumerate(insts):
        G, hz, D = ctx.get_coupling(b)
        A = np.asfortranarray(inst.A)
        ref = A.T @ A
        assert np.max(np.abs(G - ref)) <= 1e-6 * np.max(np.abs(ref))
    R = 8
    rng = np.random.default_rng(9)
    Rs = rng.normal(size=(2, R, N))
    c = rng.normal(scale=0.5, size=(2, R, N))
    out = ctx.mfz_step(R, "mfz-bn", gpu.baseline_params(), 0.4, 0.9, Rs, c, np.ones((2, R, N)))
    ctx.close()
    if N <= 2000:
        p = O.Problem(insts[1], O.CANON)
        h = p.local_field_bn(Rs[1, 3], (c[1, 3] > 0).astype(np.int32), 1.0)
        assert np.max(np.abs(out["h"][1, 3] - h)) < 2e-5 * np.max(np.abs(h))


@pytest.mark.parametrize("cdp", ["jacobi", "cg"])
def test_tile_sharded_context_world1_bitwise(gpu, O, cdp):
    """Tile sharding (sharded contexts on the symmetric path): the per-rank slot
    sums, all-reduced (identity at world 1), feed the same update in the same
    slot order, so a world-1 tile-sharded solve equals the plain symmetric
    context bit for bit (N = 1100 ragged, 2 instances x 16 replicas)."""
    insts = [O.gen_instance(1100, 0.5, 0.1, 0.01, s) for s in (21, 22)]
    R = 16
    hp = gpu.baseline_params(velo=2, n_steps=150)
    seeds = np.array([[O.mix_seed(i.seed, 1 + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    with gpu.Context(0, "f32") as plain:
        plain.set_option("refit_compact", 0)  # tile-sharded contexts refit uncompacted
        plain.set_problems(insts)
        plain.build_coupling()
        a = plain.solve(R, "mfz-bn", hp, seeds, cdp=cdp)
    with gpu.Context(0, "f32", shard=(1, 0, gpu.nccl_unique_id())) as sh:
        sh.set_problems(insts)
        sh.build_coupling()
        b = sh.solve(R, "mfz-bn", hp, seeds, cdp=cdp)
    assert np.array_equal(a["sigma"], b["sigma"])
    assert np.array_equal(a["R"], b["R"])
    assert np.array_equal(a["history"]["hamiltonian"], b["history"]["hamiltonian"])


def test_sym_phase_grid_mixed_M_matches_fp64(gpu, O):
    """A config-2-style mini phase grid on the symmetric path: instances of one
    context differ in M (alpha 0.3..0.9) and K, the gram tiles are built per run
    of equal M, items of all instances share one LPT schedule; supports agree
    with the fp64 oracle on >= 90 % of trajectories (fp32 stated tolerance)."""
    cells = [(0.3, 0.05), (0.5, 0.1), (0.7, 0.2), (0.9, 0.3), (0.4, 0.15)]
    insts = [O.gen_instance(700, al, a, 0.01, 100 + k) for k, (al, a) in enumerate(cells)]
    R = 8
    hp = O.baseline_params(velo=5, n_steps=400)
    seeds = np.array([[O.mix_seed(i.seed, 1 + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    ctx = _ctx(gpu, insts)
    res = ctx.solve(R, "mfz-bn", gpu.baseline_params(velo=5, n_steps=400), seeds)
    ctx.close()
    same, rel = 0, []
    for b, inst in enumerate(insts):
        for r in range(R):
            ref = O.Problem(inst, O.CANON).alternating_minimize(O.MFZ_BN, hp,
                                                                O.Rng(int(seeds[b, r])))
            same += np.array_equal(res["sigma"][b, r], ref["sigma"])
            g = O.rmse(res["R"][b, r], res["sigma"][b, r], inst.x_true, inst.xi_true)
            rel.append(abs(g - ref["final_rmse"]) / max(ref["final_rmse"], 1e-12))
    assert same >= 0.9 * len(insts) * R, same
    assert np.mean(rel) <= 5e-2, np.mean(rel)


def test_two_live_contexts_load_identically(gpu):
    """Regression (r01h): a second live context's zero fill of its instance
    buffer ran on the legacy stream and could land after the uploads on the
    context's non-blocking stream (bench e2e at config 2: 1212 of 1344
    instances read back with diag(G) = 0).  Every context must see its own
    upload: mixed-M instances, diag and hz bitwise equal across contexts."""
    insts = [gpu.gen_instance(2000, alpha, 0.1, 0.01, s)
             for s, alpha in enumerate((0.3, 0.9, 0.6, 0.9) * 16, start=1)]
    ctxs = []
    try:
        for _ in range(3):
            c = gpu.Context(0, "f32")
            c.set_problems(insts)
            c.build_coupling()
            ctxs.append(c)
        for b in (0, 1, 37, 63):
            ref = insts[b].A
            d_host = (np.asarray(ref) ** 2).sum(axis=0)
            outs = [c.get_coupling(b, gram=False) for c in ctxs]
            for _, hz, D in outs:
                assert np.max(np.abs(D - d_host)) <= 1e-5 * np.max(d_host)
                assert np.array_equal(hz, outs[0][1]) and np.array_equal(D, outs[0][2])
    finally:
        for c in ctxs:
            c.close()


def test_compacted_refit_matches_full_refit(gpu, O):
    """The compacted Jacobi refit (union of the replicas' supports, cmp_kernels.cuh)
    against the full-gram refit in the same solve: identical supports after the
    CIM calls that follow need not hold (fp32), but one refit from the same
    state agrees to fp32 accuracy and leaves every inactive R bitwise."""
    insts = [O.gen_instance(1100, 0.5, 0.1, 0.01, s) for s in (31, 32)]
    R = 16
    hp = gpu.baseline_params(velo=1, n_steps=200)
    seeds = np.array([[O.mix_seed(i.seed, 1 + 3 * r) for r in range(R)] for i in insts],
                     np.uint64)
    out = {}
    for cmp in (0, 1):
        with gpu.Context(0, "f32") as ctx:
            ctx.set_option("refit_compact", cmp)
            ctx.set_problems(insts)
            ctx.build_coupling()
            # velo=1: alternation 0's CIM call + refit are identical up to the refit
            out[cmp] = ctx.solve(R, "mfz-bn", gpu.baseline_params(velo=1, n_steps=200), seeds)
    h0, h1 = out[0]["history"], out[1]["history"]
    # alternation 0 shares its CIM call (same supports); its refit differs only in rounding
    assert np.array_equal(h0["support"][:, :, 0], h1["support"][:, :, 0])
    assert np.allclose(h0["rmse"][:, :, 0], h1["rmse"][:, :, 0], rtol=1e-4)
    for b, inst in enumerate(insts):
        for r in range(R):
            assert abs(out[1]["history"][b, r][0]["rmse"] - out[0]["history"][b, r][0]["rmse"]) \
                <= 1e-4 * out[0]["history"][b, r][0]["rmse"]


def test_timeline_stamps(gpu, O):
    """Option `timeline` (measurement aid, cimcs_get_timeline): after a CIM call every
    tile CTA and every update CTA of the last launch pair has stamped entry <= past its
    PDL wait <= exit, the update CTAs exit after the tile CTAs' last items, and tile
    CTA 0's per-tile stamps are ordered (accumulator free <= landed <= issued)."""
    N, B, R = 1100, 3, 16
    insts = [O.gen_instance(N, 0.5, 0.1, 0.01, s) for s in range(41, 41 + B)]
    ctx = gpu.Context(0, "f32")
    ctx.set_option("timeline", 1)
    ctx.set_problems(insts)
    ctx.build_coupling()
    rng = np.random.default_rng(3)
    Rs = np.abs(rng.normal(size=(B, R, N))) * 0.1
    c0 = rng.normal(scale=1e-2, size=(B, R, N))
    ctx.run_cim(R, "mfz-bn", gpu.baseline_params(velo=1, n_steps=20), 0.5, Rs, c0)
    tl = ctx.timeline().astype(np.int64)
    ctx.close()
    nRB = -(-N // 128)
    tile = tl[:256]
    tile = tile[tile[:, 0] > 0]
    upd = tl[256:256 + B * nRB]
    assert len(tile) >= 1 and np.all(upd[:, 0] > 0)
    assert np.all(tile[:, 0] <= tile[:, 1]) and np.all(tile[:, 1] <= tile[:, 2])
    assert np.all(upd[:, 0] <= upd[:, 1]) and np.all(upd[:, 1] <= upd[:, 2])
    assert upd[:, 1].min() >= tile[:, 2].max()  # fp32: the update waits for the whole tile grid
    per = tl[8192:8192 + 128]
    n = int((per[:, 1] > 0).sum())
    assert n >= 1
    assert np.all(per[:n, 0] <= per[:n, 1]) and np.all(per[:n, 1] <= per[:n, 2])


def test_compacted_refit_dense_unions(gpu, O):
    """Regression (found by tools/shape_fuzz.py): with dense support unions the compacted
    problem's 128-row padding exceeds ldN = round_up(N, 32) (N = 577: 5 blocks = 640 > 608)
    and the union index list was read out of bounds; the refit now falls back to the full
    sweeps there.  12 instances x 16 replicas, 5 alternations: runs, finite, and close to
    the uncompacted refit."""
    N, B, R = 577, 12, 16
    insts = [O.gen_instance(N, 0.55, 0.25, 0.01, 1000 + s) for s in range(B)]
    seeds = np.array([[O.mix_seed(i.seed, 1 + 3 * r) for r in range(R)] for i in insts], np.uint64)
    hp = gpu.baseline_params(velo=4, n_steps=134)
    res = []
    for cmp in (1, 0):
        ctx = _ctx(gpu, insts, refit_compact=cmp)
        res.append(ctx.solve(R, "mfz-bn", hp, seeds))
        ctx.close()
    assert np.all(np.isfinite(res[0]["R"]))
    same = np.all(res[0]["sigma"] == res[1]["sigma"], axis=2)
    assert same.mean() >= 0.9
    assert np.max(np.abs(res[0]["R"][same] - res[1]["R"][same])) < 1e-3
