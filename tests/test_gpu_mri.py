"""Matrix-free MRI transform chain on the GPU (csrc/mri_kernels.cuh) against
the numpy oracle of mri.cpp (oracle/mri.py, pinned by tests/test_oracle_mri.py).

The GPU chain is fp32 (shared-memory FFTs); stated tolerances: the operator
(G columns, hz, diag, G w) within 2e-5 of the largest magnitude of the
compared quantity, the local field within 2e-5 of its scale, and solves:
supports identical on >= 90 % of replicas, mean relative RMSE difference
<= 5e-2 vs the fp64 oracle solve (same bar as the dense fp32 path)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 2e-5


@pytest.fixture(scope="module")
def Mr():
    from oracle import mri
    return mri


def _ctx(P, img, mask, gamma, x=None):
    ctx = P.Context(0, "f32")
    ctx.set_mri_problem(img, mask, gamma, x)
    ctx.build_coupling()
    return ctx


@pytest.mark.parametrize("H,W,M,gamma", [(16, 16, 100, 1e-4), (8, 32, 90, 0.0),
                                         (32, 32, 400, 1e-3)])
def test_operator_matches_oracle(gpu, Mr, H, W, M, gamma):
    """assemble_operators (mri.cpp:327-343): every column G e_r, hz and diag."""
    img = Mr.phantom_image(H, W)
    mask = Mr.make_mask(H, W, M, 11)
    J, hz, t = Mr.assemble_operators(img, mask, gamma)
    with _ctx(gpu, img, mask, gamma) as ctx:
        G, ghz, gD = ctx.get_coupling(0)
    s = np.max(np.abs(J))
    assert np.max(np.abs(G - J)) <= TOL * s
    assert np.max(np.abs(ghz - hz)) <= TOL * np.max(np.abs(hz))
    assert np.max(np.abs(gD - t.diag)) <= TOL * np.max(np.abs(t.diag))


def test_full_sampling_identity_form(gpu, Mr):
    """test_mri.cpp:145-162 on the GPU: with every k-space sample and gamma = 0
    the form is the identity and hz is the target's own transform."""
    target, _ = Mr.sparsify_wavelet(Mr.phantom_image(16, 16), 0.1)
    with _ctx(gpu, target, np.arange(256), 0.0) as ctx:
        G, hz, D = ctx.get_coupling(0)
    assert np.max(np.abs(G - np.eye(256))) < 1e-5
    assert np.max(np.abs(hz - Mr.vec_image(Mr.haar2_forward(target)))) < 1e-5
    assert np.max(np.abs(D - 1.0)) < 1e-5


@pytest.mark.parametrize("size", [64, 128])
def test_step_field_matches_oracle(gpu, O, Mr, size):
    """One fused MFZ step (BN) at up to the config-3 image size: h = (sqrt(tau)/2)
    (D w - G w + hz) with G applied matrix-free, 16 replicas (D from the GPU,
    checked against the oracle's diag at 64 x 64)."""
    img, coeffs = Mr.sparsify_wavelet(Mr.phantom_image(size, size), 0.1)
    mask = Mr.make_mask(size, size, int(0.4 * size * size), 5)
    t = Mr.MriTransform(img, mask, 1e-4)
    rng = np.random.default_rng(2)
    R, N = 16, size * size
    Rs = rng.normal(size=(1, R, N)) * (rng.random((1, R, N)) < 0.2)
    c = rng.normal(scale=0.5, size=(1, R, N))
    with _ctx(gpu, img, mask, 1e-4, coeffs) as ctx:
        out = ctx.mfz_step(R, "mfz-bn", gpu.HyperParams(), 0.3, 0.9, Rs, c, np.ones((1, R, N)))
        _, ghz, D = ctx.get_coupling(0, gram=False)
    assert np.max(np.abs(ghz - t.hz)) <= TOL * np.max(np.abs(t.hz))
    if size == 64:
        assert np.max(np.abs(D - t.diag)) <= TOL * np.max(np.abs(t.diag))
    for r in (0, 7, R - 1):
        w = Rs[0, r] * (c[0, r] > 0)
        h = 0.5 * (D * w - t.apply_full(w) + t.hz)
        err = np.max(np.abs(out["h"][0, r] - h)) / np.max(np.abs(h))
        assert err < TOL, err


def test_full_sampling_recovers_sparse_image(gpu, Mr):
    """test_mri.cpp:286-306 on the GPU (fp32): full sampling, gamma 0, K = 1,
    velo 3, flat eta 0.1, CG refit -> exact support of the 26 kept
    coefficients and RMSE at fp32 level."""
    target, coeffs = Mr.sparsify_wavelet(Mr.phantom_image(16, 16), 0.1)
    hp = gpu.HyperParams()
    hp.K, hp.velo, hp.eta_init, hp.eta_end = 1.0, 3, 0.1, 0.1
    with _ctx(gpu, target, np.arange(256), 0.0, coeffs) as ctx:
        res = ctx.solve(4, "mfz-bn", hp, np.array([[19, 20, 21, 22]], np.uint64))
    for r in range(4):
        assert res["fail_alt"][0, r] == -1
        assert int(res["sigma"][0, r].sum()) == 26
        H = res["history"][0, r][: res["n_hist"][0, r]]
        assert H[-1]["hamming"] == 0.0 and H[-1]["rmse"] < 1e-5


@pytest.mark.parametrize("backend", ["mfz-bn", "mfz-cn"])
def test_solve_matches_fp64_oracle(gpu, O, Mr, backend):
    """32 x 32, 40 % k-space, gamma 1e-4, BASELINE schedule shortened to 5 x 300
    steps, 8 replicas (cluster-distributed apply): the GPU fp32 solve against the
    oracle's fp64 solve of the assembled form (Problem.from_gram, CG as
    cdp_minimize_operator), binarised and continuous feedback."""
    img, coeffs = Mr.sparsify_wavelet(Mr.phantom_image(32, 32), 0.1)
    mask = Mr.make_mask(32, 32, 410, 3)
    J, hz, _ = Mr.assemble_operators(img, mask, 1e-4)
    xi = (coeffs != 0).astype(np.int32)
    R = 8
    be = O.MFZ_BN if backend == "mfz-bn" else O.MFZ_CN
    seeds = np.array([[O.mix_seed(1, be + 3 * r) for r in range(R)]], np.uint64)
    ohp = O.baseline_params(velo=4, n_steps=300)
    p = O.Problem.from_gram(J, hz, coeffs, xi)
    with _ctx(gpu, img, mask, 1e-4, coeffs) as ctx:
        res = ctx.solve(R, backend, gpu.baseline_params(velo=4, n_steps=300), seeds)
    same, drm = 0, []
    for r in range(R):
        ref = p.alternating_minimize(be, ohp, O.Rng(int(seeds[0, r])), cdp=O.CDP_CG)
        assert not ref["failed"] and res["fail_alt"][0, r] == -1
        same += np.array_equal(res["sigma"][0, r], ref["sigma"])
        g = res["history"][0, r][res["n_hist"][0, r] - 1]["rmse"]
        o = ref["history"][-1]["rmse"]
        drm.append(abs(g - o) / max(o, 1e-12))
    assert same >= 0.9 * R, same
    assert np.mean(drm) <= 5e-2, drm


def test_operator_problem_errors(gpu, Mr):
    """Jacobi on an operator problem (cdp.cpp:158-159), fp64 contexts, the
    positive-P backend and bad masks are rejected."""
    img = Mr.phantom_image(16, 16)
    mask = Mr.make_mask(16, 16, 100, 1)
    with _ctx(gpu, img, mask, 0.0) as ctx:
        with pytest.raises(gpu.ConfigError):
            ctx.refit(2, np.ones((1, 2, 256), np.int32), np.zeros((1, 2, 256)))
        with pytest.raises(gpu.ConfigError):
            ctx.solve(2, "pp", gpu.HyperParams(), np.array([[1, 2]], np.uint64))
    with gpu.Context(0, "f64") as c64:
        with pytest.raises(gpu.ConfigError):
            c64.set_mri_problem(img, mask, 0.0)
    with gpu.Context(0, "f32") as c:
        for bad in ([0, 3, 3, 9], [0, 256]):
            with pytest.raises(gpu.InputError):
                c.set_mri_problem(img, np.array(bad), 0.0)
        with pytest.raises(gpu.InputError):
            c.set_mri_problem(np.zeros((12, 16)), np.array([1, 2]), 0.0)
        with pytest.raises(gpu.InputError):  # FFT lines longer than 128
            c.set_mri_problem(np.zeros((16, 256)), np.array([1, 2]), 0.0)


def test_lasso_warm_start_matches_oracle(gpu, Mr):
    """lasso_init(t, lambda) (mri.cpp:372-377) on the GPU chain: a fixed 300
    FISTA iterations (tol 0) agree with the fp64 oracle to 1e-4 relative, and
    the reference's default stopping rule reaches the oracle's objective (the
    fp32 objective noise moves the stopping iteration, and the LASSO objective
    is flat at its optimum, so x itself is held to 5e-2)."""
    img, coeffs = Mr.sparsify_wavelet(Mr.phantom_image(32, 32), 0.1)
    mask = Mr.make_mask(32, 32, 410, 3)
    t = Mr.MriTransform(img, mask, 1e-4)
    ref = Mr.lasso_normal_form(t.apply_fit, t.hz, 3e-4, max_iters=300, tol=0.0)
    with _ctx(gpu, img, mask, 1e-4, coeffs) as ctx:
        x, it, f = ctx.mri_lasso(3e-4, 300, 0.0)
        assert it == 300
        assert np.linalg.norm(x - ref) <= 1e-4 * np.linalg.norm(ref)
        fo = 0.5 * ref @ t.apply_fit(ref) - t.hz @ ref + 3e-4 * np.abs(ref).sum()
        assert abs(f - fo) <= 1e-5 * abs(fo)
        x2, it2, f2 = ctx.mri_lasso()  # defaults: lambda 3e-4, 5000 iterations, tol 1e-8
        ref2 = Mr.lasso_init(t, 3e-4)
        f_ref2 = 0.5 * ref2 @ t.apply_fit(ref2) - t.hz @ ref2 + 3e-4 * np.abs(ref2).sum()
        assert 1 <= it2 <= 5000
        assert f2 <= f_ref2 + 1e-5 * abs(f_ref2)
        assert np.linalg.norm(x2 - ref2) <= 5e-2 * np.linalg.norm(ref2)
        # overwhelming shrinkage returns zero exactly (test_mri.cpp:250-260)
        xz, _, _ = ctx.mri_lasso(10.0 * np.max(np.abs(t.hz)), 50, 1e-8)
        assert np.max(np.abs(xz)) == 0.0
