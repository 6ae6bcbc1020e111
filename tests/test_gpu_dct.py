"""BASELINE config 3 as the matrix-free DCT o Haar^-1 chain (csrc/dct_kernels.cuh)
against the dense fp64 operator assembled by oracle/dct_chain.py (A row by row
from the Haar-transformed DCT basis images, the dense config-3 path's matrix).

The chain is fp32 (3xTF32 tensor-core products); stated tolerances, the same as
the DFT chain's (tests/test_gpu_mri.py): hz, diag and G w within 2e-5 of the
largest magnitude of the compared quantity, the local field within 2e-5 of its
scale; one damped Jacobi refit (100 sweeps) within 1e-4 of the fp64 refit's
scale.  Whole solves are compared with the dense fp32 path on the same
instance (both fp32: the quality metrics, not trajectories)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 2e-5


@pytest.fixture(scope="module")
def Dc():
    from oracle import dct_chain
    return dct_chain


@pytest.fixture(scope="module")
def chain3():
    """config 3's chain inputs with a reduced sample (M = 2000) and its dense A"""
    from oracle import dct_chain
    from paper_2405_00366_b200 import workloads
    n, L, f, y, w = workloads.config3_chain()
    f, y = f[:2000], y[:2000]
    return n, L, f, y, w, dct_chain.assemble_A(n, L, f)


def _ctx(P, n, L, f, y, w=None):
    ctx = P.Context(0, "f32")
    ctx.set_dct_problem(n, L, f, y, w)
    ctx.build_coupling()
    return ctx


def test_hz_and_diag(gpu, Dc, chain3):
    n, L, f, y, w, A = chain3
    with _ctx(gpu, n, L, f, y) as ctx:
        _, hz, D = ctx.get_coupling(0, gram=False)
    hz_ref, D_ref = A.T @ y, Dc.diag_G(A)
    assert np.max(np.abs(hz - hz_ref)) <= TOL * np.max(np.abs(hz_ref))
    assert np.max(np.abs(D - D_ref)) <= TOL * np.max(np.abs(D_ref))


@pytest.mark.parametrize("levels", [1, 2, 3])
def test_step_field(gpu, Dc, levels):
    """One fused MFZ step (BN), 16 replicas: h = (sqrt(tau)/2)(D w - G w + hz)
    with G w matrix-free, checked against the dense fp64 operator."""
    rng = np.random.default_rng(levels)
    n, N = 128, 128 * 128
    f = rng.choice(N, size=1500, replace=False).astype(np.int32)
    y = rng.normal(size=f.size)
    A = Dc.assemble_A(n, levels, f)
    R = 16
    Rs = rng.normal(size=(1, R, N)) * (rng.random((1, R, N)) < 0.2)
    c = rng.normal(scale=0.5, size=(1, R, N))
    with _ctx(gpu, n, levels, f, y) as ctx:
        out = ctx.mfz_step(R, "mfz-bn", gpu.HyperParams(), 0.3, 0.9, Rs, c, np.ones((1, R, N)))
    D, hz = Dc.diag_G(A), A.T @ y
    for r in range(R):
        wv = Rs[0, r] * (c[0, r] > 0)
        h = 0.5 * (D * wv - Dc.apply_G(A, wv) + hz)
        err = np.max(np.abs(out["h"][0, r] - h)) / np.max(np.abs(h))
        assert err < TOL, (r, err)


def test_columns_small_sample(gpu, Dc):
    """get_coupling's G (the chain on every basis vector) for a 1-level chain
    and a handful of frequencies: every entry within 2e-5 of max |G|."""
    rng = np.random.default_rng(5)
    n = 128
    f = rng.choice(n * n, size=64, replace=False).astype(np.int32)
    A = Dc.assemble_A(n, 1, f)
    with _ctx(gpu, n, 1, f, np.ones(f.size)) as ctx:
        G, _, _ = ctx.get_coupling(0)
    J = A.T @ A
    assert np.max(np.abs(G - J)) <= TOL * np.max(np.abs(J))


def test_jacobi_refit(gpu, O, chain3):
    """cdp_minimize's damped Jacobi (cdp.cpp:48-64) on the chain vs the oracle's
    fp64 refit on the assembled G (orc_problem_init_gram)."""
    n, L, f, y, w, A = chain3
    G = A.T @ A
    p = O.Problem.from_gram(G, A.T @ y)
    R, N = 4, n * n
    rng = np.random.default_rng(9)
    sigma = (rng.random((1, R, N)) < 0.05).astype(np.int32)
    Rp = rng.normal(size=(1, R, N))
    with _ctx(gpu, n, L, f, y) as ctx:
        out = ctx.refit(R, sigma, Rp, gpu.HyperParams())
    for r in range(R):
        ref = p.cdp(sigma[0, r], Rp[0, r], O.CDP_JACOBI, O.HyperParams())
        on = sigma[0, r] != 0
        # inactive R kept bitwise (in the fp32 state)
        assert np.array_equal(out[0, r][~on], Rp[0, r][~on].astype(np.float32))
        assert np.max(np.abs(out[0, r] - ref)) <= 1e-4 * np.max(np.abs(ref[on]))


def test_score_matches_oracle(gpu, O, chain3):
    n, L, f, y, w, A = chain3
    G = A.T @ A
    p = O.Problem.from_gram(G, A.T @ y, w, (w != 0).astype(np.int32))
    R, N = 2, n * n
    rng = np.random.default_rng(4)
    sigma = (rng.random((1, R, N)) < 0.1).astype(np.int32)
    Rp = rng.normal(size=(1, R, N))
    with _ctx(gpu, n, L, f, y, w) as ctx:
        sc = ctx.score(R, Rp, sigma, 0.05)
    for r in range(R):
        obj = p.objective_at(Rp[0, r], sigma[0, r], 0.05)
        assert abs(sc["objective"][0, r] - obj) <= 1e-4 * abs(obj)


def test_solve_matches_dense_path(gpu):
    """Config 3 at full size (M = 6554), 16 replicas, 2 alternations x 200
    steps: the chain and the dense fp32 path (tcgen05 gram + symmetric tiles) on
    the same instance.  Both are fp32, so the bar is on quality: per-replica
    RMSE vs the truth within 5e-2 relative on >= 14 of 16 replicas, supports
    identical on >= 12 of 16 after the first alternation."""
    from paper_2405_00366_b200 import workloads
    insts, R, _, _ = workloads.config3()
    n, L, f, y, w = workloads.config3_chain()
    hp = gpu.baseline_params(velo=1, n_steps=200)
    seeds = np.array([[gpu.mix_seed(3, 1 + 3 * r) for r in range(R)]], np.uint64)
    with _ctx(gpu, n, L, f, insts[0].y, w) as ctx:
        a = ctx.solve(R, "mfz-bn", hp, seeds)
    with gpu.Context(0, "f32") as ctx:
        ctx.set_problems(insts)
        ctx.build_coupling()
        b = ctx.solve(R, "mfz-bn", hp, seeds)
    ha, hb = a["history"][0], b["history"][0]
    same = sum(ha[r][0]["support"] == hb[r][0]["support"] for r in range(R))
    ra = np.array([ha[r][-1]["rmse"] for r in range(R)])
    rb = np.array([hb[r][-1]["rmse"] for r in range(R)])
    close = int(np.sum(np.abs(ra - rb) <= 5e-2 * rb))
    print("dct vs dense: identical first supports", same, "rmse close", close, ra[:4], rb[:4])
    assert same >= 12 and close >= 14


def test_input_errors(gpu):
    f = np.arange(10, dtype=np.int32)
    with gpu.Context(0, "f32") as ctx:
        with pytest.raises(gpu.InputError):
            ctx.set_dct_problem(64, 3, f, np.ones(10))
        with pytest.raises(gpu.InputError):
            ctx.set_dct_problem(128, 4, f, np.ones(10))
        with pytest.raises(gpu.InputError):
            ctx.set_dct_problem(128, 3, np.array([1, 1], np.int32), np.ones(2))
        ctx.set_dct_problem(128, 2, f, np.ones(10))
        ctx.build_coupling()
        with pytest.raises(gpu.ConfigError):
            ctx.mri_lasso()
    with gpu.Context(0, "f64") as ctx:
        with pytest.raises(gpu.ConfigError):
            ctx.set_dct_problem(128, 3, f, np.ones(10))
