"""The numpy MRI-chain oracle (oracle/mri.py) pinned by the reference's own
known-answer tests, tests/test_mri.cpp (cited per test; the reference's FFTW
and Eigen are absent, so its tolerance-based checks are ported as they are).
CPU only."""
import math

import numpy as np
import pytest


@pytest.fixture(scope="module")
def Mr():
    from oracle import mri
    return mri


def test_flattening_row_major(Mr):
    """test_mri.cpp:13-23."""
    img = np.array([[1, 2, 3], [4, 5, 6]], float)
    v = Mr.vec_image(img)
    assert list(v) == [1, 2, 3, 4, 5, 6]
    assert np.array_equal(Mr.unvec_image(v, 2, 3), img)
    with pytest.raises(Mr.InputError):
        Mr.unvec_image(v, 2, 2)


def test_haar_orthonormal_invertible(Mr, O):
    """test_mri.cpp:54-66."""
    rng = O.Rng(33)
    for h, w in ((8, 8), (4, 8), (16, 2)):
        img = np.array([[rng.gauss() for _ in range(w)] for _ in range(h)])
        c = Mr.haar2_forward(img)
        assert np.max(np.abs(Mr.haar2_inverse(c) - img)) < 1e-12
        assert math.isclose(np.linalg.norm(c), np.linalg.norm(img), rel_tol=1e-12)
    with pytest.raises(Mr.InputError):
        Mr.haar2_forward(np.zeros((3, 4)))
    with pytest.raises(Mr.InputError):
        Mr.haar2_inverse(np.zeros((4, 6)))


def test_constants_compress(Mr):
    """test_mri.cpp:68-82."""
    c2 = Mr.haar2_forward(np.full((2, 2), 0.7))
    assert math.isclose(c2[0, 0], 1.4, rel_tol=1e-12)
    assert c2[0, 1] == c2[1, 0] == c2[1, 1] == 0.0
    c4 = Mr.haar2_forward(np.full((4, 4), 0.3))
    assert math.isclose(c4[0, 0], 1.2, rel_tol=1e-12)
    assert int(np.sum(c4 == 0.0)) == 15


def test_sparsify_count_and_lossless(Mr):
    """test_mri.cpp:84-102."""
    ph = Mr.phantom_image(64, 64)
    img, _ = Mr.sparsify_wavelet(ph, 1.0)
    assert np.max(np.abs(img - ph)) < 1e-12
    _, c = Mr.sparsify_wavelet(ph, 0.212)
    assert int(np.count_nonzero(c)) == 868 and c.size == 4096
    full = Mr.vec_image(Mr.haar2_forward(ph))
    nz = c != 0
    assert np.array_equal(c[nz], full[nz])
    for bad in (0.0, 1.5):
        with pytest.raises(Mr.InputError):
            Mr.sparsify_wavelet(ph, bad)


def test_sparsify_ties_keep_lower_index(Mr):
    """test_mri.cpp:104-122."""
    img = np.array([[1, 1, 0, 0], [1, 1, 0, 0], [0, 0, 1, 1], [0, 0, 1, 1]], float)
    F = Mr.haar2_forward(img)
    assert F[0, 0] == F[1, 1] > 0.0
    _, c = Mr.sparsify_wavelet(img, 1.0 / 16.0)
    assert int(np.count_nonzero(c)) == 1 and c[0] == F[0, 0] and c[5] == 0.0


def test_masks_sorted_unique_deterministic(Mr):
    """test_mri.cpp:124-143."""
    m = Mr.make_mask(64, 64, 1638, 3)
    assert m.size == 1638 and m.size / 4096 == 0.39990234375
    assert m[0] >= 0 and m[-1] < 4096 and np.all(np.diff(m) > 0)
    assert np.array_equal(Mr.make_mask(64, 64, 1638, 3), m)
    assert not np.array_equal(Mr.make_mask(64, 64, 1638, 4), m)
    assert list(Mr.make_mask(4, 4, 16, 1)) == list(range(16))
    for M in (17, 0):
        with pytest.raises(Mr.InputError):
            Mr.make_mask(4, 4, M, 1)


def test_full_sampling_is_identity_form(Mr, O):
    """test_mri.cpp:145-162."""
    target, _ = Mr.sparsify_wavelet(Mr.phantom_image(16, 16), 0.1)
    t = Mr.MriTransform(target, Mr.make_mask(16, 16, 256, 1), 0.0)
    assert t.N == 256
    v = O.Rng(44).gauss_vector(256)
    assert np.max(np.abs(t.apply_fit(v) - v)) < 1e-10
    assert np.max(np.abs(t.apply_full(v) - v)) < 1e-10
    coeffs = Mr.vec_image(Mr.haar2_forward(target))
    assert np.max(np.abs(t.hz - coeffs)) < 1e-10
    assert t.fit_error(coeffs) < 1e-18
    assert math.isclose(t.fit_error(np.zeros(256)), 0.5 * float(np.vdot(t.y, t.y).real),
                        rel_tol=1e-12)


def test_form_symmetric_and_psd(Mr, O):
    """test_mri.cpp:164-180."""
    t = Mr.MriTransform(Mr.phantom_image(16, 16), Mr.make_mask(16, 16, 100, 7), 1e-4)
    rng = O.Rng(45)
    for _ in range(5):
        u, v = rng.gauss_vector(256), rng.gauss_vector(256)
        assert math.isclose(u @ t.apply_full(v), v @ t.apply_full(u), rel_tol=1e-10)
        assert v @ t.apply_full(v) - v @ t.apply_fit(v) >= -1e-12
        assert v @ t.apply_fit(v) >= -1e-12


def test_assembled_matches_matrix_free(Mr, O):
    """test_mri.cpp:182-200."""
    target, mask, gamma = Mr.phantom_image(16, 16), Mr.make_mask(16, 16, 100, 11), 1e-4
    t = Mr.MriTransform(target, mask, gamma)
    J, hz, _ = Mr.assemble_operators(target, mask, gamma)
    assert np.max(np.abs(hz - t.hz)) < 1e-10
    assert np.max(np.abs(np.diag(J) - t.diag)) < 1e-10
    v = O.Rng(46).gauss_vector(256)
    assert np.max(np.abs(J @ v - t.apply_full(v))) < 1e-10


def test_transform_validates_inputs(Mr):
    """test_mri.cpp:202-219."""
    ok = Mr.phantom_image(8, 8)
    with pytest.raises(Mr.InputError):
        Mr.MriTransform(Mr.phantom_image(12, 16), Mr.make_mask(12, 16, 10, 1), 0.0)
    with pytest.raises(Mr.InputError):
        Mr.MriTransform(ok, Mr.make_mask(8, 8, 10, 1), -0.5)
    for bad in ([0, 3, 3, 9], [0, 64]):
        with pytest.raises(Mr.InputError):
            Mr.MriTransform(ok, bad, 0.0)


def test_lasso_identity_design_soft_threshold(Mr):
    """test_mri.cpp:221-229 (identity design: G = I, step 1)."""
    y = np.array([0.5, -0.3, 0.05, 0.0])
    x = Mr.lasso_normal_form(lambda v: v, y, 0.1)
    assert math.isclose(x[0], 0.4, rel_tol=1e-9) and math.isclose(x[1], -0.2, rel_tol=1e-9)
    assert x[2] == 0.0 and x[3] == 0.0


def test_lasso_zero_shrinkage_normal_equations(Mr, O):
    """test_mri.cpp:231-248."""
    rng = O.Rng(47)
    A = np.column_stack([rng.gauss_vector(8) for _ in range(5)])
    y = rng.gauss_vector(8)
    direct = np.linalg.lstsq(A, y, rcond=None)[0]
    G = A.T @ A
    x = Mr.lasso_normal_form(lambda v: G @ v, A.T @ y, 0.0, max_iters=200000, tol=1e-15,
                             step=1.0 / np.linalg.eigvalsh(G).max())
    assert np.linalg.norm(x - direct) < 1e-6 * np.linalg.norm(direct)


def test_lasso_overwhelming_shrinkage_is_zero(Mr, O):
    """test_mri.cpp:250-260."""
    rng = O.Rng(48)
    A = np.column_stack([rng.gauss_vector(6) for _ in range(4)])
    y = rng.gauss_vector(6)
    G = A.T @ A
    huge = 10.0 * np.max(np.abs(A.T @ y))
    x = Mr.lasso_normal_form(lambda v: G @ v, A.T @ y, huge,
                             step=1.0 / np.linalg.eigvalsh(G).max())
    assert np.max(np.abs(x)) == 0.0


def test_full_sampling_recovers_sparse_image(Mr, O):
    """test_mri.cpp:286-306 (the operator problem restated through its assembled
    form: Problem.from_gram, CG refit as cdp_minimize_operator forces)."""
    target, coeffs = Mr.sparsify_wavelet(Mr.phantom_image(16, 16), 0.1)
    J, hz, _ = Mr.assemble_operators(target, Mr.make_mask(16, 16, 256, 1), 0.0)
    xi = (coeffs != 0.0).astype(np.int32)
    assert int(xi.sum()) == 26
    p = O.Problem.from_gram(J, hz, coeffs, xi)
    hp = O.HyperParams()
    hp.K, hp.velo, hp.eta_init, hp.eta_end = 1.0, 3, 0.1, 0.1
    res = p.alternating_minimize(O.MFZ_BN, hp, O.Rng(19), cdp=O.CDP_CG)
    assert not res["failed"]
    assert res["history"][-1]["rmse"] < 1e-6
    assert res["history"][-1]["hamming"] == 0.0
    assert int(res["sigma"].sum()) == 26


def test_phantom_deterministic_bounded(Mr):
    """test_mri.cpp:308-318."""
    a = Mr.phantom_image(64, 64)
    assert np.array_equal(a, Mr.phantom_image(64, 64))
    assert a.min() >= 0.0 and a.max() <= 1.0 and a.max() - a.min() > 0.1
    assert Mr.phantom_image(32, 16).shape == (32, 16)
    with pytest.raises(Mr.InputError):
        Mr.phantom_image(0, 4)
