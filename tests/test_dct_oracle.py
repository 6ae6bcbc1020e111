"""CPU checks of config 3's dense restatement (oracle/dct_chain.py), the checker of
the matrix-free DCT o Haar^-1 chain, and of the chain's host-side inputs."""
import numpy as np


def test_dct_matrix_orthonormal():
    from oracle import dct_chain
    C = dct_chain.dct_matrix(128)
    assert np.allclose(C @ C.T, np.eye(128), atol=1e-13)


def test_rows_orthonormal_and_chain_identity():
    """A = S C2 Haar_L^-1 has orthonormal rows (A A^T = I); G w equals the chain
    Haar C^T (mask o C Haar^-1 w C^T) C evaluated with numpy transforms."""
    from oracle import dct_chain, mri
    rng = np.random.default_rng(0)
    n, L = 128, 3
    f = rng.choice(n * n, size=300, replace=False)
    A = dct_chain.assemble_A(n, L, f)
    assert np.allclose(A @ A.T, np.eye(f.size), atol=1e-12)
    C = dct_chain.dct_matrix(n)
    mask = np.zeros(n * n)
    mask[f] = 1
    w = rng.normal(size=n * n)
    X = mri.haar2_inverse(w.reshape(n, n), L)
    Y = (C @ X @ C.T) * mask.reshape(n, n)
    chain = mri.haar2_forward(C.T @ Y @ C, L).reshape(-1)
    assert np.allclose(chain, dct_chain.apply_G(A, w), atol=1e-12)
    assert np.allclose(dct_chain.diag_G(A), np.sum(A * A, axis=0))


def test_haar_levels_match_workloads():
    from oracle import mri
    from paper_2405_00366_b200 import workloads
    x = np.random.default_rng(1).normal(size=(128, 128))
    for L in (1, 2, 3):
        assert np.array_equal(mri.haar2_forward(x, L), workloads.haar2(x, L))
        assert np.allclose(workloads.ihaar2(workloads.haar2(x, L), L), x, atol=1e-13)
    assert np.array_equal(mri.haar2_forward(x), mri.haar2_forward(x, None))


def test_config3_chain_inputs_match_dense_instance():
    """config3_chain draws the same phantom / frequencies / noise as config3: its
    y is the dense instance's y up to evaluation order."""
    from oracle import dct_chain
    from paper_2405_00366_b200 import workloads
    n, L, f, y, w = workloads.config3_chain()
    assert (n, L, f.size) == (128, 3, 6554)
    A = dct_chain.assemble_A(n, L, f[:256])
    rng = np.random.Generator(np.random.PCG64(3))
    img = workloads.ellipse_phantom(n, 10, rng)
    assert np.array_equal(w, workloads.haar2(img, L).reshape(-1))
    noise = y[:256] - A @ w  # y = A w + N(0, 0.005^2)
    assert 0.003 < np.std(noise) < 0.008 and abs(np.mean(noise)) < 0.002
