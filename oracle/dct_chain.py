"""ORACLE (test infrastructure only): the dense restatement of BASELINE config 3's
sensing operator, the checker of the matrix-free DCT o Haar^-1 chain
(paper_2405_00366_b200/csrc/dct_kernels.cuh).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline may use it.

Config 3 (BASELINE.json configs[3]) has no counterpart in the reference: it is
the synthetic stand-in for the paper's MRI experiment, built from the
reference's orthonormal Haar split (mri.cpp:30-48, 122-165; restated in
oracle/mri.py, pinned by the ported test_mri.cpp known answers) stopped after
L levels, and the orthonormal 2-D DCT-II:
    A[m] = Haar_L(phi_{u_m v_m}),  phi_uv = c_u c_v^T,  c_u = row u of the DCT matrix,
so A = S C2 Haar_L^-1 and G = A^T A.  Everything here is fp64 numpy and builds
A explicitly (M x N), as the dense config-3 path does.
"""
from __future__ import annotations

import math

import numpy as np

from .mri import haar2_forward


def dct_matrix(n: int) -> np.ndarray:
    """Orthonormal DCT-II: C[u][x] = sqrt((u ? 2 : 1) / n) cos(pi (2x + 1) u / (2n))."""
    u = np.arange(n)[:, None]
    x = np.arange(n)[None, :]
    C = np.cos(math.pi * (2 * x + 1) * u / (2 * n)) * math.sqrt(2.0 / n)
    C[0] /= math.sqrt(2.0)
    return C


def assemble_A(n: int, levels: int, freqs) -> np.ndarray:
    """Dense A (M x n^2): row m = Haar_L of the basis image of freqs[m] = u n + v."""
    f = np.asarray(freqs, np.int64)
    C = dct_matrix(n)
    A = np.empty((f.size, n * n))
    for s in range(0, f.size, 256):
        g = f[s:s + 256]
        phi = C[g // n][:, :, None] * C[g % n][:, None, :]
        A[s:s + g.size] = haar2_forward(phi, levels).reshape(g.size, n * n)
    return A


def apply_G(A: np.ndarray, W: np.ndarray) -> np.ndarray:
    """G W = A^T (A W) for W [N] or [N][R] (fp64)."""
    return A.T @ (A @ W)


def diag_G(A: np.ndarray) -> np.ndarray:
    return np.einsum("mi,mi->i", A, A)
