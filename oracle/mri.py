"""ORACLE (test infrastructure only): numpy restatement of the reference's
matrix-free MRI sensing chain, /root/reference/proj/src/mri.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline may use it.

A = S F Psi^T (S: k-space mask rows, F: unitary 2-D DFT, Psi: orthonormal
multi-level Haar, Mallat layout), and the quadratic form of the alternation
  G = Re(A^H A) + gamma * Psi (Dv^T Dv + Dh^T Dh) Psi^T
with Dv / Dh second differences with reflective ends.  The reference runs
FFTW (unpinned, absent here); this restatement uses numpy's FFT with the same
unitary scaling, so parity with the reference is to rounding (its own tests
compare at 1e-10, tests/test_oracle_mri.py ports them).  Function-level
citations are to mri.cpp / mri.hpp unless noted.
"""
from __future__ import annotations

import math

import numpy as np

from .oracle import Rng, round_half_away

_S = 1.0 / math.sqrt(2.0)


class InputError(ValueError):
    pass


def _pow2(v):
    return v >= 1 and (v & (v - 1)) == 0


def vec_image(img):
    """mri.cpp:86-92: row-major flattening."""
    return np.asarray(img, np.float64).reshape(-1).copy()


def unvec_image(v, H, W):
    """mri.cpp:94-101."""
    v = np.asarray(v, np.float64)
    if v.size != H * W:
        raise InputError("unvec_image: length mismatch")
    return v.reshape(H, W).copy()


def _split(v, n):
    """haar_split, mri.cpp:29-38 (first n entries of the last axis)."""
    a, b = v[..., 0:n:2].copy(), v[..., 1:n:2].copy()
    v[..., : n // 2] = (a + b) * _S
    v[..., n // 2: n] = (a - b) * _S


def _merge(v, n):
    """haar_merge, mri.cpp:40-48."""
    a, b = v[..., : n // 2].copy(), v[..., n // 2: n].copy()
    v[..., 0:n:2] = (a + b) * _S
    v[..., 1:n:2] = (a - b) * _S


def haar2_forward(img, levels=None):
    """mri.cpp:122-141: per level, rows (first w of the first h) then columns.
    `levels` stops after that many levels (BASELINE config 3's 3-level
    transform; the reference always runs to full depth)."""
    X = np.array(img, np.float64)
    H, W = X.shape[-2], X.shape[-1]
    if not (_pow2(H) and _pow2(W)):
        raise InputError("haar2_forward: dimensions must be powers of two")
    h, w = H, W
    done = 0
    while h >= 2 and w >= 2 and (levels is None or done < levels):
        done += 1
        blk = X[..., :h, :w]
        _split(blk, w)
        blkT = np.swapaxes(blk, -1, -2).copy()
        _split(blkT, h)
        X[..., :h, :w] = np.swapaxes(blkT, -1, -2)
        h //= 2
        w //= 2
    return X


def haar2_inverse(C, levels=None):
    """mri.cpp:143-165: deepest level first, columns then rows (`levels` as in
    haar2_forward)."""
    X = np.array(C, np.float64)
    H, W = X.shape
    if not (_pow2(H) and _pow2(W)):
        raise InputError("haar2_inverse: dimensions must be powers of two")
    nlev = levels
    levels = []
    h, w = H, W
    while h >= 2 and w >= 2 and (nlev is None or len(levels) < nlev):
        levels.append((h, w))
        h //= 2
        w //= 2
    for h, w in reversed(levels):
        blkT = X[:h, :w].T.copy()
        _merge(blkT, h)
        blk = blkT.T.copy()
        _merge(blk, w)
        X[:h, :w] = blk
    return X


def second_diff_cols(x):
    """mri.cpp:51-63: along columns (i varies), reflective ends."""
    x = np.asarray(x, np.float64)
    H = x.shape[0]
    out = np.zeros_like(x)
    if H == 1:
        return out
    out[0] = x[1] - x[0]
    out[1:-1] = x[:-2] - 2.0 * x[1:-1] + x[2:]
    out[H - 1] = x[H - 2] - x[H - 1]
    return out


def second_diff_rows(x):
    """mri.cpp:65."""
    return second_diff_cols(np.asarray(x).T).T


def soft_threshold(v, t):
    """mri.cpp:67-74."""
    a = np.abs(v) - t
    return np.where(a > 0.0, np.where(v > 0.0, a, -a), 0.0)


def phantom_image(H, W):
    """mri.cpp:415-437: deterministic smooth blobs + edges in [0, 1]."""
    if H < 1 or W < 1:
        raise InputError("phantom_image: dims must be >= 1")
    img = np.zeros((H, W))
    for i in range(H):
        v = (i + 0.5) / H
        for j in range(W):
            u = (j + 0.5) / W
            val = 0.08 + 0.10 * u
            val += 0.55 * math.exp(-((u - 0.35) * (u - 0.35) + (v - 0.40) * (v - 0.40)) / 0.020)
            val += 0.40 * math.exp(-((u - 0.72) * (u - 0.72) + (v - 0.68) * (v - 0.68)) / 0.008)
            if 0.55 < u < 0.88 and 0.12 < v < 0.34:
                val += 0.30
            if (u - 0.28) * (u - 0.28) + (v - 0.78) * (v - 0.78) < 0.016:
                val += 0.35
            img[i, j] = min(max(val, 0.0), 1.0)
    return img


def sparsify_wavelet(img, target):
    """mri.cpp:167-183: keep round(target * N) largest |coeff| (stable: ties keep
    the lower linear index).  Returns (image, coeffs)."""
    if not (target > 0.0) or target > 1.0:
        raise InputError("sparsify_wavelet: target must be in (0, 1]")
    H, W = np.asarray(img).shape
    c = vec_image(haar2_forward(img))
    keep = round_half_away(target * c.size)
    order = np.argsort(-np.abs(c), kind="stable")
    kept = np.zeros_like(c)
    sel = order[: min(keep, c.size)]
    kept[sel] = c[sel]
    return haar2_inverse(unvec_image(kept, H, W)), kept


def make_mask(H, W, M, seed):
    """mri.cpp:185-207: partial Fisher-Yates over [0, HW) with the reference Rng,
    first M sorted."""
    N = H * W
    if H < 1 or W < 1:
        raise InputError("make_mask: dims must be >= 1")
    if M < 1 or M > N:
        raise InputError("make_mask: M out of range")
    pool = list(range(N))
    rng = Rng(seed)
    for i in range(M):
        pick = i + rng.uniform_below(N - i)
        pool[i], pool[pick] = pool[pick], pool[i]
    return np.array(sorted(pool[:M]), np.int64)


class MriTransform:
    """MriTransform, mri.hpp:56-99 / mri.cpp:209-322."""

    def __init__(self, target_image, mask, gamma):
        img = np.asarray(target_image, np.float64)
        self.H, self.W = img.shape
        if not (_pow2(self.H) and _pow2(self.W)):
            raise InputError("MriTransform: dimensions must be powers of two")
        if gamma < 0.0:
            raise InputError("MriTransform: gamma must be >= 0")
        idx = np.sort(np.asarray(mask, np.int64))
        if idx.size == 0 or idx[0] < 0 or idx[-1] >= self.H * self.W or np.any(np.diff(idx) == 0):
            raise InputError("MriTransform: mask indices must be unique and in range")
        self.mask = idx
        self.gamma = float(gamma)
        self.N = self.H * self.W
        self.y = self._dft2(img).reshape(-1)[idx]                      # :232-235
        self.hz = vec_image(haar2_forward(self._idft2_masked_real(self.y)))  # :236
        self._diag = None

    @property
    def diag(self):
        """mri.cpp:238-254 (one apply per basis vector; computed on first use)."""
        if self._diag is None:
            self._diag = np.array([self.apply_full(e)[r] for r, e in self._basis()])
        return self._diag

    def _basis(self):
        e = np.zeros(self.N)
        for r in range(self.N):
            e[r] = 1.0
            yield r, e
            e[r] = 0.0

    def _dft2(self, real_img):
        """mri.cpp:258-272: unitary forward 2-D DFT."""
        return np.fft.fft2(np.asarray(real_img, np.float64)) / math.sqrt(self.H * self.W)

    def _idft2_masked_real(self, kvec):
        """mri.cpp:274-288: scatter onto the mask, unitary inverse, real part."""
        K = np.zeros(self.N, np.complex128)
        K[self.mask] = kvec
        return (np.fft.ifft2(K.reshape(self.H, self.W)) * math.sqrt(self.H * self.W)).real

    def forward(self, coeffs):
        """mri.cpp:290-297: A x (masked k-space)."""
        coeffs = np.asarray(coeffs, np.float64)
        if coeffs.size != self.N:
            raise InputError("MriTransform::forward: length mismatch")
        return self._dft2(haar2_inverse(unvec_image(coeffs, self.H, self.W))).reshape(-1)[self.mask]

    def apply_fit(self, coeffs):
        """mri.cpp:299-301: Re(A^H A) x."""
        return vec_image(haar2_forward(self._idft2_masked_real(self.forward(coeffs))))

    def apply_full(self, coeffs):
        """mri.cpp:303-315: G x."""
        coeffs = np.asarray(coeffs, np.float64)
        if coeffs.size != self.N:
            raise InputError("MriTransform::apply_full: length mismatch")
        B = haar2_inverse(unvec_image(coeffs, self.H, self.W))
        img = self._idft2_masked_real(self._dft2(B).reshape(-1)[self.mask])
        if self.gamma > 0.0:
            img = img + self.gamma * (second_diff_cols(second_diff_cols(B)) +
                                      second_diff_rows(second_diff_rows(B)))
        return vec_image(haar2_forward(img))

    def fit_error(self, coeffs):
        """mri.cpp:317-319."""
        d = self.y - self.forward(coeffs)
        return 0.5 * float(np.vdot(d, d).real)


def assemble_operators(target_image, mask, gamma):
    """mri.cpp:327-343: explicit J (columns G e_r) and hz."""
    t = MriTransform(target_image, mask, gamma)
    J = np.zeros((t.N, t.N))
    for r, e in t._basis():
        J[:, r] = t.apply_full(e)
    return J, t.hz.copy(), t


def lasso_normal_form(applyG, hz, lambda_l1=3e-4, max_iters=5000, tol=1e-8, step=1.0):
    """mri.cpp:345-370: FISTA on 1/2 x'Gx - hz.x + lambda ||x||_1."""
    if lambda_l1 < 0.0:
        raise InputError("lasso: lambda_l1 must be >= 0")
    if not step > 0.0:
        raise InputError("lasso: step must be > 0")
    hz = np.asarray(hz, np.float64)
    x = np.zeros_like(hz)
    z = x.copy()
    t, f_prev = 1.0, 0.0
    for _ in range(max_iters):
        grad = applyG(z) - hz
        x_next = soft_threshold(z - step * grad, step * lambda_l1)
        t_next = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * t * t))
        z = x_next + ((t - 1.0) / t_next) * (x_next - x)
        x = x_next
        t = t_next
        f = 0.5 * float(x @ applyG(x)) - float(hz @ x) + lambda_l1 * float(np.abs(x).sum())
        if abs(f - f_prev) <= tol * max(1.0, abs(f_prev)):
            break
        f_prev = f
    return x


def lasso_init(t: MriTransform, lambda_l1, **kw):
    """mri.cpp:372-377."""
    return lasso_normal_form(t.apply_fit, t.hz, lambda_l1, **kw)
