"""Host-side preparation of the MRI transform-chain problem (the data the
reference's cmd_mri builds before MriTransform, tools/main.cpp:506-560):
phantom image (mri.cpp:415-437), orthonormal multi-level Haar in the Mallat
layout (mri.cpp:122-165), wavelet sparsification (mri.cpp:167-183) and the
k-space sampling mask (mri.cpp:185-207, through the C ABI's reference RNG).
The per-step chain itself runs matrix-free on the GPU (csrc/mri_kernels.cuh,
Context.set_mri_problem)."""
from __future__ import annotations

import math

import numpy as np

from ._lib import load
from .cimcs import InputError, _check

_S = 1.0 / math.sqrt(2.0)


def _pow2(v):
    return v >= 1 and (v & (v - 1)) == 0


def phantom_image(H: int, W: int) -> np.ndarray:
    """mri.cpp:415-437: deterministic blobs + edges, clamped to [0, 1] (scalar
    libm exp, as the reference evaluates it)."""
    if H < 1 or W < 1:
        raise InputError("phantom_image: dims must be >= 1")
    img = np.zeros((H, W))
    exp = math.exp
    for i in range(H):
        v = (i + 0.5) / H
        for j in range(W):
            u = (j + 0.5) / W
            val = 0.08 + 0.10 * u
            val += 0.55 * exp(-((u - 0.35) * (u - 0.35) + (v - 0.40) * (v - 0.40)) / 0.020)
            val += 0.40 * exp(-((u - 0.72) * (u - 0.72) + (v - 0.68) * (v - 0.68)) / 0.008)
            if 0.55 < u < 0.88 and 0.12 < v < 0.34:
                val += 0.30
            if (u - 0.28) * (u - 0.28) + (v - 0.78) * (v - 0.78) < 0.016:
                val += 0.35
            img[i, j] = min(max(val, 0.0), 1.0)
    return img


def haar2_forward(img) -> np.ndarray:
    """mri.cpp:122-141: per level, split the rows then the columns."""
    X = np.array(img, np.float64)
    H, W = X.shape
    if not (_pow2(H) and _pow2(W)):
        raise InputError("haar2_forward: dimensions must be powers of two")
    h, w = H, W
    while h >= 2 and w >= 2:
        a, b = X[:h, 0:w:2].copy(), X[:h, 1:w:2].copy()
        X[:h, : w // 2], X[:h, w // 2: w] = (a + b) * _S, (a - b) * _S
        a, b = X[0:h:2, :w].copy(), X[1:h:2, :w].copy()
        X[: h // 2, :w], X[h // 2: h, :w] = (a + b) * _S, (a - b) * _S
        h //= 2
        w //= 2
    return X


def haar2_inverse(C) -> np.ndarray:
    """mri.cpp:143-165: deepest level first, merge the columns then the rows."""
    X = np.array(C, np.float64)
    H, W = X.shape
    if not (_pow2(H) and _pow2(W)):
        raise InputError("haar2_inverse: dimensions must be powers of two")
    levels = []
    h, w = H, W
    while h >= 2 and w >= 2:
        levels.append((h, w))
        h //= 2
        w //= 2
    for h, w in reversed(levels):
        a, b = X[: h // 2, :w].copy(), X[h // 2: h, :w].copy()
        X[0:h:2, :w], X[1:h:2, :w] = (a + b) * _S, (a - b) * _S
        a, b = X[:h, : w // 2].copy(), X[:h, w // 2: w].copy()
        X[:h, 0:w:2], X[:h, 1:w:2] = (a + b) * _S, (a - b) * _S
    return X


def _round_half_away(v: float) -> int:
    """datagen.cpp:11-13."""
    return int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))


def sparsify_wavelet(img, target: float):
    """mri.cpp:167-183 -> (image, coeffs): keep the round(target N) largest
    |coefficients|, ties to the lower linear index."""
    if not (target > 0.0) or target > 1.0:
        raise InputError("sparsify_wavelet: target must be in (0, 1]")
    H, W = np.asarray(img).shape
    c = haar2_forward(img).reshape(-1)
    keep = min(_round_half_away(target * c.size), c.size)
    order = np.argsort(-np.abs(c), kind="stable")
    kept = np.zeros_like(c)
    kept[order[:keep]] = c[order[:keep]]
    return haar2_inverse(kept.reshape(H, W)), kept


def make_mask(H: int, W: int, M: int, seed: int) -> np.ndarray:
    """mri.cpp:185-207 (reference RNG stream, host C++)."""
    out = np.zeros(max(M, 0), np.int32)
    _check(load().cimcs_make_mask(H, W, M, seed, out.ctypes.data if M > 0 else None))
    return out


def problem(size: int = 128, sparseness: float = 0.1, compression: float = 0.4,
            seed: int = 1):
    """The cmd_mri inputs for one mask (tools/main.cpp:506-560): phantom ->
    sparsified target (image, coeffs), M = round(compression N) mask."""
    img, coeffs = sparsify_wavelet(phantom_image(size, size), sparseness)
    M = _round_half_away(compression * size * size)
    return img, coeffs, make_mask(size, size, M, seed)
