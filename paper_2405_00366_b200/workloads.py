"""Input generators for the BASELINE.json configurations (host side).

Configs 0-2 and 4 use the reference's own generator (`gen_instance`,
datagen.cpp:15-55, bit-identical stream) with the seeding of the reference CLI
(`instance_grid`, tools/main.cpp:335-344).  Config 3 has no counterpart in the
reference (its MRI path uses a complex DFT, full-depth Haar and a blob
phantom, mri.cpp:121-141,272-287,421-437); it is the synthetic stand-in that
BASELINE.json describes for the fastMRI image, built here:

* image: 128 x 128, 10 ellipses painted in order (later ones on top),
  centres U[-0.7,0.7]^2, semi-axes U[0.05,0.45], angle U[0,pi), intensity U[0,1];
* unknowns w: 3-level orthonormal Mallat 2-D Haar coefficients of the image
  (the reference's average/difference split, mri.cpp:30-48, stopped at 3
  levels), flattened row-major -> N = 16384, naturally sparse;
* A = S * DCT2 * Haar3^{-1}: row m = Haar3(phi_uv) for M = round(0.4 N) = 6554
  frequencies (u, v) drawn without replacement, phi_uv the orthonormal 2-D
  DCT-II basis image; y = A w + N(0, 0.005^2);
* xi = (w != 0), x_true = w.
All randomness comes from numpy's PCG64 seeded with `seed`.
"""
from __future__ import annotations

import math

import numpy as np

from .cimcs import HyperParams, Instance, baseline_params, gen_instances


def config0():
    """CPU reference workload: N=500, M=300, K=100, 1 replica, fp64, seed 0."""
    return gen_instances(500, [(0.6, 0.2, 0.01, 0)]), 1, baseline_params(), "f64"


def config1(rank: int = 0, B: int = 64):
    """Paper scale: 64 instances N=2000, alpha 0.5, a 0.1, nu 0.01; 16 replicas."""
    seeds = [1 + rank * B + s for s in range(B)]
    return gen_instances(2000, [(0.5, 0.1, 0.01, s) for s in seeds]), 16, baseline_params(), "f32"


def config2_grid(trials: int = 32, seed_base: int = 1):
    """instance_grid order alpha -> a -> nu -> trial (tools/main.cpp:335-344)."""
    grid, idx = [], 0
    for alpha in (0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9):
        for a in (0.05, 0.1, 0.15, 0.2, 0.25, 0.3):
            for _ in range(trials):
                grid.append((alpha, a, 0.01, seed_base + idx))
                idx += 1
    return grid


def config2(trials: int = 32, shard=None):
    """Phase sweep: 7 alpha x 6 a x 32 trials at N=2000, 8 replicas."""
    grid = config2_grid(trials)
    if shard is not None:
        grid = [grid[k] for k in shard]
    return gen_instances(2000, grid), 8, baseline_params(), "f32"


def _dct_matrix(n: int) -> np.ndarray:
    k = np.arange(n)[:, None]
    x = np.arange(n)[None, :]
    C = np.cos(math.pi * (2 * x + 1) * k / (2 * n)) * math.sqrt(2.0 / n)
    C[0] /= math.sqrt(2.0)
    return C  # rows = orthonormal DCT-II basis vectors


def haar2(img: np.ndarray, levels: int) -> np.ndarray:
    """Mallat 2-D Haar (rows then columns per level), orthonormal split of
    mri.cpp:30-48; works on a batch [..., h, w]."""
    X = np.array(img, dtype=np.float64, copy=True)
    s = 1.0 / math.sqrt(2.0)
    h, w = X.shape[-2], X.shape[-1]
    for _ in range(levels):
        blk = X[..., :h, :w]
        a = (blk[..., :, 0::2] + blk[..., :, 1::2]) * s
        d = (blk[..., :, 0::2] - blk[..., :, 1::2]) * s
        X[..., :h, :w] = np.concatenate([a, d], axis=-1)
        blk = X[..., :h, :w]
        a = (blk[..., 0::2, :] + blk[..., 1::2, :]) * s
        d = (blk[..., 0::2, :] - blk[..., 1::2, :]) * s
        X[..., :h, :w] = np.concatenate([a, d], axis=-2)
        h //= 2
        w //= 2
    return X


def ellipse_phantom(n: int, count: int, rng: np.random.Generator) -> np.ndarray:
    yy, xx = np.meshgrid(np.linspace(-1, 1, n), np.linspace(-1, 1, n), indexing="ij")
    img = np.zeros((n, n))
    for _ in range(count):
        cx, cy = rng.uniform(-0.7, 0.7, 2)
        ax, ay = rng.uniform(0.05, 0.45, 2)
        th = rng.uniform(0, math.pi)
        val = rng.uniform(0, 1)
        u = (xx - cx) * math.cos(th) + (yy - cy) * math.sin(th)
        v = -(xx - cx) * math.sin(th) + (yy - cy) * math.cos(th)
        img[(u / ax) ** 2 + (v / ay) ** 2 <= 1.0] = val
    return img


def config3(seed: int = 3, n: int = 128, levels: int = 3, alpha: float = 0.4,
            noise: float = 0.005):
    """MRI-shaped synthetic workload (see module docstring): 1 instance, 16 replicas."""
    rng = np.random.Generator(np.random.PCG64(seed))
    img = ellipse_phantom(n, 10, rng)
    w = haar2(img, levels).reshape(-1)
    N = n * n
    M = int(math.floor(alpha * N + 0.5))
    freqs = rng.choice(N, size=M, replace=False)
    C = _dct_matrix(n)
    A = np.empty((M, N), order="F")
    for s in range(0, M, 512):
        f = freqs[s:s + 512]
        phi = C[f // n][:, :, None] * C[f % n][:, None, :]  # basis images phi_uv
        A[s:s + len(f)] = haar2(phi, levels).reshape(len(f), N)
    y = A @ w + noise * rng.standard_normal(M)
    xi = (w != 0).astype(np.int32)
    inst = Instance(A, y, w.copy(), xi, float(xi.mean()), alpha, noise, seed)
    return [inst], 16, baseline_params(), "f32"


def config3_chain(seed: int = 3, n: int = 128, levels: int = 3, alpha: float = 0.4,
                  noise: float = 0.005):
    """Config 3 without its dense matrix: (n, levels, freqs, y, w) for
    Context.set_dct_problem.  Same draws as config3 (same phantom, frequencies
    and noise); y = S C2 w_image + noise evaluated by fast transforms."""
    rng = np.random.Generator(np.random.PCG64(seed))
    img = ellipse_phantom(n, 10, rng)
    w = haar2(img, levels).reshape(-1)
    N = n * n
    M = int(math.floor(alpha * N + 0.5))
    freqs = rng.choice(N, size=M, replace=False)
    C = _dct_matrix(n)
    spec = (C @ ihaar2(w.reshape(n, n), levels) @ C.T).reshape(-1)
    y = spec[freqs] + noise * rng.standard_normal(M)
    return n, levels, freqs.astype(np.int32), y, w.copy()


def ihaar2(X: np.ndarray, levels: int) -> np.ndarray:
    """Inverse of haar2 (column merge then row merge per level, coarsest first)."""
    X = np.array(X, dtype=np.float64, copy=True)
    s = 1.0 / math.sqrt(2.0)
    n0, m0 = X.shape[-2], X.shape[-1]
    for lev in range(levels - 1, -1, -1):
        h, w = n0 >> lev, m0 >> lev
        blk = X[..., :h, :w].copy()
        a, d = blk[..., : h // 2, :], blk[..., h // 2:, :]
        out = np.empty_like(blk)
        out[..., 0::2, :] = (a + d) * s
        out[..., 1::2, :] = (a - d) * s
        a, d = out[..., :, : w // 2], out[..., :, w // 2:]
        out2 = np.empty_like(out)
        out2[..., :, 0::2] = (a + d) * s
        out2[..., :, 1::2] = (a - d) * s
        X[..., :h, :w] = out2
    return X


def config4(N: int = 100_000, seed: int = 7):
    """Strong-scaling workload: gen_instance(N, 0.5, 0.05, 0.01, 7), 4 replicas,
    10 alternations x 500 steps.  (Host generation of the 5e9-draw reference
    stream takes minutes at full size; N can be reduced for tests.)"""
    hp = HyperParams(dt=0.01, n_steps=500, velo=9, pump_kind=1, pump_end=1.2)
    return gen_instances(N, [(0.5, 0.05, 0.01, seed)]), 4, hp, "f32"
