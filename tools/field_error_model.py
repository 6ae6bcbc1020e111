"""Error model of the fp32 tensor-core local field (numpy emulation, CPU).

Emulates the symmetric-tile contraction of sym_kernels.cuh at BASELINE config-1
shape: fp16 hi/lo splits of the scaled gram and of w, fp32 MMA accumulators per
128-row tile (one rounding per K=16 MMA), fp32 tile / slot partial sums and the
fp32 update (D w - G w), against the exact fp64 field; then the same with the
diagonal removed from the tiles and with fp64 partial sums.  Compared with the
oracle's precision study (profiles/r02_precision_study*.json: a per-element
relative field error of 2^-20 keeps every fp64 support, 2^-16 loses 25 %).
  python tools/field_error_model.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

f16, f32 = np.float16, np.float32


def split16(x, e):
    xs = np.ldexp(x, e)
    hi = xs.astype(f16).astype(np.float64)
    lo = (xs - hi).astype(f16).astype(np.float64)
    return hi, lo


def field(G, D, hz, w, zero_diag=False, f64_partials=False, T=128, K=16):
    N = G.shape[0]
    sG = 14 - int(np.floor(np.log2(np.max(np.abs(D)))))
    Gm = G.copy()
    if zero_diag:
        np.fill_diagonal(Gm, 0.0)
    gw = np.zeros(N, np.float64 if f64_partials else f32)
    nb = -(-N // T)
    for J in range(nb):
        j0, j1 = J * T, min(N, J * T + T)
        wb = w[j0:j1]
        m = np.max(np.abs(wb))
        ew = 0 if m == 0 else 14 - int(np.floor(np.log2(m)))
        w_hi, w_lo = split16(wb, ew)
        Ghi, Glo = split16(Gm[:, j0:j1], sG)
        a1 = np.zeros(N, f32)
        a2 = np.zeros(N, f32)
        for k0 in range(0, j1 - j0, K):
            sl = slice(k0, k0 + K)
            c1 = Ghi[:, sl] @ w_hi[sl] + Glo[:, sl] @ w_hi[sl]
            c2 = Ghi[:, sl] @ w_lo[sl]
            a1 = (a1.astype(np.float64) + c1).astype(f32)
            a2 = (a2.astype(np.float64) + c2).astype(f32)
        t = (a1.astype(np.float64) + a2.astype(np.float64))
        t = np.ldexp(t, -(sG + ew))
        if f64_partials:
            gw = gw + t
        else:
            gw = (gw.astype(np.float64) + t.astype(f32)).astype(f32)
    if zero_diag:
        Jw = -gw.astype(np.float64)
        return 0.5 * (Jw + hz)
    if f64_partials:
        Jw = D * w - gw
    else:
        Jw = (D.astype(f32) * w.astype(f32) - gw.astype(f32)).astype(np.float64)
    return 0.5 * (Jw + hz)


def main():
    inst = O.gen_instance(2000, 0.5, 0.1, 0.01, 1)
    p = O.Problem(inst, O.CANON)
    G, D, hz = p.G, p.gram_diag, p.hz
    rng = np.random.default_rng(0)
    out = {}
    for frac in (0.1, 0.3):
        sig = (rng.random(2000) < frac).astype(np.float64)
        R = hz + 0.1 * rng.normal(size=2000)
        w = R * sig
        exact = 0.5 * (D * w - G @ w + hz)
        for name, kw in (("current", {}), ("zero_diag", dict(zero_diag=True)),
                         ("f64_partials", dict(f64_partials=True)),
                         ("zero_diag+f64_partials", dict(zero_diag=True, f64_partials=True))):
            h = field(G, D, hz, w, **kw)
            rel = np.abs(h - exact) / np.maximum(np.abs(exact), 1e-300)
            out[f"active={frac}:{name}"] = {
                "max_err_over_max_h": float(np.max(np.abs(h - exact)) / np.max(np.abs(exact))),
                "median_rel": float(np.median(rel)), "p90_rel": float(np.quantile(rel, 0.9)),
                "log2_median_rel": float(np.log2(np.median(rel)))}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
