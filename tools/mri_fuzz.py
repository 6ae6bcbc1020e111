"""Random sizes / masks / gamma for the matrix-free MRI chain: assembled G columns, hz, diag
vs the numpy oracle of mri.cpp (oracle/mri.py), tolerance 2e-5 of the compared quantity's
scale; unsupported shapes must raise a clean error.  Run on the B200 box."""
from __future__ import annotations
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_00366_b200 as P  # noqa: E402
from oracle import mri as Mr  # noqa: E402  (the checker)


def run(cases, seed):
    rng = np.random.default_rng(seed)
    bad = 0
    for ci in range(cases):
        H = int(rng.choice([4, 8, 16, 32, 64, 128]))
        W = int(rng.choice([4, 8, 16, 32, 64, 128]))
        if H * W > 2048:
            H, W = min(H, 32), min(W, 64)
        M = int(rng.integers(max(2, H * W // 10), H * W + 1))
        gamma = float(rng.choice([0.0, 1e-4, 1e-3, 1e-2]))
        tag = f"case {ci}: {H}x{W} M={M} gamma={gamma}"
        try:
            img = Mr.phantom_image(H, W)
            mask = Mr.make_mask(H, W, M, int(rng.integers(1, 1000)))
            J, hz, t = Mr.assemble_operators(img, mask, gamma)
            with P.Context(0, "f32") as ctx:
                ctx.set_mri_problem(img, mask, gamma, None)
                ctx.build_coupling()
                G, ghz, gD = ctx.get_coupling(0)
            e = [np.max(np.abs(G - J)) / np.max(np.abs(J)),
                 np.max(np.abs(ghz - hz)) / max(np.max(np.abs(hz)), 1e-30),
                 np.max(np.abs(gD - t.diag)) / np.max(np.abs(t.diag))]
            ok = all(x <= 2e-5 for x in e)
            msg = ("OK " if ok else "MISMATCH ") + " ".join(f"{x:.1e}" for x in e)
            bad += not ok
        except (P.ConfigError, P.InputError) as ex:
            msg = "rejected cleanly: " + str(ex)[:80]
        except Exception as ex:  # noqa: BLE001
            msg = "ERROR " + str(ex)[:140]
            bad += 1
        print(tag, "->", msg, flush=True)
    return bad


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    bad = run(n, int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    print("bad:", bad)
    sys.exit(1 if bad else 0)
