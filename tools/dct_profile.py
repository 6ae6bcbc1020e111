"""Config-3 matrix-free chain: a few eager Euler steps for ncu
(ncu -k regex:dct_cluster python tools/dct_profile.py)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_00366_b200 as P  # noqa: E402
from paper_2405_00366_b200 import workloads  # noqa: E402


def main():
    n, L, f, y, w = workloads.config3_chain()
    R, N = 16, n * n
    rng = np.random.default_rng(0)
    Rs = rng.normal(size=(1, R, N)) * (rng.random((1, R, N)) < 0.2)
    c = rng.normal(scale=0.5, size=(1, R, N))
    with P.Context(0, "f32") as ctx:
        ctx.set_dct_problem(n, L, f, y, w)
        ctx.build_coupling()
        for _ in range(3):
            ctx.mfz_step(R, "mfz-bn", P.HyperParams(), 0.3, 0.9, Rs, c, np.ones((1, R, N)))
    print("ok")


if __name__ == "__main__":
    main()
