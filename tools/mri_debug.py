"""Debug helper: GPU transform-chain operator vs the oracle for one shape."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2405_00366_b200 as P
from oracle import mri as Mr

for H, W, gamma in [(16, 16, 0.0), (8, 32, 0.0), (32, 8, 0.0), (8, 8, 0.0), (4, 4, 0.0)]:
    img = Mr.phantom_image(H, W)
    mask = Mr.make_mask(H, W, H * W // 2, 11)
    J, hz, t = Mr.assemble_operators(img, mask, gamma)
    with P.Context(0, "f32") as ctx:
        ctx.set_mri_problem(img, mask, gamma)
        ctx.build_coupling()
        G, ghz, gD = ctx.get_coupling(0)
    print(H, W, "G err", np.abs(G - J).max(), "Jmax", np.abs(J).max(), "Gmax", np.abs(G).max(),
          "hz err", np.abs(ghz - hz).max(), "D err", np.abs(gD - t.diag).max())
