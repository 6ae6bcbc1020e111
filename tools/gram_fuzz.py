"""gram_tc_kernel (tcgen05 gram, forced with option gram_tc = 1) on odd sizes: the
assembled G vs A^T A in numpy fp64, tolerance 1e-6 of max |G|; covers ragged last
blocks, partial super-blocks (12 x 12 tiles) and several k-chunk counts.  B200 box."""
from __future__ import annotations
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_00366_b200 as P  # noqa: E402

bad = 0
for N, alpha, seeds in ((129, 0.5, (1,)), (1537, 0.33, (1, 2)), (1665, 0.9, (3,)), (3001, 0.5, (4,)),
                        (4737, 0.21, (5,)), (8192, 0.5, (6,)), (9001, 0.4, (7,))):
    insts = [P.gen_instance(N, alpha, 0.1, 0.01, s) for s in seeds]
    with P.Context(0, "f32") as ctx:
        ctx.set_option("gram_tc", 1)
        ctx.set_problems(insts)
        ctx.build_coupling()
        tm = ctx.timing()["gram_ms"]
        for b, inst in enumerate(insts):
            G, hz, D = ctx.get_coupling(b)
            A = np.asfortranarray(inst.A)
            ref = A.T @ A
            err = float(np.max(np.abs(G - ref)) / np.max(np.abs(ref)))
            ok = err <= 1e-6 and np.allclose(D, np.diag(ref), rtol=1e-6)
            bad += not ok
            print(f"N={N} M={inst.M} nRB={-(-N // 128)} instance {b}: max err {err:.2e} "
                  f"{'OK' if ok else 'BAD'} (gram {tm:.1f} ms)", flush=True)
print("bad:", bad)
sys.exit(1 if bad else 0)
