"""Tiny workloads that launch every kernel family once, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per gpurun call):
  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
Covers: the fp64 DMMA symmetric path (steps, Jacobi, CG, score), the fp32
tcgen05 symmetric path, the fp32 / fp64 CUDA-core grid kernels, the small-N
cluster loop, Positive-P, the matrix-free MRI chain and the gram builders.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2405_00366_b200 as P  # noqa: E402
from paper_2405_00366_b200 import mri as PM  # noqa: E402

hp = P.baseline_params(velo=1, n_steps=20)


def solve(dtype, N, R, B=2, cdp="jacobi", **opts):
    insts = P.gen_instances(N, [(0.5, 0.1, 0.01, s) for s in range(1, B + 1)])
    with P.Context(0, dtype) as ctx:
        for k, v in opts.items():
            ctx.set_option(k, v)
        ctx.set_problems(insts)
        ctx.build_coupling()
        res = ctx.solve(R, "mfz-bn", hp, P.replica_seeds(insts, R, "mfz-bn"), cdp=cdp)
    assert (res["fail_alt"] < 0).all()
    print(dtype, N, R, cdp, opts, "ok", flush=True)


solve("f64", 600, 16)                      # sym64 DMMA path
solve("f64", 600, 3, cdp="cg")             # sym64, NR 8, CG refit
solve("f32", 640, 16)                      # tcgen05 symmetric path
solve("f32", 640, 8, cdp="cg")
solve("f32", 300, 16)                      # fp32 CUDA-core grid kernel
solve("f64", 700, 4, sym64=0)              # fp64 CUDA-core grid kernel
solve("f64", 256, 2)                       # cluster loop
solve("f32", 256, 8)
insts = P.gen_instances(200, [(0.6, 0.2, 0.01, 1)])
with P.Context(0, "f64") as ctx:            # Positive-P (host noise chunks)
    ctx.set_problems(insts)
    ctx.build_coupling()
    ctx.solve(2, "pp", P.baseline_params(velo=1, n_steps=70), P.replica_seeds(insts, 2, "pp"))
print("pp ok", flush=True)
img, coeffs, mask = PM.problem(16, 0.1, 0.4, 1)
with P.Context(0, "f32") as ctx:            # matrix-free MRI chain
    ctx.set_mri_problem(img, mask, 1e-4, coeffs)
    ctx.build_coupling()
    x0, _, _ = ctx.mri_lasso(3e-4, max_iters=50)
    ctx.solve(8, "mfz-bn", hp, np.array([[P.mix_seed(1, 1 + 3 * r) for r in range(8)]], np.uint64),
              R_init=np.broadcast_to(x0, (1, 8, 256)).copy(), cdp="cg")
print("mri ok", flush=True)
