"""Driver for ncu captures of the symmetric-tile step kernels: fused Euler steps
(cimcs_mfz_step) on config-1-shaped instances (B instances, 16 replicas), then a
short solve.  argv: B, dtype (f32 -> sym_step_kernel, f64 -> sym64_step_kernel),
repetitions."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

import paper_2405_00366_b200 as P

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dtype = sys.argv[2] if len(sys.argv) > 2 else "f32"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
insts = P.gen_instances(2000, [(0.5, 0.1, 0.01, s) for s in range(1, B + 1)])
ctx = P.Context(0, dtype)
ctx.set_option("pdl", int(os.environ.get("PDL", "1")))
ctx.set_problems(insts)
ctx.build_coupling()
R = 16
rng = np.random.default_rng(1)
Rs = rng.normal(size=(B, R, 2000))
c = rng.normal(scale=0.5, size=(B, R, 2000))
e = np.ones((B, R, 2000))
hp = P.baseline_params()
for _ in range(reps):
    out = ctx.mfz_step(R, "mfz-bn", hp, 0.5, 0.9, Rs, c, e)
res = ctx.solve(R, "mfz-bn", P.baseline_params(velo=1, n_steps=200), P.replica_seeds(insts, R, "mfz-bn"))
t = ctx.timing()
print(dtype, "per-step us", 1e3 * t["cim_ms"] / 400, "refit per sweep us", 1e3 * t["refit_ms"] / 200)
ctx.close()
