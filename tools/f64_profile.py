"""Driver for ncu captures / timing of the fp64 CUDA-core step kernel on
config-1 shapes (B instances, 16 replicas, N = 2000)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2405_00366_b200 as P

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
insts = P.gen_instances(2000, [(0.5, 0.1, 0.01, s) for s in range(1, B + 1)])
ctx = P.Context(0, "f64")
ctx.set_problems(insts)
ctx.build_coupling()
R = 16
rng = np.random.default_rng(1)
Rs = rng.normal(size=(B, R, 2000))
c = rng.normal(scale=0.5, size=(B, R, 2000))
for _ in range(3):
    ctx.mfz_step(R, "mfz-bn", P.baseline_params(), 0.5, 0.9, Rs, c, np.ones((B, R, 2000)))
res = ctx.solve(R, "mfz-bn", P.baseline_params(velo=1, n_steps=100), P.replica_seeds(insts, R, "mfz-bn"))
t = ctx.timing()
print("f64 per-step us", 1e3 * t["cim_ms"] / 200)
ctx.close()
