"""Time the matrix-free MRI step (config-3 image size, 16 replicas): one
fused Euler step = mri_kernel (G w, one CTA per replica) + sym_update_kernel."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2405_00366_b200 as P
from paper_2405_00366_b200 import mri as PM

size = int(sys.argv[1]) if len(sys.argv) > 1 else 128
R = int(sys.argv[2]) if len(sys.argv) > 2 else 16
img, coeffs, mask = PM.problem(size, 0.1, 0.4, 1)
ctx = P.Context(0, "f32")
ctx.set_option("mri_cluster", int(os.environ.get("MRI_CLUSTER", "1")))
ctx.set_mri_problem(img, mask, 1e-4, coeffs)
t0 = time.perf_counter()
ctx.build_coupling()
print("build (hz + diag) ms", 1e3 * (time.perf_counter() - t0), "device", ctx.timing()["gram_ms"])
seeds = P.replica_seeds([P.Instance(np.zeros((1, size * size)), np.zeros(1), seed=1)], R, "mfz-bn")
hp = P.baseline_params(velo=1, n_steps=200)
for _ in range(2):
    res = ctx.solve(R, "mfz-bn", hp, seeds)
t = ctx.timing()
print("size", size, "R", R, "per-step us", 1e3 * t["cim_ms"] / 400, "refit ms", t["refit_ms"],
      "score ms", t["score_ms"])
ctx.close()
