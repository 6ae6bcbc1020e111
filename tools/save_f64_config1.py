"""fp64 GPU solve of BASELINE config 1 saved for tools/literal_study.py (gpurun side)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_00366_b200 as P  # noqa: E402
from paper_2405_00366_b200 import workloads as W  # noqa: E402

insts, R, hp, _ = W.config1(0, 64)
seeds = P.replica_seeds(insts, R, "mfz-bn")
with P.Context(0, "f64") as ctx:
    ctx.set_problems(insts)
    ctx.build_coupling()
    res = ctx.solve(R, "mfz-bn", hp, seeds)
    order = ctx.canon_order()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", "f64_config1_sym64.npz"), R=res["R"],
                    sigma=res["sigma"], seeds=seeds, order=np.array(order))
print("saved", order)
